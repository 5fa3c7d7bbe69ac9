"""Kernel timeline of a few pipeline rounds (torch.profiler / CUPTI): per-round device busy time,
idle gaps between kernels, and the largest gaps.  python tools/timeline.py <psgd_gpt2m|topk|thc> [rounds]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile
import paper_2407_01378_b200 as gcb

name = sys.argv[1]
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 3
n = 8
if name == "psgd_gpt2m":
    from paper_2407_01378_b200.multitensor import TensorListPipeline, gpt2_medium_sizes
    sizes = gpt2_medium_sizes()
    d = sum(sizes)
    pipe = TensorListPipeline(gcb.PowerSgdConfig(4), n, sizes, gcb.SeedSpec(2024), validate=False, compute_nmse=False)
else:
    d, cfg = {"topk": (110_000_000, gcb.TopKConfig(1_100_000)), "thc": (25_557_032, gcb.RotatedQuantConfig(4, 8)),
              "psgd": (350_000_000, gcb.PowerSgdConfig(4)),
              "topkc": (110_000_000, gcb.ChunkedTopKConfig(64, 17_187)),
              "dense16": (25_557_032, gcb.DenseConfig(16))}[name]
    pipe = gcb.make_pipeline(cfg, n, d, gcb.SeedSpec(2024), validate=False, compute_nmse=False)
g = torch.randn(n, d, device="cuda")
for r in range(3):
    pipe.run_round(g, r)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for r in range(3, 3 + rounds):
        pipe.run_round(g, r)
    torch.cuda.synchronize()
ev = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA],
            key=lambda e: e.time_range.start)
start, end = ev[0].time_range.start, max(e.time_range.end for e in ev)
busy, gaps, last = 0, [], start
for e in ev:
    s, t = e.time_range.start, e.time_range.end
    if s > last:
        gaps.append((s - last, e.name[:60]))
    busy += t - s
    last = max(last, t)
span = end - start
print(f"{name}: {rounds} rounds, span {span/1e3/rounds:.3f} ms/round, kernels busy {busy/1e3/rounds:.3f} ms/round, "
      f"idle {sum(x for x, _ in gaps)/1e3/rounds:.3f} ms/round in {len(gaps)} gaps")
for gsz, nm in sorted(gaps, reverse=True)[:12]:
    print(f"  gap {gsz:8.1f} us before {nm}")
