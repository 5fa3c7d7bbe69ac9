"""A/B of the PowerSGD P = M Q pass: tcgen05 (default) vs CUDA cores (GC_PSGD_MQ=cores).
python tools/time_mq.py [d] [n] -> per-impl ms/round and the relative difference of the estimates."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2407_01378_b200 as gcb

d = int(sys.argv[1]) if len(sys.argv) > 1 else 350_000_000
n = int(sys.argv[2]) if len(sys.argv) > 2 else 8
torch.manual_seed(0)
g = torch.randn(n, d, device="cuda")
ests = {}
for impl in ("cores", "umma"):
    os.environ["GC_PSGD_MQ"] = impl
    pipe = gcb.make_pipeline(gcb.PowerSgdConfig(4), n, d, gcb.SeedSpec(2024), validate=False, compute_nmse=False)
    r0 = pipe.run_round(g, 0)
    ests[impl] = r0.estimate_tensor.clone()
    pipe.run_round(g, 1)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for r in range(5):
        pipe.run_round(g, 2 + r)
    e.record()
    torch.cuda.synchronize()
    print(f"{impl}: {s.elapsed_time(e) / 5:.3f} ms/round", flush=True)
    del pipe
a, b = ests["cores"].double(), ests["umma"].double()
print("rel diff (norm):", float((a - b).norm() / a.norm()), " max:", float((a - b).abs().max() / a.abs().max()))
