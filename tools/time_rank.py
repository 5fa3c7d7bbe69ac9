"""Per-rank round timing (DistributedGradientPipeline on a one-rank NCCL group).

python tools/time_rank.py [--scheme thc|psgd|psgd_gpt2|fp16] [--d 350000000] [--n 1] [--q 4 --b 8]
                          [--segs 1024,4096,...] [--steps 10]
One JSON line per configuration: ms/round (CUDA events), Gelem/s, algorithmic-bytes rate."""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist

ap = argparse.ArgumentParser()
ap.add_argument("--scheme", default="thc")
ap.add_argument("--d", type=int, default=350_000_000)
ap.add_argument("--n", type=int, default=1)
ap.add_argument("--q", type=int, default=4)
ap.add_argument("--b", type=int, default=8)
ap.add_argument("--rank", type=int, default=4)
ap.add_argument("--block", type=int, default=1024)
ap.add_argument("--segs", default="1000000")
ap.add_argument("--steps", type=int, default=10)
a = ap.parse_args()
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
import paper_2407_01378_b200 as gcb
from paper_2407_01378_b200.distributed import DistributedGradientPipeline


def make():
    if a.scheme == "thc":
        return DistributedGradientPipeline(gcb.RotatedQuantConfig(a.q, a.b, a.block), a.n, a.d, gcb.SeedSpec(2024),
                                           validate=False)
    if a.scheme == "psgd":
        return DistributedGradientPipeline(gcb.PowerSgdConfig(a.rank), a.n, a.d, gcb.SeedSpec(2024), validate=False)
    if a.scheme == "fp16":
        return DistributedGradientPipeline(gcb.DenseConfig(16), a.n, a.d, gcb.SeedSpec(2024), validate=False)
    if a.scheme == "psgd_gpt2":
        from paper_2407_01378_b200.multitensor import TensorListPipeline, gpt2_medium_sizes
        return TensorListPipeline(gcb.PowerSgdConfig(a.rank), a.n, gpt2_medium_sizes(), gcb.SeedSpec(2024),
                                  validate=False, compute_nmse=False)
    if a.scheme == "psgd_gpt2_dist":
        from paper_2407_01378_b200.distributed import DistributedTensorListPipeline
        from paper_2407_01378_b200.multitensor import gpt2_medium_sizes
        return DistributedTensorListPipeline(gcb.PowerSgdConfig(a.rank), a.n, gpt2_medium_sizes(), gcb.SeedSpec(2024),
                                             validate=False)
    raise SystemExit(a.scheme)


if a.scheme.startswith("psgd_gpt2"):
    from paper_2407_01378_b200.multitensor import gpt2_medium_sizes
    a.d = sum(gpt2_medium_sizes())
g = [torch.randn(a.n, a.d, device="cuda") for _ in range(2)]
for seg in [int(x) for x in a.segs.split(",")]:
    os.environ["GC_THC_RANK_SEG_TILES"] = str(seg)
    pipe = make()
    for r in range(3):
        pipe.run_round(g[r % 2], r)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    t_host = time.perf_counter()
    for r in range(a.steps):
        pipe.run_round(g[r % 2], 3 + r)
    host_ms = (time.perf_counter() - t_host) * 1e3 / a.steps   # host time to issue a round (no final sync)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / a.steps
    if a.scheme == "thc":
        w = 0.5 if a.b <= 4 else 1
        alg = (12 * a.n + 4 + w * (a.n + 1)) * a.d
    elif a.scheme.startswith("psgd"):
        alg = (12 * a.n + 4) * a.d
    else:
        alg = (4 * a.n + 4) * a.d
    print(json.dumps({"scheme": a.scheme, "d": a.d, "n": a.n, "q": a.q, "b": a.b, "seg_tiles": seg,
                      "ms": round(ms, 4), "gelem_s": round(a.d / ms / 1e6, 2), "alg_GBps": round(alg / ms / 1e6, 1),
                      "hbm_frac": round(alg / ms / 1e6 / 6548.5, 4), "host_issue_ms": round(host_ms, 4)}), flush=True)
    del pipe
dist.destroy_process_group()
