"""Short run of one scheme for ncu: python tools/prof_scheme.py <topk|topkc|psgd|dense16> [d] [n] [rounds]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2407_01378_b200 as gcb
name = sys.argv[1]
d = int(sys.argv[2]) if len(sys.argv) > 2 else 27_500_000
n = int(sys.argv[3]) if len(sys.argv) > 3 else 8
rounds = int(sys.argv[4]) if len(sys.argv) > 4 else 1
cfg = {"topk": gcb.TopKConfig(d // 100), "topkc": gcb.ChunkedTopKConfig(64, max(1, d // 6400)),
       "psgd": gcb.PowerSgdConfig(4), "dense16": gcb.DenseConfig(16)}[name]
g = torch.randn(n, d, device="cuda")
pipe = gcb.make_pipeline(cfg, n, d, gcb.SeedSpec(2024), validate=False, compute_nmse=False)
for r in range(rounds):
    pipe.run_round(g, r)
torch.cuda.synchronize()
print("done")
