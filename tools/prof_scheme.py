"""Short run of one scheme for ncu: python tools/prof_scheme.py <topk|topkc|psgd|psgd_gpt2m|dense16> [d] [n] [rounds]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2407_01378_b200 as gcb
name = sys.argv[1]
d = int(sys.argv[2]) if len(sys.argv) > 2 else 27_500_000
n = int(sys.argv[3]) if len(sys.argv) > 3 else 8
rounds = int(sys.argv[4]) if len(sys.argv) > 4 else 1
cfg = {"topk": lambda: gcb.TopKConfig(d // 100), "topkc": lambda: gcb.ChunkedTopKConfig(64, max(1, d // 6400)),
       "psgd": lambda: gcb.PowerSgdConfig(4), "dense16": lambda: gcb.DenseConfig(16),
       "psgd_gpt2m": lambda: None}[name]()
if name == "psgd_gpt2m":   # chunked PowerSGD over GPT-2-medium's 292 tensors
    from paper_2407_01378_b200.multitensor import TensorListPipeline, gpt2_medium_sizes
    sizes = gpt2_medium_sizes()
    d = sum(sizes)
    g = torch.randn(n, d, device="cuda")
    pipe = TensorListPipeline(gcb.PowerSgdConfig(4), n, sizes, gcb.SeedSpec(2024), validate=False, compute_nmse=False)
else:
    g = torch.randn(n, d, device="cuda")
    pipe = gcb.make_pipeline(cfg, n, d, gcb.SeedSpec(2024), validate=False, compute_nmse=False)
for r in range(rounds):
    pipe.run_round(g, r)
torch.cuda.synchronize()
print("done")
