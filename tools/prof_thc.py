"""Short THC run for ncu captures: python tools/prof_thc.py [d] [n] [fused 0/1] [rounds]."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2407_01378_b200 as gcb
d = int(sys.argv[1]) if len(sys.argv) > 1 else 4_000_000
n = int(sys.argv[2]) if len(sys.argv) > 2 else 8
fused = bool(int(sys.argv[3])) if len(sys.argv) > 3 else True
rounds = int(sys.argv[4]) if len(sys.argv) > 4 else 2
g = torch.randn(n, d, device="cuda")
pipe = gcb.make_pipeline(gcb.RotatedQuantConfig(4, 8), n, d, gcb.SeedSpec(2024), fused=fused, validate=False,
                         compute_nmse=False)
for r in range(rounds):
    pipe.run_round(g, r)
torch.cuda.synchronize()
print("done")
