"""cProfile of the host side of per-rank PowerSGD rounds (GPT-2-medium tensor list): where the
Python / ctypes time goes and which calls wait on the device.
python tools/prof_host.py [psgd_gpt2 | psgd_gpt2_dist] [rounds]"""
import cProfile, os, pstats, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist

scheme = sys.argv[1] if len(sys.argv) > 1 else "psgd_gpt2"
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 10
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29537")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
import paper_2407_01378_b200 as gcb
from paper_2407_01378_b200.multitensor import TensorListPipeline, gpt2_medium_sizes
from paper_2407_01378_b200.distributed import DistributedTensorListPipeline
sizes = gpt2_medium_sizes()
D = sum(sizes)
if scheme == "psgd_gpt2":
    pipe = TensorListPipeline(gcb.PowerSgdConfig(4), 1, sizes, gcb.SeedSpec(2024), validate=False, compute_nmse=False)
else:
    pipe = DistributedTensorListPipeline(gcb.PowerSgdConfig(4), 1, sizes, gcb.SeedSpec(2024), validate=False)
g = [torch.randn(1, D, device="cuda") for _ in range(2)]
for r in range(3):
    pipe.run_round(g[r % 2], r)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for r in range(rounds):
    pipe.run_round(g[r % 2], 3 + r)
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
dist.destroy_process_group()
