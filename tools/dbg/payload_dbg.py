import sys, os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2407_01378_b200 as gcb
from paper_2407_01378_b200 import payloads as pl
n, d, k = 4, 300_000, 3_000
seeds = gcb.SeedSpec(12)
grads = [seeds.rng("grad-worker", 0, w).standard_normal(d).astype(np.float32) * 1e3 for w in range(n)]
pipe = gcb.make_pipeline(gcb.TopKConfig(k), n, d, seeds)
pipe._engine.capture = True
pipe.run_round(grads, 0)
idx, val = pipe._engine.last["idx"], pipe._engine.last["val"]
torch.cuda.synchronize()
dev = pl.encode_sparse_payloads_device(idx, val).cpu().numpy()
for w in range(n):
    host = np.frombuffer(pl.encode_payload(pl.SparsePayload(idx[w].cpu().numpy(), val[w].cpu().numpy())), np.uint8)
    bad = np.nonzero(dev[w] != host)[0]
    print(w, len(bad), bad[:10], dev[w][bad[:6]], host[bad[:6]])
    v = val[w].cpu().numpy()
    print(' vals', v[:4], v[-4:], v.dtype, np.abs(v).max(), (v.astype(np.float16).astype(np.float32) != v).sum())
