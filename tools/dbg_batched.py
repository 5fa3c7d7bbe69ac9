"""Debug: batched TMA P = M Q against the register-fed kernel for a shape group."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2407_01378_b200 as gcb
from paper_2407_01378_b200 import _native
from paper_2407_01378_b200.configs import matrix_shape_for
torch.cuda.set_device(0)
sizes = [64 * 64, 4096, 128 * 128, 64 * 64, 100, 200 * 200, 128 * 128]
n, D = 2, sum(sizes)
offs = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int64)
ts = [0, 1, 3]
d = 4096
rows, cols = matrix_shape_for(d)
r = 4
ro = torch.tensor([w * D + int(offs[t]) for t in ts for w in range(n)], dtype=torch.int64, device="cuda")
batch = _native.PsgdBatch(len(ts), n, ro.data_ptr(), D, None, 1, 0)
hoffs = (ctypes.c_int64 * len(ts))(*[int(offs[t]) for t in ts])
g = torch.randn(n, D, device="cuda")
res = torch.randn(n, D, device="cuda")
q = torch.randn(len(ts), cols, r, device="cuda")
ws = torch.empty(int(_native.lib().gc_psgd_workspace_bytes(len(ts) * n, rows, cols, r)), dtype=torch.uint8, device="cuda")
p1 = torch.empty(len(ts) * n, rows, r, device="cuda")
p2 = torch.empty(len(ts) * n, rows, r, device="cuda")
r1, r2 = res.clone(), res.clone()
sp = torch.cuda.current_stream().cuda_stream
print("supported", _native.lib().gc_psgd_mq_tma_supported_batched(ctypes.byref(batch), hoffs, d, rows, cols, r, g.data_ptr(), r1.data_ptr()))
_native.call("gc_psgd_mq_deferred_batched", ctypes.byref(batch), hoffs, d, rows, cols, r, g.data_ptr(), r1.data_ptr(),
             q.data_ptr(), None, None, p1.data_ptr(), ws.data_ptr(), sp)
_native.call("gc_psgd_mq_fused", ctypes.byref(batch), d, rows, cols, r, g.data_ptr(), r2.data_ptr(), q.data_ptr(),
             p2.data_ptr(), ws.data_ptr(), sp)
torch.cuda.synchronize()
print("resid equal", torch.equal(r1, r2), (r1 - r2).abs().max().item())
diff = (r1 != r2).nonzero()
print("first diffs", diff[:10].tolist(), "count", diff.shape[0])
for k, t in enumerate(ts):
    for w in range(n):
        v = k * n + w
        print(k, t, w, "P max diff", (p1[v] - p2[v]).abs().max().item(), "scale", p2[v].abs().max().item())
