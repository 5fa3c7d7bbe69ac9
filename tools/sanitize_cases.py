"""Small rounds of the kernels with mbarrier / TMEM / DSMEM / cluster / shared-memory protocols,
for compute-sanitizer (memcheck, racecheck, synccheck):

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py [case ...]

cases: thc_fused (n = 8, B = 1024, 2 rounds), thc_rank (per-rank K1/K2/K3 on a one-rank gloo
group), psgd_umma (register-fed tcgen05 P = M Q), psgd_tma (TMA-fed tcgen05 P = M Q with the
deferred EF update, TMA Q = M^T P_hat, Cholesky orthonormalization; 3 rounds), psgd_batched (one
tensor map per tensor of a shape group), psgd_mtp_ef (cluster / DSMEM Q + EF pass), psgd_mtp_umma
(tcgen05 Q = M^T P_hat at ranks 4 / 8 / 16: several TMEM fold groups, a partial chunk and row),
psgd_async (cp.async-fed deferred P = M Q: unaligned batched groups over 3 rounds), psgd_pair
(row-pair tensor maps for cols = 2 mod 4: GPT-2-like shapes, deferred EF, 3 rounds), topk, topkc."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2407_01378_b200 as gcb

cases = sys.argv[1:] or ["thc_fused", "thc_rank", "psgd_umma", "psgd_tma", "psgd_batched", "psgd_mtp_ef",
                         "psgd_mtp_umma", "psgd_async", "psgd_pair",
                         "topk", "topkc"]
torch.cuda.set_device(0)
S = gcb.SeedSpec(7)


def rounds(pipe, g, k=2):
    for r in range(k):
        pipe.run_round(g, r)
    torch.cuda.synchronize()


for c in cases:
    if c == "thc_fused":
        n, d = 8, (1 << 15) + 77
        rounds(gcb.make_pipeline(gcb.RotatedQuantConfig(4, 8), n, d, S, fused=True), torch.randn(n, d, device="cuda"))
    elif c == "thc_rank":
        import torch.distributed as dist
        from paper_2407_01378_b200.distributed import DistributedGradientPipeline
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29561")
        if not dist.is_initialized():
            dist.init_process_group("gloo", rank=0, world_size=1)
        d = (1 << 15) + 77
        rounds(DistributedGradientPipeline(gcb.RotatedQuantConfig(4, 8), 1, d, S), torch.randn(1, d, device="cuda"))
    elif c == "psgd_umma":
        n, d = 2, 300 * 257
        rounds(gcb.make_pipeline(gcb.PowerSgdConfig(4), n, d, S), torch.randn(n, d, device="cuda"))
    elif c == "psgd_tma":
        n, d = 2, 40004   # 201 x 200: TMA boxes, a partly filled last row (tail kernel), deferred EF
        pipe = gcb.make_pipeline(gcb.PowerSgdConfig(4), n, d, S, compute_nmse=False)
        rounds(pipe, torch.randn(n, d, device="cuda"), 3)
        pipe.residuals
    elif c == "psgd_batched":
        from paper_2407_01378_b200.multitensor import TensorListPipeline
        sizes = [64 * 64, 4096, 128 * 128, 100, 200 * 200]
        pipe = TensorListPipeline(gcb.PowerSgdConfig(4), 2, sizes, S, compute_nmse=False)
        rounds(pipe, torch.randn(2, sum(sizes), device="cuda"), 3)
        pipe.residuals
    elif c == "psgd_mtp_ef":
        os.environ["GC_PSGD_MTP_EF"] = "1"
        n, d = 2, 256 * 256
        pipe = gcb.make_pipeline(gcb.PowerSgdConfig(4), n, d, S, compute_nmse=False)
        rounds(pipe, torch.randn(n, d, device="cuda"))
        os.environ["GC_PSGD_MTP_EF"] = "0"
    elif c == "psgd_mtp_umma":
        import ctypes
        from paper_2407_01378_b200 import _native
        os.environ["GC_PSGD_MTP"] = "umma"
        rows, cols = 1100, 260          # 35 chunks of 32 rows: three fold groups, a partial chunk
        d = rows * cols - 40            # and a partly filled last row (d % 4 == 0: aligned worker rows)
        for r in (4, 8, 16):
            c = torch.randn(2, d, device="cuda")
            ph = torch.randn(rows, r, device="cuda")
            batch = _native.PsgdBatch(1, 2, None, d, None, 1, 0)
            ws = torch.empty(int(_native.lib().gc_psgd_workspace_bytes(2, rows, cols, r)), dtype=torch.uint8,
                             device="cuda")
            q = torch.empty(2, cols, r, device="cuda")
            _native.call("gc_psgd_mtp", ctypes.byref(batch), d, rows, cols, r, c.data_ptr(), ph.data_ptr(),
                         q.data_ptr(), ws.data_ptr(), torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        del os.environ["GC_PSGD_MTP"]
    elif c == "psgd_async":
        from paper_2407_01378_b200.multitensor import TensorListPipeline
        sizes = [150 * 150, 77 * 77, 150 * 150 - 7, 600 * 602 + 3]   # > 16 chunks: TMEM fold groups
        pipe = TensorListPipeline(gcb.PowerSgdConfig(4), 2, sizes, S, compute_nmse=False)
        rounds(pipe, torch.randn(2, sum(sizes), device="cuda"), 3)
        pipe.residuals
    elif c == "psgd_pair":
        from paper_2407_01378_b200.multitensor import TensorListPipeline
        sizes = [150 * 150, 150 * 150 - 8, 4, 602 * 602 - 10]   # cols 150 / 602: = 2 (mod 4), aligned starts
        pipe = TensorListPipeline(gcb.PowerSgdConfig(4), 2, sizes, S, compute_nmse=False)
        rounds(pipe, torch.randn(2, sum(sizes), device="cuda"), 3)
        pipe.residuals
    elif c == "topk":
        n, d = 2, 1 << 16
        rounds(gcb.make_pipeline(gcb.TopKConfig(d // 100), n, d, S), torch.randn(n, d, device="cuda"))
    elif c == "topkc":
        n, d = 2, 1 << 16
        rounds(gcb.make_pipeline(gcb.ChunkedTopKConfig(64, 10), n, d, S), torch.randn(n, d, device="cuda"))
    print("case ok:", c, flush=True)
