"""Quick timing probe of the THC paths at config 2 (d=25,557,032, n=8 simulated workers)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2407_01378_b200 as gcb

d = int(sys.argv[1]) if len(sys.argv) > 1 else 25_557_032
n = int(sys.argv[2]) if len(sys.argv) > 2 else 8
for fused in ((True,) if os.environ.get("FUSED_ONLY") else (True, False)):
    for q, b in ((4, 8), (4, 4)):
        g = torch.randn(n, d, device="cuda")
        pipe = gcb.make_pipeline(gcb.RotatedQuantConfig(q, b), n, d, gcb.SeedSpec(2024), fused=fused, validate=False,
                                 compute_nmse=False)
        for r in range(3):
            pipe.run_round(g, r)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        K = 10
        s.record()
        for r in range(3, 3 + K):
            pipe.run_round(g, r)
        e.record(); torch.cuda.synchronize()
        ms = s.elapsed_time(e) / K
        bytes_ = (12 * n + 4) * d
        print(f"fused={fused} q={q} b={b}: {ms:.3f} ms/round  {d/ms/1e6:.2f} Gelem/s(d)  {n*d/ms/1e6:.1f} Gworker-elem/s  "
              f"{bytes_/ms/1e6:.0f} GB/s algorithmic")
