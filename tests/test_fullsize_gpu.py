"""Parity at BASELINE.json's full sizes, where the NumPy oracle is too slow to run: size-independent
properties checked exactly (or to the floating-point contract) on the device.

* THC cfg2 (d = 25,557,032, n = 8, q = 4, b = 8 and q = b = 4): the fused single-kernel round
  and the independent multi-kernel path (rotate / quantize / saturating fold / decode kernels,
  each pinned to the oracle at small sizes) agree bit for bit on estimates, residuals and
  overflow counters over several EF rounds.
* TopK cfg3 (d = 110,000,000, k = 1 %, n = 8): per worker the k indices are strictly ascending,
  carry the largest magnitudes with the lower index winning ties, the values are the fp16 round
  trip of the corrected vector, the residual is corrected minus the payload, and the estimate is
  the worker-order f32 scatter sum / n -- all exact, over rounds that exercise the threshold hint.
* PowerSGD cfg4 (d = 350,000,000 as one 18,709 x 18,708 matrix, r = 4, n = 8): P_hat equals the
  reference orthonormalisation of the fp64 product sum_w M_w Q, and the estimate / residuals equal
  the fp64 factor products, within the 1e-5 relative contract.
"""
import numpy as np
import pytest
import torch

from oracle import gradcomp_oracle as orc
from tests.gpu_util import needs_gpu

pytestmark = [pytest.mark.gpu, needs_gpu]


def _randn(n, d, seed, scale=1.0):
    gen = torch.Generator(device="cuda").manual_seed(seed)
    return torch.randn(n, d, device="cuda", generator=gen) * scale


@pytest.mark.parametrize("q,b", [(4, 8), (4, 4)])
def test_thc_cfg2_fused_equals_multikernel(q, b):
    import paper_2407_01378_b200 as gcb
    n, d = 8, 25_557_032
    cfg = gcb.RotatedQuantConfig(q, b, 1024)
    fused = gcb.make_pipeline(cfg, n, d, gcb.SeedSpec(2024), fused=True, validate=False)
    multi = gcb.make_pipeline(cfg, n, d, gcb.SeedSpec(2024), fused=False, validate=False)
    assert fused._engine.fused and not multi._engine.fused
    for r in range(3):
        g = _randn(n, d, 100 + r)
        a, m = fused.run_round(g, r), multi.run_round(g, r)
        assert torch.equal(a.estimate_tensor, m.estimate_tensor), r
        assert torch.equal(fused.residuals_tensor, multi.residuals_tensor), r
        oa, om = a.overflow, m.overflow
        assert (oa.clip_events, oa.total_adds) == (om.clip_events, om.total_adds)
        assert oa.code_sigma == pytest.approx(om.code_sigma, rel=1e-12)
        assert a.nmse == pytest.approx(m.nmse, rel=1e-9)


def _fp16_round_trip(x: torch.Tensor) -> torch.Tensor:
    y = x.to(torch.float16).to(torch.float32)
    return torch.where(torch.isinf(y), torch.copysign(torch.full_like(y, 65504.0), x), y)


def test_topk_cfg3_selection_invariants():
    import paper_2407_01378_b200 as gcb
    n, d = 8, 110_000_000
    k = d // 100
    pipe = gcb.make_pipeline(gcb.TopKConfig(k), n, d, gcb.SeedSpec(2024), validate=False, compute_nmse=False)
    pipe._engine.capture = True
    idx_all = torch.arange(d, device="cuda")
    for r in range(4):
        # fresh Gaussian gradients each round; round 2's cancel the carried residual, so the
        # corrected vectors shrink ~100x, the boundary bin falls below the threshold hint and the
        # collect pass has to run again
        g = _randn(n, d, 200 + r, 0.01 if r == 2 else 1.0)
        if r == 2:
            g -= pipe.residuals_tensor
        corrected = g + pipe.residuals_tensor   # f32(g + r) exactly as ef_apply
        res = pipe.run_round(g, r)
        idx, val = pipe._engine.last["idx"].long(), pipe._engine.last["val"]
        est = torch.zeros(d, dtype=torch.float32, device="cuda")
        for w in range(n):
            c, iw, vw = corrected[w], idx[w], val[w]
            assert iw.numel() == k
            assert bool((iw[1:] > iw[:-1]).all()), (r, w)            # strictly ascending
            mag = c.abs()
            sel = torch.zeros(d, dtype=torch.bool, device="cuda")
            sel[iw] = True
            t = mag[iw].min()
            assert float(mag[~sel].max()) <= float(t), (r, w)        # the k largest magnitudes
            ties_out = idx_all[(~sel) & (mag == t)]
            if ties_out.numel():                                      # lower index wins ties
                assert int(iw[mag[iw] == t].max()) < int(ties_out.min()), (r, w)
            assert torch.equal(vw, _fp16_round_trip(c[iw])), (r, w)   # fp16 payload values
            exp_res = c.clone()
            exp_res[iw] = c[iw] - vw                                  # ef_update
            assert torch.equal(pipe.residuals_tensor[w], exp_res), (r, w)
            est[iw] += vw                                             # worker-order f32 scatter sum
        assert torch.equal(res.estimate_tensor, est / n), r
        del corrected


def test_powersgd_cfg4_factors_within_tolerance():
    import paper_2407_01378_b200 as gcb
    n, d, rank = 8, 350_000_000, 4
    pipe = gcb.make_pipeline(gcb.PowerSgdConfig(rank), n, d, gcb.SeedSpec(2024), validate=False,
                             compute_nmse=False)
    pipe._engine.capture = True
    g = _randn(n, d, 300)
    res = pipe.run_round(g, 0)
    grp = pipe._engine.group
    rows, cols = grp.rows, grp.cols
    last = pipe._engine.last
    q = last["seed_q"].double()                                     # [cols, r]
    # fp64 reference of P = sum_w M_w Q (residuals start at zero: M_w = g_w zero-padded)
    p64 = torch.zeros(rows, rank, dtype=torch.float64, device="cuda")
    m = torch.zeros(rows * cols, dtype=torch.float64, device="cuda")
    for w in range(n):
        m[:d] = g[w].double()
        p64 += m.view(rows, cols) @ q
    p_hat_ref = torch.from_numpy(orc.orthonormalize(p64.cpu().numpy())).cuda().double()
    p_hat = last["p_hat"].double()
    assert float((p_hat - p_hat_ref).abs().max()) <= 1e-5 * float(p_hat_ref.abs().max())
    eye = p_hat.T @ p_hat
    assert float((eye - torch.eye(rank, dtype=torch.float64, device="cuda")).abs().max()) <= 1e-5
    # Q_w = M_w^T P_hat; estimate = P_hat (sum_w Q_w)^T / n; residual_w = M_w - P_hat Q_w^T
    q_sum = torch.zeros(cols, rank, dtype=torch.float64, device="cuda")
    for w in range(n):
        m[:d] = g[w].double()
        q_w = m.view(rows, cols).T @ p_hat
        q_sum += q_w
        if w in (0, n - 1):
            own = (p_hat @ q_w.T).reshape(-1)[:d]
            ref_res = g[w].double() - own
            err = (pipe.residuals_tensor[w].double() - ref_res).abs().max()
            assert float(err) <= 1e-5 * float(g[w].abs().max()), w
    est_ref = ((p_hat @ q_sum.T) / n).reshape(-1)[:d]
    err = (res.estimate_tensor.double() - est_ref).abs().max()
    assert float(err) <= 1e-5 * float(est_ref.abs().max())
