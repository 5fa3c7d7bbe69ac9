"""TopK-Chunked (bit-exact) and PowerSGD (fp32 tolerance) on the GPU vs golden vectors / oracle."""
import numpy as np
import pytest

from tests.gpu_util import needs_gpu, oracle_rounds, run_golden_case

pytestmark = [pytest.mark.gpu, needs_gpu]

# north star: PowerSGD floats within 1e-5 relative (fp32).  Relative to the vector's scale:
# normwise ||ours - ref|| <= 1e-5 ||ref|| and elementwise |ours - ref| <= 1e-5 max|ref|.
PSGD_TOL = 1e-5


def assert_close_fp32(ours, ref, what=""):
    ours, ref = np.asarray(ours, np.float64), np.asarray(ref, np.float64)
    scale = float(np.max(np.abs(ref))) if ref.size else 0.0
    assert np.linalg.norm(ours - ref) <= PSGD_TOL * max(np.linalg.norm(ref), 1e-30), what
    assert np.max(np.abs(ours - ref), initial=0.0) <= PSGD_TOL * max(scale, 1e-30), what


def _ledger(res, n):
    return {ph: [[res.ledger.bits_sent(worker=w, phase=ph), res.ledger.bits_received(worker=w, phase=ph)]
                 for w in range(n)] for ph in res.ledger.phases()}


@pytest.mark.parametrize("name", ["chunked_a", "chunked_b", "chunked_c"])
def test_chunked_golden_bit_exact(name):
    for st, res, pipe, a in run_golden_case(name):
        r = st["round"]
        assert np.array_equal(res.estimate.logical, a[f"estimate_{r}"]), f"round {r} estimate"
        assert np.array_equal(np.stack(pipe.residuals), a[f"residuals_{r}"]), f"round {r} residuals"
        assert res.nmse == pytest.approx(st["nmse"], rel=1e-9, abs=1e-15)
        assert res.input_bits_per_coord == pytest.approx(st["input_bits_per_coord"], rel=1e-15)
        assert _ledger(res, pipe.group.size) == st["ledger"]


@pytest.mark.parametrize("n,d,C,J", [(8, 1_000_000, 64, 156), (3, 100_003, 100, 17), (4, 70_000, 7, 1000),
                                     (2, 65_536, 1024, 8), (5, 4096, 64, 64)])
def test_chunked_vs_oracle(n, d, C, J):
    import paper_2407_01378_b200 as gcb
    seeds = gcb.SeedSpec(21)
    rng = np.random.default_rng(21)
    grads = [[(rng.standard_normal(d) * rng.uniform(0.1, 3)).astype(np.float32) for _ in range(n)]
             for _ in range(2)]
    outs = oracle_rounds("chunked_topk", dict(chunk_size=C, chunks_selected=J), grads, 21)
    pipe = gcb.make_pipeline(gcb.ChunkedTopKConfig(C, J), n, d, seeds)
    pipe._engine.capture = True
    for r in range(2):
        res = pipe.run_round(grads[r], r)
        assert np.array_equal(pipe._engine.last["selected"].cpu().numpy(), outs[r]["selected"])
        assert np.array_equal(pipe._engine.last["norms"].cpu().numpy(), np.stack(outs[r]["norms"]))
        assert np.array_equal(res.estimate.logical, outs[r]["estimate"])
        assert np.array_equal(np.stack(pipe.residuals), np.stack(outs[r]["residuals"]))


@pytest.mark.parametrize("name", ["psgd_a", "psgd_b", "psgd_c"])
def test_psgd_golden_within_tolerance(name):
    for st, res, pipe, a in run_golden_case(name):
        r = st["round"]
        assert_close_fp32(res.estimate.logical, a[f"estimate_{r}"], f"round {r} estimate")
        assert_close_fp32(np.stack(pipe.residuals), a[f"residuals_{r}"], f"round {r} residuals")
        if f"warm_q_{r}" in a:
            assert_close_fp32(pipe._warm_q, a[f"warm_q_{r}"], f"round {r} warm q")
        assert res.nmse == pytest.approx(st["nmse"], rel=1e-5)
        assert res.input_bits_per_coord == pytest.approx(st["input_bits_per_coord"], rel=1e-15)
        assert _ledger(res, pipe.group.size) == st["ledger"]


@pytest.mark.parametrize("nmse", [True, False])
@pytest.mark.parametrize("n,d,rank", [(4, 1_000_000, 4), (2, 350_001, 1), (3, 100_000, 8), (8, 4096, 2),
                                      (2, 50_000, 16), (2, 60_001, 9), (3, 100_000, 20), (2, 100_003, 32),
                                      (2, 200_000, 64), (2, 200_000, 100), (2, 300_000, 256)])
def test_psgd_vs_oracle_multi_round(n, d, rank, nmse):
    """Every rank the reference accepts (compressors.py:100-112): ranks outside the compiled set run
    their factor passes in rank chunks (16s, 8, rest); nmse=True decodes estimate and EF update
    separately, nmse=False in one pass."""
    import paper_2407_01378_b200 as gcb
    seeds = gcb.SeedSpec(31)
    grads = [[seeds.rng("grad-worker", r, w).standard_normal(d).astype(np.float32) for w in range(n)]
             for r in range(3)]
    outs = oracle_rounds("powersgd", dict(rank=rank), grads, 31)
    pipe = gcb.make_pipeline(gcb.PowerSgdConfig(rank), n, d, seeds, compute_nmse=nmse)
    if rank in (20, 64, 100):
        assert pipe._engine.group.chunks == {20: [16, 4], 64: [16] * 4, 100: [16] * 6 + [4]}[rank]
    for r in range(3):
        res = pipe.run_round(grads[r], r)
        assert_close_fp32(res.estimate.logical, outs[r]["estimate"], f"round {r}")
        assert_close_fp32(np.stack(pipe.residuals), np.stack(outs[r]["residuals"]), f"round {r} residuals")


@pytest.mark.parametrize("n,d,rank", [(4, 1_000_000, 4), (3, 999_997, 8), (2, 350_001, 1), (8, 4096, 2),
                                      (2, 50_000, 16), (3, 100_003, 3)])
def test_psgd_mtp_ef_vs_oracle(n, d, rank):
    """Without the nmse hook Q_w and the EF update run fused (gc_psgd_mtp_ef) where the shape allows:
    estimate, residuals and warm Q against the oracle over rounds, and against the unfused kernels."""
    import paper_2407_01378_b200 as gcb
    seeds = gcb.SeedSpec(37)
    grads = [[seeds.rng("grad-worker", r, w).standard_normal(d).astype(np.float32) for w in range(n)]
             for r in range(3)]
    outs = oracle_rounds("powersgd", dict(rank=rank), grads, 37)
    pipe = gcb.make_pipeline(gcb.PowerSgdConfig(rank), n, d, seeds, compute_nmse=False)
    ref = gcb.make_pipeline(gcb.PowerSgdConfig(rank), n, d, seeds, compute_nmse=False)
    for r in range(3):
        if r == 0:
            pipe._engine.group._mtp_ef_cache = True    # opt-in path under test
            ref._engine.group._mtp_ef_cache = False
        res = pipe.run_round(grads[r], r)
        alt = ref.run_round(grads[r], r)
        assert_close_fp32(res.estimate.logical, outs[r]["estimate"], f"round {r}")
        assert_close_fp32(np.stack(pipe.residuals), np.stack(outs[r]["residuals"]), f"round {r} residuals")
        assert_close_fp32(res.estimate.logical, alt.estimate.logical, f"round {r} vs unfused")
        assert_close_fp32(np.stack(pipe.residuals), np.stack(ref.residuals), f"round {r} residuals vs unfused")
    grp = pipe._engine.group
    if grp.rank <= 8 and grp.rows >= 16 and grp.cols % 4 == 0 and grp.batch.rows_aligned:
        assert grp._mtp_ef_ok()


@pytest.mark.parametrize("rank", [4, 20])
def test_psgd_zero_gradients_complete_basis_and_redraw(rank):
    """All-zero gradients: MGS completes with canonical vectors; round 1's warm Q is zero and is redrawn."""
    import paper_2407_01378_b200 as gcb
    n, d = 2, 10_000
    grads = [[np.zeros(d, np.float32) for _ in range(n)] for _ in range(2)]
    outs = oracle_rounds("powersgd", dict(rank=rank), grads, 41)
    pipe = gcb.make_pipeline(gcb.PowerSgdConfig(rank), n, d, gcb.SeedSpec(41))
    pipe._engine.capture = True
    for r in range(2):
        res = pipe.run_round(grads[r], r)
        assert not np.any(res.estimate.logical)
        ph = pipe._engine.last["p_hat"].cpu().numpy()
        assert np.array_equal(ph, outs[r]["p_hat"])
        assert_close_fp32(pipe._engine.last["seed_q"].cpu().numpy(), outs[r]["seed_q"])
