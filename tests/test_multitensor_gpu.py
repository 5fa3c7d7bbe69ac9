"""Chunked (per-tensor) pipelines over a flat gradient: every tensor must
match an independent reference pipeline run on its slice."""
import numpy as np
import pytest

from tests.gpu_util import needs_gpu, oracle_rounds

pytestmark = [pytest.mark.gpu, needs_gpu]

# a miniature transformer: embedding, biases / norms (bypass), square and non-square matrices,
# repeated shapes (batched groups), a 4096-element tensor (64 x 64, not bypassed)
SIZES = [6000, 64, 64, 3 * 4096, 192, 4096, 64, 64, 64, 3 * 4096, 192, 4096, 4096, 64, 10_000]


def _grads(n, D, rounds, seed):
    rng = np.random.default_rng(seed)
    return [[rng.standard_normal(D).astype(np.float32) for _ in range(n)] for _ in range(rounds)]


@pytest.mark.parametrize("nmse,mtp_ef", [(True, False), (False, False), (False, True)])
@pytest.mark.parametrize("rank,warm", [(4, True), (2, False), (1, True), (12, True)])
def test_powersgd_per_tensor_matches_reference(rank, warm, nmse, mtp_ef):
    """nmse False: ef_apply fused into the first pass of each tensor; mtp_ef: Q_w and the EF update
    in one pass (gc_psgd_mtp_ef, opt-in) for the batched groups whose shapes allow it."""
    import paper_2407_01378_b200 as gcb
    from paper_2407_01378_b200.multitensor import TensorListPipeline
    from paper_2407_01378_b200.schemes import PowerSgdGroup
    n, seed = 3, 51
    D = sum(SIZES)
    offs = np.concatenate([[0], np.cumsum(SIZES)[:-1]])
    grads = _grads(n, D, 3, seed)
    pipe = TensorListPipeline(gcb.PowerSgdConfig(rank, warm), n, SIZES, gcb.SeedSpec(seed), compute_nmse=nmse)
    if mtp_ef:
        for grp in pipe.groups:
            grp._mtp_ef_cache = True
    results = [pipe.run_round(grads[r], r) for r in range(3)]
    for t, (off, s) in enumerate(zip(offs, SIZES)):
        outs = oracle_rounds("powersgd", dict(rank=rank, warm_start=warm),
                             [[g[off:off + s] for g in grads[r]] for r in range(3)], seed)
        for r in range(3):
            ref = outs[r]["estimate"].astype(np.float64)
            got = results[r].estimate.logical[off:off + s].astype(np.float64)
            scale = max(np.max(np.abs(ref)), 1e-30)
            assert np.max(np.abs(got - ref)) <= 1e-5 * scale, (t, r)
        res_ref = np.stack(outs[2]["residuals"])
        res_got = np.stack(pipe.residuals)[:, off:off + s]
        assert np.max(np.abs(res_got - res_ref)) <= 1e-5 * max(np.max(np.abs(res_ref)), 1e-30), t
        if s >= 4096 and warm:
            assert np.max(np.abs(pipe.warm_q(t) - outs[2]["warm_q"])) <= 1e-5 * np.max(np.abs(outs[2]["warm_q"]))
    if mtp_ef and rank in PowerSgdGroup.RANKS:   # the fused pass ran for the aligned groups (64 x 64 batch of three, 100 x 100)
        assert sum(bool(grp._mtp_ef_ok()) for grp in pipe.groups) >= 2


def test_topk_per_tensor_bit_exact():
    import paper_2407_01378_b200 as gcb
    from paper_2407_01378_b200.multitensor import TensorListPipeline
    n, seed = 2, 61
    sizes = [5000, 100, 777]
    D = sum(sizes)
    offs = np.concatenate([[0], np.cumsum(sizes)[:-1]])
    grads = _grads(n, D, 2, seed)
    pipe = TensorListPipeline(gcb.TopKConfig(50), n, sizes, gcb.SeedSpec(seed))
    results = [pipe.run_round(grads[r], r) for r in range(2)]
    for off, s in zip(offs, sizes):
        outs = oracle_rounds("topk", dict(k=50), [[g[off:off + s] for g in grads[r]] for r in range(2)], seed)
        for r in range(2):
            assert np.array_equal(results[r].estimate.logical[off:off + s], outs[r]["estimate"])
        assert np.array_equal(np.stack(pipe.residuals)[:, off:off + s], np.stack(outs[1]["residuals"]))
    # nmse of the flat vector against the fp64 mean of the corrected gradients (pipelines.py:176-181)
    res0 = np.zeros((n, D), np.float32)
    for r in range(2):
        corrected = np.stack(grads[r]) + res0
        ref = corrected.astype(np.float64).mean(axis=0)
        est = results[r].estimate.logical.astype(np.float64)
        want = np.sum((est - ref) ** 2) / np.sum(ref ** 2)
        assert abs(results[r].nmse - want) <= 1e-9 * want, (r, results[r].nmse, want)
        if r == 0:
            res0 = np.stack([np.concatenate([oracle_rounds("topk", dict(k=50), [[g[o:o + s] for g in grads[0]]],
                                                           seed)[0]["residuals"][w] for o, s in zip(offs, sizes)])
                             for w in range(n)])


def test_gpt2_medium_layout():
    from paper_2407_01378_b200.multitensor import gpt2_medium_sizes
    import paper_2407_01378_b200 as gcb
    sizes = gpt2_medium_sizes()
    assert len(sizes) == 292 and sum(sizes) == 354_823_168
    comp = [s for s in sizes if s >= 4096]
    assert len(comp) == 122 and sum(s for s in sizes if s < 4096) == 223_232
    shapes = sorted({gcb.matrix_shape_for(s) for s in comp})
    assert shapes == [(64, 64), (1024, 1024), (1774, 1774), (2048, 2048), (7174, 7174)]
