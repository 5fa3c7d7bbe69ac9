"""Edge cases on the GPU vs the oracle: tiny / ragged dims, rotation blocks capped by the padded
length, full rotations (B > 4096), many workers (generic path beyond the fused kernel's 16),
all-zero and constant inputs (degenerate ranges), huge magnitudes (fp16 saturation)."""
import numpy as np
import pytest

from tests.gpu_util import needs_gpu, oracle_rounds

pytestmark = [pytest.mark.gpu, needs_gpu]


def _grads(seed, n, d, rounds, kind="gauss"):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(rounds):
        if kind == "zeros":
            out.append([np.zeros(d, np.float32) for _ in range(n)])
        elif kind == "const":
            out.append([np.full(d, 0.75, np.float32) for _ in range(n)])
        elif kind == "huge":
            out.append([(rng.standard_normal(d) * 3e4).astype(np.float32) for _ in range(n)])
        else:
            out.append([rng.standard_normal(d).astype(np.float32) for _ in range(n)])
    return out


def _check(scheme, params, cfg, n, d, grads, seed, exact=True, **kw):
    import paper_2407_01378_b200 as gcb
    outs = oracle_rounds(scheme, params, grads, seed)
    pipe = gcb.make_pipeline(cfg, n, d, gcb.SeedSpec(seed), **kw)
    for r, g in enumerate(grads):
        res = pipe.run_round(g, r)
        o = outs[r]
        if exact:
            assert np.array_equal(res.estimate.logical, o["estimate"]), (scheme, d, r)
            assert np.array_equal(np.stack(pipe.residuals), np.stack(o["residuals"])), (scheme, d, r)
        else:
            ref = o["estimate"].astype(np.float64)
            den = max(np.linalg.norm(ref), 1e-30)
            assert np.linalg.norm(res.estimate.logical - ref) <= 1e-5 * den + 1e-30
        if scheme == "rotated_quant":
            assert res.overflow.clip_events == o["clip_events"]
            assert res.overflow.total_adds == o["total_adds"]
            assert res.overflow.code_sigma == pytest.approx(o["code_sigma"], rel=1e-12, abs=1e-15)
        assert res.nmse == pytest.approx(o["nmse"], rel=1e-6, abs=1e-12) or (np.isinf(o["nmse"]) and np.isinf(res.nmse))


@pytest.mark.parametrize("d", [1, 2, 3, 5, 31, 33, 1023, 1024, 1025, 4097])
@pytest.mark.parametrize("fused", [True, False])
def test_thc_tiny_and_ragged_dims(d, fused):
    import paper_2407_01378_b200 as gcb
    _check("rotated_quant", dict(quant_bits=4, wire_bits=5, rotation_block=64), gcb.RotatedQuantConfig(4, 5, 64),
           3, d, _grads(d, 3, d, 2), 13, fused=fused)


@pytest.mark.parametrize("blk,d", [(2, 300), (1 << 13, 20_000), (1 << 16, 70_000), (1 << 20, 1 << 20)])
def test_thc_block_sizes(blk, d):
    import paper_2407_01378_b200 as gcb
    _check("rotated_quant", dict(quant_bits=3, wire_bits=4, rotation_block=blk), gcb.RotatedQuantConfig(3, 4, blk),
           4, d, _grads(blk, 4, d, 2), 17)


@pytest.mark.parametrize("n", [1, 2, 5, 16, 17, 24])
def test_thc_worker_counts(n):
    import paper_2407_01378_b200 as gcb
    d = 50_001
    _check("rotated_quant", dict(quant_bits=4, wire_bits=8), gcb.RotatedQuantConfig(4, 8), n, d,
           _grads(n, n, d, 2), 19)


@pytest.mark.parametrize("kind", ["zeros", "const", "huge"])
@pytest.mark.parametrize("scheme", ["rotated_quant", "topk", "chunked_topk", "dense16"])
def test_degenerate_inputs(kind, scheme):
    import paper_2407_01378_b200 as gcb
    n, d = 3, 10_000
    grads = _grads(7, n, d, 2, kind)
    if scheme == "rotated_quant":
        _check(scheme, dict(quant_bits=4, wire_bits=4), gcb.RotatedQuantConfig(4, 4), n, d, grads, 7)
    elif scheme == "topk":
        _check(scheme, dict(k=100), gcb.TopKConfig(100), n, d, grads, 7)
    elif scheme == "chunked_topk":
        _check(scheme, dict(chunk_size=64, chunks_selected=5), gcb.ChunkedTopKConfig(64, 5), n, d, grads, 7)
    else:
        outs = oracle_rounds("dense", dict(bits=16), grads, 7, ef=False)
        pipe = gcb.make_pipeline(gcb.DenseConfig(16), n, d, gcb.SeedSpec(7))
        for r, g in enumerate(grads):
            assert np.array_equal(pipe.run_round(g, r).estimate.logical, outs[r]["estimate"])


@pytest.mark.parametrize("d,k", [(1, 1), (7, 7), (100, 1), (4096, 4096)])
def test_topk_small(d, k):
    import paper_2407_01378_b200 as gcb
    _check("topk", dict(k=k), gcb.TopKConfig(k), 2, d, _grads(d, 2, d, 2), 23)


@pytest.mark.parametrize("d,C,J", [(1, 1, 1), (10, 64, 1), (1000, 1, 1000), (999, 1000, 1), (65_537, 129, 100)])
def test_chunked_small(d, C, J):
    import paper_2407_01378_b200 as gcb
    _check("chunked_topk", dict(chunk_size=C, chunks_selected=J), gcb.ChunkedTopKConfig(C, J), 3, d,
           _grads(d, 3, d, 2), 29)


@pytest.mark.parametrize("d,rank,bypass", [(1, 1, 4096), (4095, 4, 4096), (4096, 4, 4096), (5000, 3, 0),
                                           (100_000, 7, 4096), (20, 4, 0)])
def test_powersgd_shapes(d, rank, bypass):
    import paper_2407_01378_b200 as gcb
    _check("powersgd", dict(rank=rank, bypass_below=bypass), gcb.PowerSgdConfig(rank, True, bypass), 2, d,
           _grads(d, 2, d, 3), 37, exact=False)


def test_validation_errors_match_reference():
    import paper_2407_01378_b200 as gcb
    with pytest.raises(ValueError):
        gcb.make_pipeline(gcb.TopKConfig(20), 2, 10, gcb.SeedSpec(1))
    with pytest.raises(ValueError):
        gcb.make_pipeline(gcb.ChunkedTopKConfig(4, 5), 2, 10, gcb.SeedSpec(1))
    with pytest.raises(ValueError):
        gcb.make_pipeline(gcb.DenseConfig(16), 2, 10, gcb.SeedSpec(1), error_feedback=True)
    pipe = gcb.make_pipeline(gcb.TopKConfig(2), 2, 10, gcb.SeedSpec(1))
    with pytest.raises(ValueError):
        pipe.run_round([np.ones(10, np.float32)], 0)
    with pytest.raises(ValueError):
        pipe.run_round([np.ones(9, np.float32)] * 2, 0)
    bad = np.ones(10, np.float32)
    bad[3] = np.nan
    with pytest.raises(ValueError):
        pipe.run_round([bad, np.ones(10, np.float32)], 0)
    assert gcb.make_pipeline(gcb.TopKConfig(2), 2, 8, gcb.SeedSpec(1), error_feedback=False).residuals is None
