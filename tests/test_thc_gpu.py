"""THC on the GPU vs the reference golden vectors and the oracle (bit-exact)."""
import numpy as np
import pytest
import torch

from oracle import gradcomp_oracle as orc
from tests.golden_util import load
from tests.gpu_util import needs_gpu, oracle_rounds, run_golden_case

pytestmark = [pytest.mark.gpu, needs_gpu]

THC_CASES = ["thc_a", "thc_b", "thc_c", "thc_d", "thc_e", "thc_f"]


@pytest.mark.parametrize("fused", [True, False])
@pytest.mark.parametrize("name", THC_CASES)
def test_thc_golden_rounds_bit_exact(name, fused):
    for st, res, pipe, a in run_golden_case(name, fused=fused):
        r = st["round"]
        assert np.array_equal(res.estimate.logical, a[f"estimate_{r}"]), f"round {r} estimate"
        assert not np.any(res.estimate.values[pipe.dim:])
        if pipe.error_feedback:
            assert np.array_equal(np.stack(pipe.residuals), a[f"residuals_{r}"]), f"round {r} residuals"
        assert res.overflow.clip_events == st["clip_events"]
        assert res.overflow.total_adds == st["total_adds"]
        assert res.overflow.code_sigma == pytest.approx(st["code_sigma"], rel=1e-12)
        assert res.range_clips == st["range_clips"]
        assert res.nmse == pytest.approx(st["nmse"], rel=1e-9, abs=1e-15)
        assert res.input_bits_per_coord == pytest.approx(st["input_bits_per_coord"], rel=1e-15)
        led = {ph: [[res.ledger.bits_sent(worker=w, phase=ph), res.ledger.bits_received(worker=w, phase=ph)]
                    for w in range(pipe.group.size)] for ph in res.ledger.phases()}
        assert led == st["ledger"]


@pytest.mark.parametrize("fused", [True, False])
@pytest.mark.parametrize("name", ["thc_steps_a", "thc_steps_b", "thc_steps_c"])
def test_thc_codes_match_reference(name, fused):
    """Codes / sums / estimate from fixed corrected inputs (EF off) against the reference's steps."""
    import paper_2407_01378_b200 as gcb
    meta, a = load(name)
    pipe = gcb.make_pipeline(gcb.RotatedQuantConfig(meta["q"], meta["b"], meta["max_block"]), meta["n"], meta["d"],
                             gcb.SeedSpec(meta["seed"]), False, fused=fused)
    pipe._engine.capture = True
    res = pipe.run_round(list(a["corrected"]), meta["round"])
    active = pipe._engine.active
    codes = pipe._engine.last["codes"].cpu().numpy()
    assert np.array_equal(codes, a["codes"][:, :active])
    assert not np.any(a["codes"][:, active:])
    assert np.array_equal(res.estimate.logical, a["estimate"])
    assert res.overflow.clip_events == meta["clip_events"]
    if not pipe._engine.fused:
        last = pipe._engine.last
        assert np.array_equal(last["x_rot"].cpu().numpy(), a["rotated"][:, :active])
        assert np.array_equal(last["shared"].cpu().numpy(), a["shared"][: active // pipe._engine.B])
    # signs bitmask vs reference +-1 signs
    words = pipe._engine.signs.cpu().numpy().view(np.uint32)
    bits = ((words[:, None] >> np.arange(32, dtype=np.uint32)) & 1).reshape(-1)[:active]
    assert np.array_equal(bits * 2.0 - 1.0, a["signs"][:active])


@pytest.mark.parametrize("q,b,blk,n,d", [(4, 4, 1024, 4, 1 << 20), (4, 8, 1024, 4, 1 << 20),
                                          (4, 8, 1024, 8, 1_000_003), (3, 6, 256, 3, 300_000),
                                          (4, 4, 64, 2, 65_537), (8, 12, 512, 5, 100_000)])
def test_thc_vs_oracle_multi_round(q, b, blk, n, d):
    """cfg1-style parity: 2 rounds with carried EF, estimate and residuals bitwise."""
    import paper_2407_01378_b200 as gcb
    seed = 2024
    seeds = gcb.SeedSpec(seed)
    grads = [[seeds.rng("grad-worker", r, w).standard_normal(d).astype(np.float32) for w in range(n)]
             for r in range(2)]
    outs = oracle_rounds("rotated_quant", dict(quant_bits=q, wire_bits=b, rotation_block=blk), grads, seed)
    for fused in (True, False):
        pipe = gcb.make_pipeline(gcb.RotatedQuantConfig(q, b, blk), n, d, seeds, fused=fused)
        for r in range(2):
            res = pipe.run_round(grads[r], r)
            o = outs[r]
            assert np.array_equal(res.estimate.logical, o["estimate"]), (fused, r)
            assert np.array_equal(np.stack(pipe.residuals), np.stack(o["residuals"])), (fused, r)
            assert res.overflow.clip_events == o["clip_events"]
            assert res.overflow.total_adds == o["total_adds"]
            assert res.nmse == pytest.approx(o["nmse"], rel=1e-9)


def test_thc_device_tensor_inputs_and_determinism():
    import paper_2407_01378_b200 as gcb
    n, d = 8, 3_000_000
    g = torch.randn(n, d, device="cuda")
    outs = []
    for _ in range(2):
        pipe = gcb.make_pipeline(gcb.RotatedQuantConfig(4, 8), n, d, gcb.SeedSpec(7))
        r0 = pipe.run_round(g, 0)
        r1 = pipe.run_round(g, 1)
        # results stay valid after later rounds (fresh per-round output buffers)
        outs.append((r0.estimate_tensor, r1.estimate_tensor, pipe.residuals_tensor.clone()))
    for x, y in zip(*outs):
        assert torch.equal(x, y)
    assert not torch.equal(outs[0][0], outs[0][1])


@pytest.mark.parametrize("n,d", [(8, 3_000_017), (3, 70_001), (1, 5_000)])
def test_thc_host_streamed_round_matches_device_round(n, d):
    """Host inputs take the streamed path (PCIe in / kernel / PCIe out overlapped over tile
    segments, residual double-buffered); results equal the device-input round bit for bit."""
    import paper_2407_01378_b200 as gcb
    seeds = gcb.SeedSpec(11)
    grads = [[seeds.rng("grad-worker", r, w).standard_normal(d).astype(np.float32) for w in range(n)]
             for r in range(3)]
    host = gcb.make_pipeline(gcb.RotatedQuantConfig(4, 8), n, d, seeds)
    dev = gcb.make_pipeline(gcb.RotatedQuantConfig(4, 8), n, d, seeds)
    for r in range(4):
        gr = grads[r % 3]
        # round 0: list of numpy rows; 1: pinned rows; 2: one pinned [n, d] tensor (strided segment
        # copies); 3: one [n, d] numpy array
        feed = {0: gr, 1: [torch.from_numpy(x).pin_memory() for x in gr],
                2: torch.from_numpy(np.stack(gr)).pin_memory(), 3: np.stack(gr)}[r]
        a = host.run_round(feed, r)
        b = dev.run_round(torch.from_numpy(np.stack(gr)).cuda(), r)
        assert a.estimate_host is not None and b.estimate_host is None
        assert np.array_equal(a.estimate.logical, b.estimate.logical), r
        assert torch.equal(host.residuals_tensor, dev.residuals_tensor), r
        assert a.overflow.clip_events == b.overflow.clip_events
        assert a.overflow.code_sigma == b.overflow.code_sigma
        assert a.nmse == pytest.approx(b.nmse, rel=1e-12)


def test_thc_host_streamed_round_rejects_nonfinite_without_state_change():
    """pipelines.py:184-197: a non-finite gradient raises ValueError before any EF state change,
    even though the streamed round has already run tiles of earlier segments."""
    import paper_2407_01378_b200 as gcb
    n, d = 4, 2_000_000
    seeds = gcb.SeedSpec(3)
    pipe = gcb.make_pipeline(gcb.RotatedQuantConfig(4, 4), n, d, seeds)
    g0 = [seeds.rng("grad-worker", 0, w).standard_normal(d).astype(np.float32) for w in range(n)]
    pipe.run_round(g0, 0)
    before = pipe.residuals_tensor.clone()
    bad = [x.copy() for x in g0]
    bad[2][d - 10] = np.inf
    with pytest.raises(ValueError, match="finite"):
        pipe.run_round(bad, 1)
    assert torch.equal(pipe.residuals_tensor, before)
    ref = gcb.make_pipeline(gcb.RotatedQuantConfig(4, 4), n, d, seeds)
    ref.run_round(g0, 0)
    a, b = pipe.run_round(g0, 1), ref.run_round(g0, 1)
    assert np.array_equal(a.estimate.logical, b.estimate.logical)


@pytest.mark.parametrize("L,B,d,segs", [(1, 1024, 3_000_017, [(0, 1000), (1000, 2930)]),
                                        (2, 256, 400_000, [(0, 7), (7, 391)]),
                                        (3, 1024, 1_048_576, [(0, 1024)])])
def test_rank_k1_sign_draw_matches_signs_pass(L, B, d, segs):
    """Per-rank K1 drawing the rotation signs itself (gc_thc_rank_ranges_signs) against the separate
    gc_thc_signs pass + K1: identical sign words for every tile of every segment (written once, by
    worker 0's warps) and identical (-lo, hi) block tables."""
    import ctypes
    import paper_2407_01378_b200 as gcb
    from paper_2407_01378_b200 import _native
    P = 1 << (d - 1).bit_length()
    geom = _native.ThcGeom(d, P, B, 4, 8, float(B) ** -0.5)
    active = int(_native.lib().gc_thc_active_len(ctypes.byref(geom)))
    tiles, nb = -(-active // 1024), active // B
    assert segs[-1][1] == tiles
    gen = torch.Generator(device="cuda").manual_seed(3)
    g = torch.randn(L, d, device="cuda", generator=gen)
    r = torch.randn(L, d, device="cuda", generator=gen)
    rot = gcb.SeedSpec(77).pcg("rotation-signs", 5)
    sp = torch.cuda.current_stream().cuda_stream
    s_ref = torch.empty(tiles * 32, dtype=torch.int32, device="cuda")
    s_gen = torch.full((tiles * 32,), -1, dtype=torch.int32, device="cuda")
    n_ref = torch.empty(L, nb, 2, device="cuda")
    n_gen = torch.empty(L, nb, 2, device="cuda")
    _native.call("gc_thc_signs", ctypes.byref(rot), tiles * 1024, s_ref.data_ptr(), sp)
    for tb, te in segs:
        _native.call("gc_thc_rank_ranges", ctypes.byref(geom), L, g.data_ptr(), r.data_ptr(), d, tb, te,
                     s_ref.data_ptr(), n_ref.data_ptr(), sp)
        _native.call("gc_thc_rank_ranges_signs", ctypes.byref(geom), L, g.data_ptr(), r.data_ptr(), d, tb, te,
                     ctypes.byref(rot), s_gen.data_ptr(), n_gen.data_ptr(), sp)
    torch.cuda.synchronize()
    assert torch.equal(s_gen, s_ref)
    assert torch.equal(n_gen, n_ref)
