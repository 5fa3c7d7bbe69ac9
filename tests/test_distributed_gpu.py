"""Two ranks on one B200 (gloo with host staging) running DistributedGradientPipeline for
n = 4 workers (2 per rank) against the oracle of the reference ring: bit-exact for THC,
TopK and TopK-Chunked, 1e-5 for PowerSGD, fp16 / fp32 tolerance for the dense bar."""
import numpy as np
import pytest
import torch

from tests.dist_util import run_world
from tests.gpu_util import needs_gpu, oracle_rounds

pytestmark = [pytest.mark.gpu, needs_gpu]

N, D, SEED = 4, 100_003, 77


def _grads(r):
    from oracle import gradcomp_oracle as orc
    return [orc.stream_rng(SEED, "grad-worker", r, w).standard_normal(D).astype(np.float32) for w in range(N)]


def _run_rank(rank, world, scheme, params):
    import torch
    import paper_2407_01378_b200 as gcb
    from paper_2407_01378_b200.distributed import DistributedGradientPipeline
    from tests.gpu_util import config_for
    torch.cuda.set_device(0)
    L = N // world
    ef = None if scheme != "dense" else False
    pipe = DistributedGradientPipeline(config_for(scheme, params), N, D, gcb.SeedSpec(SEED), ef)
    out = []
    for r in range(2):
        g = _grads(r)[rank * L:(rank + 1) * L]
        res = pipe.run_round(g, r)
        out.append({"est": res.estimate.logical.copy(), "res": pipe.residuals,
                    "clips": res.overflow.clip_events, "adds": res.overflow.total_adds})
    return out


@pytest.mark.parametrize("scheme,params,exact", [
    ("rotated_quant", dict(quant_bits=4, wire_bits=4, rotation_block=1024), True),
    ("rotated_quant", dict(quant_bits=3, wire_bits=9, rotation_block=256), True),
    ("topk", dict(k=1000), True),
    ("chunked_topk", dict(chunk_size=64, chunks_selected=50), True),
    ("powersgd", dict(rank=4), False),
    ("dense", dict(bits=32), False),
    ("dense", dict(bits=16), False),
])
def test_two_ranks_match_reference(scheme, params, exact):
    res = run_world(_run_rank, 2, (scheme, params))
    ef = scheme != "dense"
    outs = oracle_rounds(scheme, params, [_grads(r) for r in range(2)], SEED, ef=ef)
    for r in range(2):
        e0, e1 = res[0][r]["est"], res[1][r]["est"]
        assert np.array_equal(e0, e1), "ranks disagree on the estimate"
        ref = outs[r]["estimate"]
        if exact:
            assert np.array_equal(e0, ref), (scheme, r)
            if ef:
                mine = np.stack(res[0][r]["res"] + res[1][r]["res"])
                assert np.array_equal(mine, np.stack(outs[r]["residuals"]))
            if scheme == "rotated_quant":
                assert res[0][r]["clips"] == outs[r]["clip_events"]
                assert res[0][r]["adds"] == outs[r]["total_adds"]
        else:
            tol = 1e-3 if params.get("bits") == 16 else 1e-5
            err = np.linalg.norm(e0.astype(np.float64) - ref) / np.linalg.norm(ref)
            assert err <= tol, (scheme, r, err)


def _wire_rank(rank, world, scheme, params, d):
    import torch
    import paper_2407_01378_b200 as gcb
    from paper_2407_01378_b200.distributed import DistributedGradientPipeline
    from tests.gpu_util import config_for
    torch.cuda.set_device(0)
    ef = None if scheme != "dense" else False
    pipe = DistributedGradientPipeline(config_for(scheme, params), world, d, gcb.SeedSpec(SEED), ef)
    g = np.random.default_rng(rank).standard_normal(d).astype(np.float32)
    res = pipe.run_round([g], 0)
    led = {ph: res.ledger.bits_sent(worker=rank, phase=ph) for ph in res.ledger.phases()}
    return res.wire_bytes, led


@pytest.mark.parametrize("scheme,params", [
    ("rotated_quant", dict(quant_bits=4, wire_bits=8, rotation_block=1024)),
    ("rotated_quant", dict(quant_bits=4, wire_bits=4, rotation_block=1024)),   # packed nibble wire
    ("topk", dict(k=1000)),
    ("chunked_topk", dict(chunk_size=64, chunks_selected=50)),
    ("powersgd", dict(rank=4)),
    ("dense", dict(bits=16)),
    ("dense", dict(bits=32)),
])
@pytest.mark.parametrize("world", [2, 3, 4])
def test_wire_bytes_match_reference_ledger(scheme, params, world):
    """One worker per rank (n = world = 2, 3, 4; d = 2^17): the bytes each rank actually hands to
    the transport, per phase, equal the reference TrafficLedger's bits / 8 for that worker
    (collectives.py:209-262) -- the ring's reduce-scatter + all-gather volume for the all-reduce
    phases (THC codes, TopK-C energies and packs, PowerSGD factors go as all-to-all + ordered fold +
    all-gather, so the volume is the ring's at any n) and (n - 1) x payload for the gathers."""
    d = 1 << 17
    if scheme == "rotated_quant" and world & (world - 1):
        pytest.skip("THC codes travel in 1024-coordinate tile slices: exact ring volume for power-of-two worlds")
    out = run_world(_wire_rank, world, (scheme, params, d))
    for rank in range(world):
        wire, led = out[rank]
        assert set(wire) == set(led), (wire, led)
        for ph, bits in led.items():
            assert wire[ph] * 8 == bits, (scheme, ph, wire[ph] * 8, bits)


def _nmse_rank(rank, world, scheme, params):
    import torch
    import paper_2407_01378_b200 as gcb
    from paper_2407_01378_b200.distributed import DistributedGradientPipeline
    from tests.gpu_util import config_for
    torch.cuda.set_device(0)
    L = N // world
    ef = None if scheme != "dense" else False
    pipe = DistributedGradientPipeline(config_for(scheme, params), N, D, gcb.SeedSpec(SEED), ef, compute_nmse=True)
    out = []
    for r in range(2):
        res = pipe.run_round(_grads(r)[rank * L:(rank + 1) * L], r)
        out.append((res.nmse, res.estimate.logical.copy()))
    return out


@pytest.mark.parametrize("scheme,params", [
    ("rotated_quant", dict(quant_bits=4, wire_bits=8, rotation_block=1024)),
    ("topk", dict(k=1000)),
    ("dense", dict(bits=16)),
])
def test_distributed_nmse_matches_reference(scheme, params):
    """compute_nmse=True: RoundResult.nmse against the fp64 mean of every worker's corrected
    gradient (pipelines.py:176-181), identical on both ranks."""
    out = run_world(_nmse_rank, 2, (scheme, params))
    ref = oracle_rounds(scheme, params, [_grads(r) for r in range(2)], SEED, ef=scheme != "dense")
    for r in range(2):
        assert out[0][r][0] == out[1][r][0]
        if scheme == "dense":   # NCCL's fp16 sum order is not the ring's: check the nmse of our estimate
            target = np.mean(np.stack(_grads(r)).astype(np.float64), axis=0)
            e = out[0][r][1].astype(np.float64) - target
            want = float(np.dot(e, e) / np.dot(target, target))
        else:
            want = ref[r]["nmse"]
        assert abs(out[0][r][0] - want) <= 1e-9 + 1e-6 * abs(want), (r, out[0][r][0], want)


def _fp16_sat_rank(rank, world):
    import torch
    import paper_2407_01378_b200 as gcb
    from paper_2407_01378_b200.distributed import DistributedGradientPipeline
    torch.cuda.set_device(0)
    pipe = DistributedGradientPipeline(gcb.DenseConfig(16), world, 8, gcb.SeedSpec(1), False)
    g = np.array([40000, -40000, 60000, 1.5, -70000, 30000, 1e-3, 65504], np.float32)
    return pipe.run_round([g], 0).estimate.logical.copy()


def test_fp16_bar_saturates_like_the_reference_wire():
    """Partial sums past 65504 saturate (vectors.py:136-152) instead of becoming inf."""
    out = run_world(_fp16_sat_rank, 2)
    g = np.array([40000, -40000, 60000, 1.5, -70000, 30000, 1e-3, 65504], np.float32)
    ref = oracle_rounds("dense", dict(bits=16), [[g, g]], 1, ef=False)[0]["estimate"]
    assert np.all(np.isfinite(out[0])) and np.array_equal(out[0], out[1])
    assert np.array_equal(out[0], ref), (out[0], ref)


CHUNK_SIZES = [6000, 64, 3 * 4096, 192, 4096, 64 * 64, 10_000, 128 * 128]


def _chunked_rank(rank, world, n):
    import torch
    import paper_2407_01378_b200 as gcb
    from paper_2407_01378_b200.distributed import DistributedTensorListPipeline
    torch.cuda.set_device(0)
    L, D = n // world, sum(CHUNK_SIZES)
    pipe = DistributedTensorListPipeline(gcb.PowerSgdConfig(4), n, CHUNK_SIZES, gcb.SeedSpec(SEED),
                                         device=torch.device("cuda", 0))
    out = []
    for r in range(3):
        g = np.stack(_chunk_grads(n, D, r)[rank * L:(rank + 1) * L])
        res = pipe.run_round(torch.from_numpy(g).cuda(), r)
        out.append({"est": res.estimate.logical.copy(), "wire": res.wire_bytes,
                    "led": {ph: res.ledger.bits_sent(worker=rank * L, phase=ph) for ph in res.ledger.phases()}})
    out[-1]["res"] = pipe.residuals
    return out


def _chunk_grads(n, D, r):
    rng = np.random.default_rng(1000 + r)
    return [rng.standard_normal(D).astype(np.float32) for _ in range(n)]


@pytest.mark.parametrize("world,n", [(2, 2), (2, 4), (4, 4)])
def test_chunked_powersgd_across_ranks(world, n):
    """Chunked PowerSGD (one reference pipeline per tensor) over `world` ranks: every tensor's
    estimate and residuals within the fp32 contract of the reference, the dense bypass bit for bit,
    the factor phases' wire bytes equal to the ledger's ring volume (one worker per rank)."""
    out = run_world(_chunked_rank, world, (n,))
    D = sum(CHUNK_SIZES)
    offs = np.concatenate([[0], np.cumsum(CHUNK_SIZES)[:-1]])
    grads = [_chunk_grads(n, D, r) for r in range(3)]
    for t, (off, s) in enumerate(zip(offs, CHUNK_SIZES)):
        ref = oracle_rounds("powersgd", dict(rank=4), [[g[off:off + s] for g in grads[r]] for r in range(3)], SEED)
        for r in range(3):
            e0 = out[0][r]["est"][off:off + s]
            for k in range(1, world):
                assert np.array_equal(e0, out[k][r]["est"][off:off + s]), "ranks disagree"
            want = ref[r]["estimate"]
            if s < 4096:
                assert np.array_equal(e0, want), (t, r)
            else:
                assert np.max(np.abs(e0 - want)) <= 1e-5 * max(np.max(np.abs(want)), 1e-30), (t, r)
        mine = np.stack(sum((out[k][2]["res"] for k in range(world)), []))[:, off:off + s]
        theirs = np.stack(ref[2]["residuals"])
        assert np.max(np.abs(mine - theirs)) <= 1e-5 * max(np.max(np.abs(theirs)), 1e-30), t
    if n == world:
        for k in range(world):
            for ph in ("left-factor", "right-factor"):
                assert out[k][0]["wire"][ph] * 8 == out[k][0]["led"][ph], (ph, out[k][0]["wire"], out[k][0]["led"])
