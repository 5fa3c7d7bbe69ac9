"""The per-rank pipeline over a real NCCL communicator.

NCCL needs one GPU per rank and this box has one, so the NCCL path runs as a one-rank group:
every collective of the exchange plan (range all-reduce MAX, code all-to-all on byte views,
all-gathers of sums / payloads / factors, the FP16 bar's half all-reduce) is still issued to
NCCL (Comm does not shortcut one-rank NCCL groups) and the round must equal the reference's.
With world_size GPUs available (`GC_NCCL_WORLD`), the same test runs over that many ranks."""
import os

import numpy as np
import pytest
import torch

from tests.dist_util import run_world
from tests.gpu_util import needs_gpu, oracle_rounds

pytestmark = [pytest.mark.gpu, needs_gpu]

D, SEED = 50_003, 41


def _world():
    return max(1, min(int(os.environ.get("GC_NCCL_WORLD", "1")), torch.cuda.device_count()))


def _grads(n, r):
    from oracle import gradcomp_oracle as orc
    return [orc.stream_rng(SEED, "grad-worker", r, w).standard_normal(D).astype(np.float32) for w in range(n)]


def _rank(rank, world, scheme, params, n, seg_tiles=None):
    import os
    if seg_tiles:
        os.environ["GC_THC_RANK_SEG_TILES"] = str(seg_tiles)
    import torch
    import torch.distributed as dist
    import paper_2407_01378_b200 as gcb
    from paper_2407_01378_b200.distributed import DistributedGradientPipeline
    from tests.gpu_util import config_for
    assert dist.get_backend() == "nccl"
    L = n // world
    ef = None if scheme != "dense" else False
    pipe = DistributedGradientPipeline(config_for(scheme, params), n, D, gcb.SeedSpec(SEED), ef,
                                       device=torch.device("cuda", rank))
    out = []
    for r in range(2):
        res = pipe.run_round(_grads(n, r)[rank * L:(rank + 1) * L], r)
        out.append({"est": res.estimate.logical.copy(), "res": pipe.residuals, "clips": res.overflow.clip_events,
                    "wire": res.wire_bytes})
    return out


@pytest.mark.parametrize("scheme,params,exact", [
    ("rotated_quant", dict(quant_bits=4, wire_bits=8, rotation_block=1024), True),
    ("rotated_quant", dict(quant_bits=4, wire_bits=4, rotation_block=256), True),
    ("rotated_quant", dict(quant_bits=3, wire_bits=12, rotation_block=1024), True),
    ("topk", dict(k=500), True),
    ("chunked_topk", dict(chunk_size=64, chunks_selected=40), True),
    ("powersgd", dict(rank=4), False),
    ("dense", dict(bits=16), False),
    ("dense", dict(bits=32), False),
])
@pytest.mark.parametrize("per_rank", [1, 3])
def test_nccl_round_matches_reference(scheme, params, exact, per_rank):
    world = _world()
    n = per_rank * world
    out = run_world(_rank, world, (scheme, params, n), backend="nccl")
    ef = scheme != "dense"
    ref = oracle_rounds(scheme, params, [_grads(n, r) for r in range(2)], SEED, ef=ef)
    for r in range(2):
        got = out[0][r]["est"]
        for o in out[1:]:
            assert np.array_equal(o[r]["est"], got)
        want = ref[r]["estimate"]
        if exact:
            assert np.array_equal(got, want), (scheme, r)
            if ef:
                assert np.array_equal(np.stack(sum((o[r]["res"] for o in out), [])), np.stack(ref[r]["residuals"]))
            if scheme == "rotated_quant":
                assert out[0][r]["clips"] == ref[r]["clip_events"]
        else:
            tol = 1e-3 if params.get("bits") == 16 else 1e-5
            err = np.linalg.norm(got.astype(np.float64) - want) / np.linalg.norm(want)
            assert err <= tol, (scheme, r, err)


@pytest.mark.parametrize("params", [dict(quant_bits=4, wire_bits=8, rotation_block=1024),
                                    dict(quant_bits=4, wire_bits=4, rotation_block=128),
                                    dict(quant_bits=5, wire_bits=16, rotation_block=32)])
@pytest.mark.parametrize("per_rank", [1, 3])
def test_nccl_thc_segments(params, per_rank):
    """The per-rank THC round over 5-tile segments (K1 / async range all-reduce / K2 pipelined)."""
    world = _world()
    n = per_rank * world
    out = run_world(_rank, world, ("rotated_quant", params, n, 5), backend="nccl")
    ref = oracle_rounds("rotated_quant", params, [_grads(n, r) for r in range(2)], SEED)
    for r in range(2):
        assert np.array_equal(out[0][r]["est"], ref[r]["estimate"]), r
        assert np.array_equal(np.stack(sum((o[r]["res"] for o in out), [])), np.stack(ref[r]["residuals"]))
        assert out[0][r]["clips"] == ref[r]["clip_events"]
