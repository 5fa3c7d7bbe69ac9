"""Payload wire codec (compressors.py:292-373) vs the reference's own bytes, and the device
SparsePayload encoder vs the host codec."""
import struct

import numpy as np
import pytest
import torch

from tests.golden_util import GOLDEN
from tests.gpu_util import needs_gpu


def _golden():
    with np.load(f"{GOLDEN}/payloads.npz") as z:
        return {k: z[k] for k in z.files}


def _payloads(g):
    from paper_2407_01378_b200 import payloads as pl
    return {
        "sparse": pl.SparsePayload(g["sparse_idx"], g["sparse_val"]),
        "chunkset": pl.ChunkSetPayload(g["chunk_ids"], 64, g["chunk_vals"]),
        "quant": pl.QuantPayload(g["quant_codes"], g["quant_ranges"], 0xDEADBEEFCAFE, 4, 1024),
        "lowrank": pl.LowRankPayload(g["lr_left"], g["lr_right"], (30, 20)),
        "dense16": pl.DensePayload(g["dense_vals"], 16),
        "dense32": pl.DensePayload(g["dense_vals"], 32),
    }


def test_encode_matches_reference_bytes_and_round_trips():
    from paper_2407_01378_b200 import payloads as pl
    g = _golden()
    with np.errstate(over="ignore"):
        for name, p in _payloads(g).items():
            blob = pl.encode_payload(p)
            assert blob == g[f"{name}_bytes"].tobytes(), name
            assert pl.payload_bits(p) == int(g[f"{name}_bits"]), name
            back = pl.decode_payload(blob)
            assert type(back) is type(p)
            assert pl.encode_payload(back) == blob, name


def test_reference_golden_literals():
    """tests/test_compressors.py:120-138 of the reference (struct literals)."""
    from paper_2407_01378_b200 import payloads as pl
    p = pl.SparsePayload(np.array([1, 5], dtype=np.int32), np.array([1.5, -2.0], dtype=np.float32))
    expect = struct.pack("<B", 1) + struct.pack("<I", 2) + struct.pack("<2i", 1, 5) + struct.pack("<2e", 1.5, -2.0)
    assert pl.encode_payload(p) == expect
    d = pl.DensePayload(np.array([0.5, 3.0], dtype=np.float32), 16)
    assert pl.encode_payload(d) == struct.pack("<BBI", 5, 16, 2) + struct.pack("<2e", 0.5, 3.0)


def test_payload_validation_errors():
    from paper_2407_01378_b200 import payloads as pl
    with pytest.raises(ValueError, match="ascending"):
        pl.SparsePayload(np.array([3, 1]), np.array([1.0, 2.0]))
    with pytest.raises(ValueError, match="num_ids"):
        pl.ChunkSetPayload(np.array([0]), 4, np.zeros(3))
    with pytest.raises(ValueError, match="bound"):
        pl.QuantPayload(np.array([9, 0], dtype=np.int8), np.zeros((1, 2)), 0, 4, 2)
    with pytest.raises(ValueError, match="bits"):
        pl.DensePayload(np.zeros(2), 8)
    with pytest.raises(ValueError, match="unknown payload tag"):
        pl.decode_payload(b"\x09")


@pytest.mark.gpu
@needs_gpu
def test_device_sparse_payload_bytes_match_host_codec():
    """TopK round on the GPU -> wire bytes built on the device == encode_payload of the payload."""
    import paper_2407_01378_b200 as gcb
    from paper_2407_01378_b200 import payloads as pl
    n, d, k = 4, 300_000, 3_000
    seeds = gcb.SeedSpec(12)
    grads = [seeds.rng("grad-worker", 0, w).standard_normal(d).astype(np.float32) * 1e3 for w in range(n)]
    pipe = gcb.make_pipeline(gcb.TopKConfig(k), n, d, seeds)
    pipe._engine.capture = True
    pipe.run_round(grads, 0)
    idx, val = pipe._engine.last["idx"], pipe._engine.last["val"]
    dev = pl.encode_sparse_payloads_device(idx, val).cpu().numpy()
    for w in range(n):
        host = pl.encode_payload(pl.SparsePayload(idx[w].cpu().numpy(), val[w].cpu().numpy()))
        assert dev[w].tobytes() == host, w
    empty = pl.encode_sparse_payloads_device(idx[:, :0].contiguous(), val[:, :0].contiguous()).cpu().numpy()
    assert all(row.tobytes() == pl.encode_payload(pl.SparsePayload(np.zeros(0), np.zeros(0))) for row in empty)


@pytest.mark.gpu
@needs_gpu
@pytest.mark.parametrize("d,q,b,blk", [(300_001, 4, 8, 1024), (5000, 3, 4, 256)])
def test_device_quant_payload_bytes_match_host_codec(d, q, b, blk):
    """THC round on the GPU (multi-kernel path, codes and consensus ranges captured) -> QuantPayload
    wire bytes built on the device == encode_payload of the padded payload (zero tail included)."""
    import paper_2407_01378_b200 as gcb
    from paper_2407_01378_b200 import payloads as pl
    n = 3
    seeds = gcb.SeedSpec(21)
    grads = [seeds.rng("grad-worker", 0, w).standard_normal(d).astype(np.float32) for w in range(n)]
    pipe = gcb.make_pipeline(gcb.RotatedQuantConfig(q, b, blk), n, d, seeds, fused=False)
    pipe._engine.capture = True
    pipe.run_round(grads, 0)
    eng = pipe._engine
    codes, shared = eng.last["codes"], eng.last["shared"].float().reshape(-1, 2)
    P, B = eng.P, eng.B
    rot = 0x1234_5678_9ABC_DEF0
    dev = pl.encode_quant_payloads_device(codes, shared, q, B, P, rot).cpu().numpy()
    for w in range(n):
        full = np.zeros(P, np.int8)
        full[: codes.shape[1]] = codes[w].cpu().numpy()
        rng = np.zeros((P // B, 2), np.float32)
        rng[: shared.shape[0]] = shared.cpu().numpy()
        host = pl.encode_payload(pl.QuantPayload(full, rng, rot, q, B))
        assert dev[w].tobytes() == host, w
        back = pl.decode_payload(dev[w].tobytes())
        assert np.array_equal(back.codes, full) and np.array_equal(back.ranges, rng)
