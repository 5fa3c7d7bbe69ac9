"""INTEGRATION.md §2, complete: the THC scheme core of the reference bound to libgradcomp_b200.so
through its C ABI with ctypes (include/gradcomp_b200.h), as a maintainer of the Python reference
would add it (e.g. as gradcomp/_b200.py).  Reference-side code: it uses the reference's own
TrafficLedger / OverflowStats and returns exactly what GradientPipeline._round_quant returns
(pipelines.py:260-322): (estimate f32[d], own list[f32[d]], input_bits, OverflowStats, range_clips).
Device buffers come from torch; the library never allocates.

Exercised by `bash tools/run_reference_tests.sh run-core` (tools/ref_shim/core_plugin.py swaps
GradientPipeline._round_quant for `round_quant_b200` and runs the reference's own tests)."""
from __future__ import annotations

import ctypes
import math
import os

import numpy as np
import torch

_LIB_PATH = os.environ.get(
    "GRADCOMP_B200_LIB",
    os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "..", "paper_2407_01378_b200",
                 "libgradcomp_b200.so"))
_lib = ctypes.CDLL(os.path.abspath(_LIB_PATH))


class Pcg64(ctypes.Structure):        # gc_pcg64
    _fields_ = [("state_hi", ctypes.c_uint64), ("state_lo", ctypes.c_uint64),
                ("inc_hi", ctypes.c_uint64), ("inc_lo", ctypes.c_uint64)]


class ThcGeom(ctypes.Structure):      # gc_thc_geom
    _fields_ = [("dim", ctypes.c_int64), ("padded", ctypes.c_int64), ("block", ctypes.c_int64),
                ("quant_bits", ctypes.c_int32), ("wire_bits", ctypes.c_int32), ("scale", ctypes.c_double)]


P, I32, I64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
G = ctypes.POINTER(ThcGeom)
_lib.gc_last_error.restype = ctypes.c_char_p
_lib.gc_pcg64_from_seed.argtypes = [ctypes.c_uint64, ctypes.POINTER(Pcg64)]
_lib.gc_pcg64_from_seed.restype = None
_lib.gc_thc_active_len.argtypes = [G]
_lib.gc_thc_active_len.restype = I64
_lib.gc_thc_workspace_bytes.argtypes = [G, I32]
_lib.gc_thc_workspace_bytes.restype = I64
_lib.gc_thc_signs.argtypes = [ctypes.POINTER(Pcg64), I64, P, P]
_lib.gc_thc_rotate.argtypes = [G, I32, P, P, I64, P, P, P, P, P]
_lib.gc_range_consensus.argtypes = [I32, I64, P, P, P]
_lib.gc_thc_quantize.argtypes = [G, I32, P, P, ctypes.POINTER(Pcg64), P, P, P]
_lib.gc_sat_fold.argtypes = [I32, I64, P, I64, I64, I64, I32, P, P, P]
_lib.gc_thc_decode_estimate.argtypes = [G, I32, P, I32, P, P, P, P, P]
_lib.gc_thc_decode_ef.argtypes = [G, I32, P, P, P, P, P, I64, P, P]


def _check(rc: int) -> None:
    if rc:
        raise RuntimeError(_lib.gc_last_error().decode())


def _pcg(seeds, tag: str, round_index: int, worker=None) -> Pcg64:
    """SeedSpec.stream_seed (vectors.py:64-76) -> the PCG64 state numpy would seed from it."""
    out = Pcg64()
    _lib.gc_pcg64_from_seed(seeds.stream_seed(tag, round_index, worker), ctypes.byref(out))
    return out


def round_quant_b200(pipe, corrected, ledger, round_index):
    """Drop-in for GradientPipeline._round_quant (pipelines.py:260-322) on the B200 kernels:
    rotation, range consensus, stochastic quantization, saturating ring fold, estimate decode and
    the own decode, bit for bit the reference's values."""
    from gradcomp.collectives import WorkerGroup  # noqa: F401  (the reference's own types)
    from gradcomp.metrics import OverflowStats

    cfg, n, d = pipe.config, pipe.group.size, pipe.dim
    padded = 1 << (d - 1).bit_length()
    block = 1 << min(padded.bit_length() - 1, cfg.rotation_block.bit_length() - 1)   # transforms.py:78
    geom = ThcGeom(d, padded, block, cfg.quant_bits, cfg.wire_bits, float(block) ** -0.5)
    gp = ctypes.byref(geom)
    active = int(_lib.gc_thc_active_len(gp))
    nb = active // block
    dev = torch.device("cuda", torch.cuda.current_device())
    st = torch.cuda.current_stream().cuda_stream
    c = torch.from_numpy(np.ascontiguousarray(np.stack(corrected), dtype=np.float32)).to(dev)
    ws_bytes = int(_lib.gc_thc_workspace_bytes(gp, n))
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=dev)
    signs = torch.empty(-(-active // 32), dtype=torch.int32, device=dev)
    x_rot = torch.empty(n, active, dtype=torch.float32, device=dev)
    ranges = torch.empty(n, nb, 2, dtype=torch.float32, device=dev)
    shared = torch.empty(nb, 2, dtype=torch.float32, device=dev)
    codes = torch.empty(n, active, dtype=torch.int8, device=dev)
    sum_bytes = 1 if cfg.wire_bits <= 8 else (2 if cfg.wire_bits <= 16 else 4)
    sums = torch.empty(active, dtype={1: torch.int8, 2: torch.int16, 4: torch.int32}[sum_bytes], device=dev)
    counters = torch.zeros(4, dtype=torch.int64, device=dev)   # clamps, sum z, sum z^2, clip events
    est = torch.empty(d, dtype=torch.float32, device=dev)
    neg_own = torch.zeros(n, d, dtype=torch.float32, device=dev)
    zeros = torch.zeros(n, d, dtype=torch.float32, device=dev)

    rot = _pcg(pipe.seeds, "rotation-signs", round_index)                            # transforms.py:80-82
    _check(_lib.gc_thc_signs(ctypes.byref(rot), active, signs.data_ptr(), st))
    # rht_forward + chunk_ranges (pipelines.py:263-270); corrected already has EF applied
    _check(_lib.gc_thc_rotate(gp, n, c.data_ptr(), None, d, signs.data_ptr(), x_rot.data_ptr(), ranges.data_ptr(),
                              ws.data_ptr(), st))
    # ElemMin / ElemMax ring consensus (pipelines.py:271-288)
    _check(_lib.gc_range_consensus(n, nb, ranges.data_ptr(), shared.data_ptr(), st))
    coins = (Pcg64 * n)(*[_pcg(pipe.seeds, "stochastic-round", round_index, w) for w in range(n)])   # :293
    _check(_lib.gc_thc_quantize(gp, n, x_rot.data_ptr(), shared.data_ptr(), coins, codes.data_ptr(),
                                counters.data_ptr(), st))
    # SatIntSum ring (pipelines.py:297-305): ring block j starts at worker j, clamp every hop
    ring_block = -(-padded // n)
    if n > 1:
        _check(_lib.gc_sat_fold(n, active, codes.data_ptr(), active, 0, ring_block, cfg.wire_bits, sums.data_ptr(),
                                counters[3:].data_ptr(), st))
        sums_ptr, sb = sums.data_ptr(), sum_bytes
    else:
        sums_ptr, sb = codes.data_ptr(), 1
    # dequantize_sum + rht_inverse, / n (pipelines.py:307-311)
    _check(_lib.gc_thc_decode_estimate(gp, n, sums_ptr, sb, shared.data_ptr(), signs.data_ptr(), est.data_ptr(),
                                       ws.data_ptr(), st))
    # own decode (pipelines.py:312-318): the EF kernel writes r = (g + r) - own; with g = r = 0 that
    # is -own exactly, so the reference's ef_update(corrected, own) sees the kernel's own bit for bit
    _check(_lib.gc_thc_decode_ef(gp, n, codes.data_ptr(), shared.data_ptr(), signs.data_ptr(), zeros.data_ptr(),
                                 neg_own.data_ptr(), d, ws.data_ptr(), st))
    own_h = (-neg_own).cpu().numpy()
    cnt = counters.cpu().numpy()
    # ledger (the reference's ring charges, collectives.py:209-233) and the result fields (:319-322)
    num_blocks = padded // block
    for phase, length, bits in (("range-consensus", num_blocks, 32), ("range-consensus", num_blocks, 32),
                                ("code-aggregate", padded, cfg.wire_bits)):
        if n > 1:
            per = 2 * (n - 1) * math.ceil(length / n) * bits
            for w in range(n):
                ledger.add(phase, w, sent=per, received=per)
    total = n * padded                                            # np.std over n * P codes, zeros included
    var = (total * int(cnt[2]) - int(cnt[1]) ** 2) / (total * total)
    overflow = OverflowStats(int(cnt[3]), (n - 1) * ring_block * n if n > 1 else 0, math.sqrt(max(var, 0.0)))
    input_bits = float(cfg.wire_bits * padded + 64 * num_blocks)
    return est.cpu().numpy(), [own_h[w].copy() for w in range(n)], input_bits, overflow, int(cnt[0])
