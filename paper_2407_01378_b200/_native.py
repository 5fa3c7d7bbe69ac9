"""ctypes binding of libgradcomp_b200.so (the C ABI declared in include/gradcomp_b200.h).

There is no fallback: if the library is missing the import fails loudly, and every
entry point raises on a non-zero status with the library's own error message.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_int, c_int32, c_int64, c_size_t, c_uint64, c_void_p

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GRADCOMP_B200_LIB", os.path.join(_HERE, "libgradcomp_b200.so"))

GC_OK = 0
GC_ERR_INVALID = -1
GC_ERR_CUDA = -2
GC_ERR_UNSUPPORTED = -3

# gc_topk_select flags (include/gradcomp_b200.h)
TOPK_FP16_VALUES = 1
TOPK_EF_UPDATE = 2


class Pcg64(ctypes.Structure):
    """gc_pcg64: numpy PCG64 state (128-bit state and increment)."""

    _fields_ = [("state_hi", c_uint64), ("state_lo", c_uint64), ("inc_hi", c_uint64), ("inc_lo", c_uint64)]

    @property
    def state(self) -> int:
        return (self.state_hi << 64) | self.state_lo

    @property
    def inc(self) -> int:
        return (self.inc_hi << 64) | self.inc_lo

    @classmethod
    def from_ints(cls, state: int, inc: int) -> "Pcg64":
        m = (1 << 64) - 1
        return cls(state >> 64, state & m, inc >> 64, inc & m)


class ThcGeom(ctypes.Structure):
    _fields_ = [("dim", c_int64), ("padded", c_int64), ("block", c_int64), ("quant_bits", c_int32),
                ("wire_bits", c_int32), ("scale", c_double)]


class PsgdBatch(ctypes.Structure):
    """gc_psgd_batch: T same-shape tensors x L workers (row_offsets / est_offsets are device int64)."""

    _fields_ = [("tensors", c_int32), ("workers", c_int32), ("row_offsets", c_void_p), ("ld", c_int64),
                ("est_offsets", c_void_p), ("rows_aligned", c_int32), ("est_accumulate", c_int32)]


P = c_void_p
I64 = c_int64
I32 = c_int32

# symbol -> (restype, argtypes).  Kept in the order of include/gradcomp_b200.h.
SIGNATURES = {
    "gc_version": (c_int, []),
    "gc_last_error": (c_char_p, []),
    "gc_splitmix64": (c_uint64, [c_uint64]),
    "gc_fnv1a64": (c_uint64, [c_char_p, c_size_t]),
    "gc_stream_seed": (c_uint64, [c_uint64, c_char_p, c_size_t, c_uint64, c_int64]),
    "gc_pcg64_from_seed": (None, [c_uint64, POINTER(Pcg64)]),
    "gc_pcg64_advance": (None, [POINTER(Pcg64), c_uint64, c_uint64]),
    "gc_pcg64_next": (c_uint64, [POINTER(Pcg64)]),
    "gc_check_finite": (c_int, [I64, P, I64, I64, P, P]),
    "gc_nmse_accumulate": (c_int, [I32, I64, P, P, I64, P, P, P]),
    # THC
    "gc_thc_active_len": (c_int64, [POINTER(ThcGeom)]),
    "gc_thc_workspace_bytes": (c_int64, [POINTER(ThcGeom), I32]),
    "gc_thc_signs": (c_int, [POINTER(Pcg64), I64, P, P]),
    "gc_thc_rotate": (c_int, [POINTER(ThcGeom), I32, P, P, I64, P, P, P, P, P]),
    "gc_range_consensus": (c_int, [I32, I64, P, P, P]),
    "gc_thc_quantize": (c_int, [POINTER(ThcGeom), I32, P, P, POINTER(Pcg64), P, P, P]),
    "gc_sat_fold": (c_int, [I32, I64, P, I64, I64, I64, I32, P, P, P]),
    "gc_thc_decode_estimate": (c_int, [POINTER(ThcGeom), I32, P, I32, P, P, P, P, P]),
    "gc_thc_decode_ef": (c_int, [POINTER(ThcGeom), I32, P, P, P, P, P, I64, P, P]),
    "gc_thc_rank_ranges": (c_int, [POINTER(ThcGeom), I32, P, P, I64, I64, I64, P, P, P]),
    "gc_thc_rank_ranges_signs": (c_int, [POINTER(ThcGeom), I32, P, P, I64, I64, I64, POINTER(Pcg64), P, P, P]),
    "gc_thc_merge_ranges": (c_int, [I32, I64, P, P, P]),
    "gc_thc_rank_quant": (c_int, [POINTER(ThcGeom), I32, P, P, P, I64, I64, I64, P, P, POINTER(Pcg64), P, I64, I32,
                                  P, P]),
    "gc_thc_rank_decode": (c_int, [POINTER(ThcGeom), I32, P, I32, P, P, P, P]),
    "gc_thc_round_fused": (c_int, [POINTER(ThcGeom), I32, P, P, I64, P, POINTER(Pcg64), P, P, P, P, P]),
    "gc_thc_round_fused_range": (c_int, [POINTER(ThcGeom), I32, P, P, P, I64, I64, I64, P, POINTER(Pcg64), P, P, P,
                                          P, P]),
    # float folds
    "gc_float_fold": (c_int, [I32, I64, P, I64, I64, I64, I32, I32, I32, P, P]),
    "gc_float_fold_batched": (c_int, [I32, I32, I64, P, I64, I64, I32, I32, I32, P, I64, P]),
    "gc_float_fold_batched_slice": (c_int, [I32, I32, I64, P, I64, I64, I64, I64, I32, I32, I32, P, I64, P]),
    "gc_segment_fold_ef": (c_int, [I32, I32, P, P, P, P, I64, P, P]),
    "gc_segment_ef_fold": (c_int, [I32, I32, P, P, P, P, I64, P, P]),
    "gc_scale_div": (c_int, [I64, P, I32, P, P]),
    "gc_fp16_round": (c_int, [I64, P, P, P]),
    "gc_fold_to_half": (c_int, [I32, I64, P, I64, P, P]),
    "gc_half_mean_sat": (c_int, [I64, P, I32, P, P]),
    # TopK
    "gc_topk_workspace_bytes": (c_int64, [I32, I64]),
    "gc_topk_select": (c_int, [I32, I64, P, I64, I64, P, P, P, P, I32, P, P]),
    "gc_encode_sparse_payloads": (c_int, [I32, I64, P, P, P, I64, P]),
    "gc_sparse_accumulate": (c_int, [I32, I64, P, P, I64, P, P]),
    "gc_sparse_mean_workspace_bytes": (c_int64, [I32, I64]),
    "gc_quant_payload_nbytes": (c_int64, [I64, I64]),
    "gc_encode_quant_payloads": (c_int, [I32, I32, I64, I64, P, I64, I64, I64, P, I64, c_uint64, P, I64, P]),
    "gc_sparse_mean": (c_int, [I32, I64, P, P, I64, I32, P, P, P]),
    "gc_sparse_ef_update": (c_int, [I32, I64, P, P, P, I64, P]),
    # TopK-Chunked
    "gc_ef_apply": (c_int, [I32, I64, P, P, I64, P, I64, P]),
    "gc_chunk_norms": (c_int, [I32, I64, I64, P, I64, P, P, P]),
    "gc_chunk_norms_ef": (c_int, [I32, I64, I64, P, P, I64, P, P]),
    "gc_chunk_pack": (c_int, [I32, I64, I64, I64, P, P, I64, P, P, P]),
    "gc_chunk_scatter": (c_int, [I64, I64, I64, P, P, I32, P, P, P]),
    "gc_chunk_ef_update": (c_int, [I32, I64, I64, I64, P, P, P, P, I64, P]),
    # PowerSGD
    "gc_psgd_splits": (c_int, [I32, I64]),
    "gc_psgd_workspace_bytes": (c_int64, [I32, I64, I64, I32]),
    "gc_psgd_vectorizable": (c_int, [I64, P, P, I64]),
    "gc_psgd_mq": (c_int, [POINTER(PsgdBatch), I64, I64, I64, I32, P, P, P, P]),
    "gc_psgd_mq_fused": (c_int, [POINTER(PsgdBatch), I64, I64, I64, I32, P, P, P, P, P, P]),
    "gc_psgd_mq_tma_supported": (c_int, [POINTER(PsgdBatch), I64, I64, I64, I32, P, P]),
    "gc_psgd_mq_deferred": (c_int, [POINTER(PsgdBatch), I64, I64, I64, I32, P, P, P, P, P, P, P, P]),
    "gc_psgd_mq_tma_supported_batched": (c_int, [POINTER(PsgdBatch), P, I64, I64, I64, I32, P, P]),
    "gc_psgd_mq_deferred_batched": (c_int, [POINTER(PsgdBatch), P, I64, I64, I64, I32, P, P, P, P, P, P, P, P]),
    "gc_psgd_mq_deferred_supported": (c_int, [POINTER(PsgdBatch), P, I64, I64, I64, I32, P, P]),
    "gc_psgd_mtp": (c_int, [POINTER(PsgdBatch), I64, I64, I64, I32, P, P, P, P, P]),
    "gc_psgd_mtp_batched": (c_int, [POINTER(PsgdBatch), P, I64, I64, I64, I32, P, P, P, P, P]),
    "gc_psgd_mtp_ef_supported": (c_int, [I64, I64, I32, I32]),
    "gc_psgd_mtp_ef": (c_int, [POINTER(PsgdBatch), I64, I64, I64, I32, P, P, P, P]),
    "gc_psgd_orthonormalize": (c_int, [I32, I64, I32, P, P, P, P, P]),
    "gc_psgd_orth_workspace_bytes": (I64, [I32, I64, I32]),
    "gc_psgd_decode": (c_int, [POINTER(PsgdBatch), I32, I64, I64, I64, I32, P, P, P, P, P, P]),
    "gc_psgd_decode_fused": (c_int, [POINTER(PsgdBatch), I32, I64, I64, I64, I32, P, P, P, P, P, P]),
    "gc_psgd_gram_workspace_bytes": (I64, [I32, I32]),
    "gc_psgd_gram": (c_int, [I32, I64, I32, P, P, P, P]),
    "gc_fill_zero": (c_int, [P, I64, P]),
    "gc_pack_nibbles": (c_int, [I64, P, P, P]),
    "gc_unpack_nibbles": (c_int, [I64, P, P, P]),
    "gc_copy_rows_async": (c_int, [P, I64, P, I64, I64, I64, P]),
}

_lib = None


def _load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"libgradcomp_b200.so not found at {LIB_PATH}; build it with `make` or "
            "`python -c 'import __graft_entry__ as g; g.build()'` (there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name, None)
        if fn is None:
            continue  # reported by missing_symbols(); calling it raises below
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def lib():
    return _load()


def missing_symbols() -> list[str]:
    lb = _load()
    return [name for name in SIGNATURES if getattr(lb, name, None) is None]


class NativeError(RuntimeError):
    pass


def check(rc: int, what: str = "") -> None:
    if rc == GC_OK:
        return
    msg = _load().gc_last_error().decode(errors="replace")
    if rc == GC_ERR_INVALID:
        raise ValueError(f"{what}: {msg}" if what else msg)
    raise NativeError(f"{what}: {msg} (status {rc})" if what else f"{msg} (status {rc})")


_fns = {}


def call(name: str, *args) -> None:
    fn = _fns.get(name)
    if fn is None:
        fn = getattr(_load(), name, None)
        if fn is None:
            raise NativeError(f"{name} is not exported by {LIB_PATH}")
        _fns[name] = fn
    rc = fn(*args)
    if rc != GC_OK:
        check(rc, name)


try:   # the raw handle without building a torch.cuda.Stream object (host issue time per launch)
    import torch as _torch
    _raw_stream = _torch._C._cuda_getCurrentRawStream
    _cur_dev = _torch._C._cuda_getDevice
except (ImportError, AttributeError):   # pragma: no cover - older torch
    _raw_stream = _cur_dev = None


def current_stream_handle() -> int:
    """cudaStream_t of torch's current stream on the current device, as an int."""
    if _raw_stream is not None:
        return _raw_stream(_cur_dev())
    import torch
    return torch.cuda.current_stream().cuda_stream
