"""Payload types and the reference's binary wire codec (compressors.py:150-373).

The engine keeps payloads in device buffers (TopK: int32 indices + fp16-valued floats per
worker; TopK-Chunked: chunk ids + packed fp16 values; THC: int8 codes + the shared block grid;
PowerSGD: the two factors).  These classes mirror the reference's frozen payload dataclasses
(same validation and `ValueError`s) and `encode_payload` / `decode_payload` produce and parse
the same little-endian bytes (`pkg/README.md:157-173`):

    Sparse   <B tag=1><I count><i4 idx * count><f2 val * count>
    ChunkSet <B tag=2><I num_ids><I chunk_size><i4 ids><f2 values>
    Quant    <B tag=3><B quant_bits><I block_size><I num_codes><I num_blocks><i1 codes><f4 ranges><Q rot id>
    LowRank  <B tag=4><I rows><I cols><I rank><f4 left><f4 right>
    Dense    <B tag=5><B bits><I count><f2|f4 values>

`encode_sparse_payloads_device` builds the Sparse byte streams of all workers directly from the
device buffers with one kernel (gc_encode_sparse_payloads), so a TopK round can hand wire bytes
to a transport without a host round trip.
"""

from __future__ import annotations

import ctypes
import struct
from dataclasses import dataclass
from typing import Union

import numpy as np
import torch

from . import _native


@dataclass(frozen=True)
class SparsePayload:
    """compressors.py:150-166: ascending indices and their fp16-rounded values."""

    indices: np.ndarray
    values: np.ndarray

    def __post_init__(self) -> None:
        idx = np.ascontiguousarray(self.indices, dtype=np.int32)
        vals = np.ascontiguousarray(self.values, dtype=np.float32)
        if idx.shape != vals.shape or idx.ndim != 1:
            raise ValueError("indices and values must be 1-d and equal length")
        if idx.size and (np.any(np.diff(idx) <= 0) or idx[0] < 0):
            raise ValueError("indices must be strictly ascending and non-negative")
        idx.flags.writeable = False
        vals.flags.writeable = False
        object.__setattr__(self, "indices", idx)
        object.__setattr__(self, "values", vals)


@dataclass(frozen=True)
class ChunkSetPayload:
    """compressors.py:169-190: ascending chunk ids and their dense values."""

    chunk_ids: np.ndarray
    chunk_size: int
    values: np.ndarray

    def __post_init__(self) -> None:
        ids = np.ascontiguousarray(self.chunk_ids, dtype=np.int32)
        vals = np.ascontiguousarray(self.values, dtype=np.float32)
        if ids.ndim != 1 or vals.ndim != 1:
            raise ValueError("chunk_ids and values must be 1-d")
        if ids.size and (np.any(np.diff(ids) <= 0) or ids[0] < 0):
            raise ValueError("chunk_ids must be strictly ascending and non-negative")
        if vals.size != ids.size * self.chunk_size:
            raise ValueError("values length must be num_ids * chunk_size")
        ids.flags.writeable = False
        vals.flags.writeable = False
        object.__setattr__(self, "chunk_ids", ids)
        object.__setattr__(self, "values", vals)


@dataclass(frozen=True)
class QuantPayload:
    """compressors.py:193-216: integer codes on a shared per-block grid, plus the grid."""

    codes: np.ndarray
    ranges: np.ndarray
    rotation_id: int
    quant_bits: int
    block_size: int

    def __post_init__(self) -> None:
        codes = np.ascontiguousarray(self.codes, dtype=np.int8)
        ranges = np.ascontiguousarray(self.ranges, dtype=np.float32)
        if codes.ndim != 1 or ranges.ndim != 2 or ranges.shape[1] != 2:
            raise ValueError("codes must be 1-d and ranges shaped (num_blocks, 2)")
        if codes.size != ranges.shape[0] * self.block_size:
            raise ValueError("codes length must be num_blocks * block_size")
        bound = (1 << (self.quant_bits - 1)) - 1
        if codes.size and int(np.abs(codes.astype(np.int64)).max()) > bound:
            raise ValueError("codes exceed the zero-mean grid bound")
        codes.flags.writeable = False
        ranges.flags.writeable = False
        object.__setattr__(self, "codes", codes)
        object.__setattr__(self, "ranges", ranges)


@dataclass(frozen=True)
class LowRankPayload:
    """compressors.py:219-244: factor pair, estimate = left @ right.T reshaped to shape."""

    left: np.ndarray
    right: np.ndarray
    shape: tuple

    def __post_init__(self) -> None:
        left = np.ascontiguousarray(self.left, dtype=np.float32)
        right = np.ascontiguousarray(self.right, dtype=np.float32)
        shape = (int(self.shape[0]), int(self.shape[1]))
        if left.ndim != 2 or right.ndim != 2 or left.shape[1] != right.shape[1]:
            raise ValueError("left and right must be 2-d with a common rank axis")
        if left.shape[0] != shape[0] or right.shape[0] != shape[1]:
            raise ValueError("factor row counts must match shape")
        left.flags.writeable = False
        right.flags.writeable = False
        object.__setattr__(self, "left", left)
        object.__setattr__(self, "right", right)
        object.__setattr__(self, "shape", shape)

    @property
    def rank(self) -> int:
        return self.left.shape[1]


@dataclass(frozen=True)
class DensePayload:
    """compressors.py:247-260: uncompressed values at a declared wire width."""

    values: np.ndarray
    bits: int

    def __post_init__(self) -> None:
        if self.bits not in (16, 32):
            raise ValueError("bits must be 16 or 32")
        vals = np.ascontiguousarray(self.values, dtype=np.float32)
        if vals.ndim != 1:
            raise ValueError("values must be 1-d")
        vals.flags.writeable = False
        object.__setattr__(self, "values", vals)


Payload = Union[SparsePayload, ChunkSetPayload, QuantPayload, LowRankPayload, DensePayload]

_TAGS = {SparsePayload: 1, ChunkSetPayload: 2, QuantPayload: 3, LowRankPayload: 4, DensePayload: 5}


def payload_bits(payload: Payload) -> int:
    """compressors.py:266-285: logical wire size charged by the ledger."""
    if isinstance(payload, SparsePayload):
        return 48 * payload.indices.size
    if isinstance(payload, ChunkSetPayload):
        return 16 * payload.values.size
    if isinstance(payload, QuantPayload):
        return payload.quant_bits * payload.codes.size + 64 * payload.ranges.shape[0]
    if isinstance(payload, LowRankPayload):
        return 32 * payload.rank * (payload.shape[0] + payload.shape[1])
    if isinstance(payload, DensePayload):
        return payload.bits * payload.values.size
    raise TypeError(f"unknown payload type {type(payload).__name__}")


def encode_payload(payload: Payload) -> bytes:
    """compressors.py:292-325: little-endian wire bytes."""
    tag = _TAGS.get(type(payload))
    if tag is None:
        raise TypeError(f"unknown payload type {type(payload).__name__}")
    parts = [struct.pack("<B", tag)]
    if tag == 1:
        parts += [struct.pack("<I", payload.indices.size), payload.indices.astype("<i4").tobytes(),
                  payload.values.astype("<f2").tobytes()]
    elif tag == 2:
        parts += [struct.pack("<II", payload.chunk_ids.size, payload.chunk_size),
                  payload.chunk_ids.astype("<i4").tobytes(), payload.values.astype("<f2").tobytes()]
    elif tag == 3:
        parts += [struct.pack("<BIII", payload.quant_bits, payload.block_size, payload.codes.size,
                              payload.ranges.shape[0]),
                  payload.codes.astype("<i1").tobytes(), payload.ranges.astype("<f4").tobytes(),
                  struct.pack("<Q", payload.rotation_id & ((1 << 64) - 1))]
    elif tag == 4:
        parts += [struct.pack("<III", payload.shape[0], payload.shape[1], payload.rank),
                  payload.left.astype("<f4").tobytes(), payload.right.astype("<f4").tobytes()]
    else:
        parts += [struct.pack("<BI", payload.bits, payload.values.size),
                  payload.values.astype("<f2" if payload.bits == 16 else "<f4").tobytes()]
    return b"".join(parts)


def decode_payload(blob: bytes) -> Payload:
    """compressors.py:328-373: parse bytes produced by encode_payload."""
    tag = blob[0]
    off = 1

    def take(fmt):
        nonlocal off
        vals = struct.unpack_from(fmt, blob, off)
        off += struct.calcsize(fmt)
        return vals

    def arr(dtype, count):
        nonlocal off
        a = np.frombuffer(blob, dtype=dtype, count=count, offset=off)
        off += a.nbytes
        return a

    if tag == 1:
        (count,) = take("<I")
        idx = arr("<i4", count)
        return SparsePayload(idx, arr("<f2", count).astype(np.float32))
    if tag == 2:
        num_ids, chunk_size = take("<II")
        ids = arr("<i4", num_ids)
        return ChunkSetPayload(ids, chunk_size, arr("<f2", num_ids * chunk_size).astype(np.float32))
    if tag == 3:
        quant_bits, block_size, num_codes, num_blocks = take("<BIII")
        codes = arr("<i1", num_codes)
        ranges = arr("<f4", 2 * num_blocks).reshape(num_blocks, 2)
        (rotation_id,) = take("<Q")
        return QuantPayload(codes, ranges, rotation_id, quant_bits, block_size)
    if tag == 4:
        rows, cols, rank = take("<III")
        left = arr("<f4", rows * rank).reshape(rows, rank)
        right = arr("<f4", cols * rank).reshape(cols, rank)
        return LowRankPayload(left, right, (rows, cols))
    if tag == 5:
        bits, count = take("<BI")
        return DensePayload(arr("<f2" if bits == 16 else "<f4", count).astype(np.float32), bits)
    raise ValueError(f"unknown payload tag {tag}")


def sparse_payload_nbytes(k: int) -> int:
    """Bytes of one encoded SparsePayload with k entries (tag + count + 4k + 2k)."""
    return 5 + 6 * k


def encode_sparse_payloads_device(idx: torch.Tensor, val: torch.Tensor) -> torch.Tensor:
    """Wire bytes of L SparsePayloads straight from the device TopK buffers.

    idx: int32 [L, k] ascending indices; val: float32 [L, k] (fp16-valued).  Returns a uint8
    device tensor [L, 5 + 6k]; row w equals encode_payload(SparsePayload(idx[w], val[w]))."""
    if idx.dim() != 2 or idx.shape != val.shape or idx.dtype != torch.int32 or val.dtype != torch.float32:
        raise ValueError("need int32 indices and float32 values shaped [workers, k]")
    L, k = idx.shape
    idx, val = idx.contiguous(), val.contiguous()
    out = torch.empty(L, sparse_payload_nbytes(k), dtype=torch.uint8, device=idx.device)
    _native.call("gc_encode_sparse_payloads", L, k, idx.data_ptr(), val.data_ptr(), out.data_ptr(),
                 out.stride(0), torch.cuda.current_stream().cuda_stream)
    return out


def quant_payload_nbytes(num_codes: int, num_blocks: int) -> int:
    """Bytes of one encoded QuantPayload (compressors.py:305-317)."""
    return 14 + num_codes + 8 * num_blocks + 8


def encode_quant_payloads_device(codes: torch.Tensor, ranges: torch.Tensor, quant_bits: int, block_size: int,
                                 num_codes: int, rotation_id: int = 0) -> torch.Tensor:
    """Wire bytes of L QuantPayloads straight from a THC round's device buffers.

    codes: int8 [L, active] (the engine's codes over the non-zero prefix); ranges: float32
    [active_blocks, 2] (the shared consensus grid); num_codes: the padded length P.  Codes and
    ranges past the given prefix are the zeros of the padded tail.  Returns uint8 [L, nbytes];
    row w equals encode_payload(QuantPayload(codes_w padded, ranges padded, rotation_id, q, B))."""
    if codes.dim() != 2 or codes.dtype != torch.int8 or ranges.dim() != 2 or ranges.shape[1] != 2 \
            or ranges.dtype != torch.float32 or num_codes % block_size:
        raise ValueError("need int8 codes [workers, n] and float32 ranges [blocks, 2], num_codes % block_size == 0")
    L = codes.shape[0]
    codes, ranges = codes.contiguous(), ranges.contiguous()
    nblocks = num_codes // block_size
    out = torch.empty(L, quant_payload_nbytes(num_codes, nblocks), dtype=torch.uint8, device=codes.device)
    _native.call("gc_encode_quant_payloads", L, quant_bits, block_size, num_codes, codes.data_ptr(),
                 codes.stride(0), codes.shape[1], nblocks, ranges.data_ptr(), ranges.shape[0],
                 rotation_id & ((1 << 64) - 1), out.data_ptr(), out.stride(0),
                 torch.cuda.current_stream().cuda_stream)
    return out
