"""Compressor configs, scheme labels, wire-size accounting and budget solvers.

Mirror of the reference's config surface (pkg/src/gradcomp/compressors.py:49-143, 266-285,
638-656): same names, fields, validation ranges and error types.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Union


class DegenerateMatrixError(ValueError):
    """compressors.py:41-42."""


@dataclass(frozen=True)
class TopKConfig:
    """compressors.py:49-57."""

    k: int

    def __post_init__(self) -> None:
        if self.k < 1:
            raise ValueError("k must be positive")


@dataclass(frozen=True)
class ChunkedTopKConfig:
    """compressors.py:60-75."""

    chunk_size: int
    chunks_selected: int
    permute: bool = False

    def __post_init__(self) -> None:
        if self.chunk_size < 1 or self.chunks_selected < 1:
            raise ValueError("chunk_size and chunks_selected must be positive")


@dataclass(frozen=True)
class RotatedQuantConfig:
    """compressors.py:78-97."""

    quant_bits: int
    wire_bits: int
    rotation_block: int = 1024

    def __post_init__(self) -> None:
        if not 2 <= self.quant_bits <= 8:
            raise ValueError("quant_bits must be in [2, 8]")
        if self.wire_bits < self.quant_bits or self.wire_bits > 32:
            raise ValueError("wire_bits must be in [quant_bits, 32]")
        if self.rotation_block < 2 or self.rotation_block & (self.rotation_block - 1):
            raise ValueError("rotation_block must be a power of two >= 2")


@dataclass(frozen=True)
class PowerSgdConfig:
    """compressors.py:100-112."""

    rank: int
    warm_start: bool = True
    bypass_below: int = 4096

    def __post_init__(self) -> None:
        if self.rank < 1:
            raise ValueError("rank must be positive")
        if self.bypass_below < 0:
            raise ValueError("bypass_below must be non-negative")


@dataclass(frozen=True)
class DenseConfig:
    """compressors.py:115-123."""

    bits: int = 16

    def __post_init__(self) -> None:
        if self.bits not in (16, 32):
            raise ValueError("bits must be 16 or 32")


CompressorConfig = Union[TopKConfig, ChunkedTopKConfig, RotatedQuantConfig, PowerSgdConfig, DenseConfig]


def scheme_label(config: CompressorConfig) -> str:
    """compressors.py:131-143."""
    if isinstance(config, TopKConfig):
        return "topk"
    if isinstance(config, ChunkedTopKConfig):
        return "chunked_topk_perm" if config.permute else "chunked_topk"
    if isinstance(config, RotatedQuantConfig):
        return "rotated_quant"
    if isinstance(config, PowerSgdConfig):
        return "powersgd"
    if isinstance(config, DenseConfig):
        return f"dense_fp{config.bits}"
    raise TypeError(f"unknown config type {type(config).__name__}")


def matrix_shape_for(size: int) -> tuple[int, int]:
    """Most-square (rows, cols) with rows*cols >= size (compressors.py:530-538)."""
    if size < 1:
        raise ValueError("size must be positive")
    rows = math.isqrt(size)
    if rows * rows < size:
        rows += 1
    return rows, math.ceil(size / rows)


def topk_for_budget(logical_len: int, bits_per_coord: float) -> int:
    """compressors.py:638-643."""
    k = round(bits_per_coord * logical_len / 48.0)
    if not 1 <= k <= logical_len:
        raise ValueError("budget resolves to an unusable k")
    return int(k)


def chunks_for_budget(logical_len: int, chunk_size: int, bits_per_coord: float) -> int:
    """compressors.py:646-656."""
    num_chunks = math.ceil(logical_len / chunk_size)
    j = round((bits_per_coord * logical_len / 16.0 - num_chunks) / chunk_size)
    if not 1 <= j <= num_chunks:
        raise ValueError("budget resolves to an unusable chunk count")
    return int(j)
