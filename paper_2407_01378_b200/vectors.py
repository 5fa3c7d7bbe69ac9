"""Seeds, padded gradient vectors and chunk geometry (mirror of gradcomp.vectors).

Seed derivation is native (gc_stream_seed / gc_pcg64_from_seed) so the device kernels
regenerate exactly the draws the reference gets from numpy's PCG64
(reference: pkg/src/gradcomp/vectors.py:26-76).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _native

HALF_MAX = 65504.0          # vectors.py:19
_MASK64 = (1 << 64) - 1


def splitmix64(value: int) -> int:
    """vectors.py:26-31 (native)."""
    return int(_native.lib().gc_splitmix64(value & _MASK64))


def fnv1a64(text: str) -> int:
    """vectors.py:34-39 (native)."""
    b = text.encode("utf-8")
    return int(_native.lib().gc_fnv1a64(b, len(b)))


@dataclass(frozen=True)
class SeedSpec:
    """Root of all randomness for one experiment (vectors.py:42-76).

    stream_seed(tag, round, worker) follows the reference's splitmix64/fnv1a64 chain;
    pcg(tag, round, worker) is the PCG64 state numpy would seed from it, which the kernels
    consume; rng(...) returns the numpy Generator (used on the host only for the PowerSGD
    seed matrix, whose ziggurat normals stay on the host as in the reference).
    """

    experiment_seed: int

    def __post_init__(self) -> None:
        if not 0 <= self.experiment_seed <= _MASK64:
            raise ValueError("experiment_seed must fit in 64 bits")

    def stream_seed(self, tag: str, round_index: int = 0, worker: int | None = None) -> int:
        if round_index < 0:
            raise ValueError("round_index must be non-negative")
        if worker is not None and worker < 0:
            raise ValueError("worker must be non-negative")
        b = tag.encode("utf-8")
        return int(_native.lib().gc_stream_seed(self.experiment_seed, b, len(b), round_index,
                                                -1 if worker is None else worker))

    def pcg(self, tag: str, round_index: int = 0, worker: int | None = None) -> _native.Pcg64:
        out = _native.Pcg64()
        _native.lib().gc_pcg64_from_seed(self.stream_seed(tag, round_index, worker), out)
        return out

    def rng(self, tag: str, round_index: int = 0, worker: int | None = None) -> np.random.Generator:
        return np.random.Generator(np.random.PCG64(self.stream_seed(tag, round_index, worker)))


def next_pow2(n: int) -> int:
    return 1 << (n - 1).bit_length()


class GradientVector:
    """A float32 vector padded to a power-of-two length (vectors.py:83-119).

    Host-backed (`values` numpy) or device-backed (`tensor`, a CUDA tensor holding the
    logical prefix); device-backed vectors copy to the host lazily on first access of
    `values` / `logical`, so a round can stay on the GPU end to end.
    """

    def __init__(self, values=None, logical_len: int | None = None, *, tensor=None, padded_len=None):
        self._tensor = tensor
        if tensor is not None:
            self.logical_len = int(logical_len if logical_len is not None else tensor.numel())
            self._padded = int(padded_len if padded_len is not None else next_pow2(self.logical_len))
            self._values = None
            return
        vals = np.array(values, dtype=np.float32, copy=True, order="C")
        if vals.ndim != 1 or vals.size == 0:
            raise ValueError("values must be a non-empty 1-d array")
        if vals.size & (vals.size - 1):
            raise ValueError("padded length must be a power of two")
        if logical_len is None or not 1 <= logical_len <= vals.size:
            raise ValueError("logical_len out of range")
        if not np.all(np.isfinite(vals)):
            bad = int(np.flatnonzero(~np.isfinite(vals))[0])
            raise ValueError(f"non-finite value at index {bad}")
        if np.any(vals[logical_len:]):
            raise ValueError("padding tail must be exactly zero")
        vals.flags.writeable = False
        self._values = vals
        self.logical_len = int(logical_len)
        self._padded = vals.size

    @property
    def padded_len(self) -> int:
        return self._padded

    @property
    def tensor(self):
        """Device tensor of the logical prefix (None for host-built vectors)."""
        return self._tensor

    @property
    def values(self) -> np.ndarray:
        if self._values is None:
            buf = np.zeros(self._padded, dtype=np.float32)
            buf[: self.logical_len] = self._tensor.detach().cpu().numpy()
            buf.flags.writeable = False
            self._values = buf
        return self._values

    @property
    def logical(self) -> np.ndarray:
        return self.values[: self.logical_len]


def pad_to_pow2(raw) -> GradientVector:
    """vectors.py:122-133."""
    arr = np.ascontiguousarray(raw, dtype=np.float32)
    if arr.ndim != 1 or arr.size == 0:
        raise ValueError("input must be a non-empty 1-d array")
    if not np.all(np.isfinite(arr)):
        bad = int(np.flatnonzero(~np.isfinite(arr))[0])
        raise ValueError(f"non-finite value at index {bad}")
    buf = np.zeros(next_pow2(arr.size), dtype=np.float32)
    buf[: arr.size] = arr
    return GradientVector(buf, arr.size)


@dataclass(frozen=True)
class ChunkGeometry:
    """vectors.py:155-177."""

    chunk_size: int
    num_chunks: int

    def __post_init__(self) -> None:
        if self.chunk_size < 1 or self.num_chunks < 1:
            raise ValueError("chunk_size and num_chunks must be positive")

    @classmethod
    def for_dim(cls, logical_len: int, chunk_size: int) -> "ChunkGeometry":
        if logical_len < 1:
            raise ValueError("logical_len must be positive")
        return cls(chunk_size, math.ceil(logical_len / chunk_size))

    def covered_len(self) -> int:
        return self.chunk_size * self.num_chunks
