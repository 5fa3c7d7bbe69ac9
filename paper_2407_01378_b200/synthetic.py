"""Synthetic gradient stream on the GPU: the input of the scheme / nmse sweeps.

Model: the reference's SyntheticGradSpec (trainbench.py:31-113).  A shared magnitude envelope
env = |AR(1)(rho)| lifted by `spike_boost` on hot rows of width 2^round(log2(1/(1-rho))), fixed
signs, and per round

    base    = signs * env + noise_sigma * zeta_r                       (trainbench.py:94-96)
    g_{r,w} = f32(base + divergence * (env * xi_{r,w} + noise_sigma * eta_{r,w}))   (:99-108)

The round-independent part -- envelope, hot rows and signs, drawn from the "grad-shared" stream --
is the reference's exactly: numpy PCG64 from the same SeedSpec chain, scipy's lfilter for the
AR(1) (trainbench.py:68-71, 82-93), computed once on the host.  The per-round Gaussian fields
zeta, xi, eta are drawn on the GPU (torch's Philox, one generator per (tag, round, worker) seeded
from the reference's stream seeds) instead of numpy's ziggurat: numpy's generator is a
sequential rejection sampler (a normal consumes a variable number of draws), so reproducing it
bit for bit at 10^8..10^9 coordinates per round would be a CPU-speed serial walk -- the reason
SURVEY §8(f) asks for a GPU generator.  The gradients are therefore the reference's model with
the same spatial structure and the same distribution per round, not the reference's values;
parity tests use the oracle's exact stream, sweeps use this one (fresh gradients every round).
"""

from __future__ import annotations

import math

import numpy as np
import torch

from .vectors import SeedSpec


def row_width(rho: float) -> int:
    """trainbench.py:74-78."""
    if rho <= 0.0:
        return 1
    return 1 << max(0, round(math.log2(1.0 / (1.0 - rho))))


class SyntheticGradients:
    """Worker gradients of round r as one [n, dim] float32 CUDA tensor (fresh every round)."""

    def __init__(self, dim: int, seeds: SeedSpec, *, rho: float = 0.99, spike_density: float = 0.05,
                 spike_boost: float = 10.0, noise_sigma: float = 0.1, divergence: float = 0.3, device=None):
        if dim < 2:
            raise ValueError("dim must be at least 2")
        if not -1.0 < rho < 1.0:
            raise ValueError("rho must be in (-1, 1)")
        if not 0.0 <= spike_density <= 1.0:
            raise ValueError("spike_density must be a probability")
        if noise_sigma < 0 or divergence < 0 or spike_boost < 1:
            raise ValueError("noise_sigma, divergence >= 0 and spike_boost >= 1 required")
        from scipy.signal import lfilter
        self.dim, self.seeds = dim, seeds
        self.noise_sigma, self.divergence = float(noise_sigma), float(divergence)
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        rng = seeds.rng("grad-shared")                                        # trainbench.py:82-93
        innovations = rng.standard_normal(dim)
        signs = rng.integers(0, 2, dim) * 2.0 - 1.0
        env = np.abs(lfilter([math.sqrt(1.0 - rho * rho)], [1.0, -rho], innovations))
        del innovations
        if spike_density > 0.0:
            width = row_width(rho)
            hot_rows = rng.random(-(-dim // width)) < spike_density
            env += spike_boost * np.repeat(hot_rows, width)[:dim]
        self.env = torch.from_numpy(env).to(self.device)                       # fp64, as the reference
        self.signed_env = torch.from_numpy(signs * env).to(self.device)
        del env, signs

    def _normal(self, tag: str, round_index: int, worker=None) -> torch.Tensor:
        gen = torch.Generator(device=self.device)
        gen.manual_seed(self.seeds.stream_seed(tag, round_index, worker) & ((1 << 63) - 1))
        return torch.randn(self.dim, dtype=torch.float64, device=self.device, generator=gen)

    def base(self, round_index: int) -> torch.Tensor:
        """trainbench.py:94-96: signs * env + noise_sigma * zeta_r (fp64)."""
        return self.signed_env + self.noise_sigma * self._normal("grad-noise", round_index)

    def round(self, round_index: int, num_workers: int, out: torch.Tensor | None = None) -> torch.Tensor:
        """trainbench.py:99-113 for workers 0..num_workers-1 -> [num_workers, dim] float32."""
        if out is None:
            out = torch.empty(num_workers, self.dim, dtype=torch.float32, device=self.device)
        base = self.base(round_index)
        for w in range(num_workers):
            xi = self._normal("grad-worker-xi", round_index, w)
            eta = self._normal("grad-worker-eta", round_index, w)
            out[w].copy_(base + self.divergence * (self.env * xi + self.noise_sigma * eta))
        return out
