"""GradientPipeline on B200: drop-in for gradcomp.pipelines (pkg/src/gradcomp/pipelines.py:97-472).

Same constructor, `run_round`, `RoundResult`, `residuals` / `_warm_q` state and error
behaviour as the reference; every scheme core runs as sm_100a kernels from
libgradcomp_b200.so.  The n workers of a pipeline are simulated on one GPU (their
collectives become ring-ordered folds in HBM / shared memory); the multi-GPU form with
one rank per worker group is paper_2407_01378_b200.distributed.

Inputs may be numpy arrays / GradientVector (copied to the device) or torch tensors
(a CUDA [n, d] float32 tensor is used in place).  Outputs stay on the device; the
RoundResult materialises host copies lazily, so the numbers a reference caller reads
are identical while a device caller never synchronises.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _native
from .configs import (
    ChunkedTopKConfig, CompressorConfig, DenseConfig, PowerSgdConfig, RotatedQuantConfig, TopKConfig,
    scheme_label,
)
from .ledger import OverflowStats, TrafficLedger, WorkerGroup
from .vectors import ChunkGeometry, GradientVector, SeedSpec, next_pow2
from . import schemes


def _stream_ptr() -> int:
    return _native.current_stream_handle()


class RoundResult:
    """pipelines.py:59-76.  Fields are read lazily from the device."""

    def __init__(self, scheme: str, round_index: int, estimate_dev: torch.Tensor, dim: int,
                 ledger: TrafficLedger, input_bits: float, stats: "schemes.RoundStats"):
        self.scheme = scheme
        self.round_index = round_index
        self.ledger = ledger
        self.input_bits_per_coord = input_bits / dim
        self._est = estimate_dev
        self._dim = dim
        self._stats = stats
        self._estimate = None
        self._est_host = None

    @property
    def estimate(self) -> GradientVector:
        if self._estimate is None:
            src = self._est_host if self._est_host is not None else self._est
            self._estimate = GradientVector(tensor=src, logical_len=self._dim, padded_len=next_pow2(self._dim))
        return self._estimate

    @property
    def estimate_host(self) -> torch.Tensor | None:
        """Pinned host copy of the estimate, already complete, when the round was fed from host
        memory (the streamed path copies it back segment by segment); None otherwise."""
        return self._est_host

    @property
    def estimate_tensor(self) -> torch.Tensor:
        """Device estimate of the mean (logical length), no host copy."""
        return self._est

    @property
    def nmse(self) -> float:
        return self._stats.nmse()

    @property
    def overflow(self) -> OverflowStats:
        return self._stats.overflow()

    @property
    def range_clips(self) -> int:
        return self._stats.range_clips()


class GradientPipeline:
    """pipelines.py:97-393 (n simulated workers on the current CUDA device)."""

    def __init__(self, config: CompressorConfig, num_workers: int, dim: int, seeds: SeedSpec,
                 error_feedback: bool | None = None, *, device=None, validate: bool = True,
                 compute_nmse: bool = True, fused: bool = True):
        if num_workers < 1:
            raise ValueError("num_workers must be positive")
        if dim < 1:
            raise ValueError("dim must be positive")
        self.config = config
        self.scheme = scheme_label(config)
        self.group = WorkerGroup(num_workers)
        self.dim = dim
        self.seeds = seeds
        if isinstance(config, DenseConfig):
            if error_feedback:
                raise ValueError("dense baselines do not carry error feedback")
            error_feedback = False
        elif error_feedback is None:
            error_feedback = True
        self.error_feedback = bool(error_feedback)
        self._validate_config()
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.validate = validate
        self.compute_nmse = compute_nmse
        self._res = (torch.zeros(num_workers, dim, dtype=torch.float32, device=self.device)
                     if self.error_feedback else None)
        self._warm_q_dev: torch.Tensor | None = None
        self._stage: torch.Tensor | None = None
        self._engine = schemes.make_engine(config, num_workers, dim, seeds, self.device, fused=fused)

    def _validate_config(self) -> None:
        """pipelines.py:137-143."""
        cfg, d = self.config, self.dim
        if isinstance(cfg, TopKConfig) and cfg.k > d:
            raise ValueError("k exceeds the dimension")
        if isinstance(cfg, ChunkedTopKConfig):
            if cfg.chunks_selected > ChunkGeometry.for_dim(d, cfg.chunk_size).num_chunks:
                raise ValueError("chunks_selected exceeds the chunk count")

    # -- EF state (pipelines.py:129-134), exposed like the reference -----------------
    @property
    def residuals(self):
        if self._res is None:
            return None
        self._engine.sync_residuals(self._res)
        host = self._res.cpu().numpy()
        return [host[i].copy() for i in range(self.group.size)]

    @residuals.setter
    def residuals(self, value):
        self._engine.drop_deferred()
        if value is None:
            self._res = None
            self.error_feedback = False
            return
        if len(value) != self.group.size:
            raise ValueError("need one residual per worker")
        rows = [torch.as_tensor(np.asarray(v, dtype=np.float32) if not torch.is_tensor(v) else v,
                                dtype=torch.float32).reshape(-1) for v in value]
        self._res = torch.stack(rows).to(self.device).contiguous()
        self.error_feedback = True

    @property
    def residuals_tensor(self) -> torch.Tensor | None:
        if self._res is not None:
            self._engine.sync_residuals(self._res)
        return self._res

    @property
    def _warm_q(self):
        wq = self._engine.warm_q()
        return None if wq is None else wq.cpu().numpy()

    # -- round entry (pipelines.py:147-182) ---------------------------------------------
    def run_round(self, worker_grads, round_index: int) -> RoundResult:
        host_rows = self._host_rows(worker_grads)
        if host_rows is not None:
            return self._run_streamed(host_rows, round_index)
        grads = self._checked(worker_grads)
        ledger = TrafficLedger()
        est, input_bits, stats = self._engine.run(grads, self._res, round_index, ledger,
                                                  nmse=self.compute_nmse)
        return RoundResult(self.scheme, round_index, est, self.dim, ledger, input_bits, stats)

    # -- host-fed THC round: PCIe in, kernel and PCIe out overlapped -----------------------
    def _host_rows(self, worker_grads):
        """The n gradients as 1-d CPU float32 tensors when every one is host memory and the scheme
        streams (fused THC); None otherwise (the generic copy-then-run path)."""
        eng = self._engine
        if not (isinstance(eng, schemes.ThcEngine) and eng.fused) or eng.capture:
            return None
        if isinstance(worker_grads, np.ndarray) and worker_grads.ndim == 2:
            worker_grads = torch.from_numpy(np.ascontiguousarray(worker_grads, dtype=np.float32))
        if torch.is_tensor(worker_grads):
            # one [n, d] host tensor: every segment of all n rows is one strided PCIe copy
            if worker_grads.is_cuda or worker_grads.dim() != 2:
                return None
            if tuple(worker_grads.shape) != (self.group.size, self.dim):
                raise ValueError("need [num_workers, dim] gradients")
            return worker_grads.to(torch.float32).contiguous()
        if len(worker_grads) != self.group.size:
            raise ValueError("need exactly one gradient per worker")
        rows = []
        for x in worker_grads:
            if isinstance(x, GradientVector):
                x = x.tensor if x.tensor is not None else x.logical
            if torch.is_tensor(x):
                if x.is_cuda:
                    return None
                t = x
            else:
                t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32))
            if t.dim() != 1 or t.numel() != self.dim:
                raise ValueError("gradient length does not match the pipeline dim")
            rows.append(t.to(torch.float32).contiguous())
        return rows

    def _run_streamed(self, host_rows, round_index: int) -> RoundResult:
        """run_round for host inputs: ThcEngine.run_streamed writes the new residual to a second
        buffer, so a non-finite input (found by the per-segment checks) raises ValueError with the
        EF state untouched, as pipelines.py:184-197 does before any state change."""
        stage = self._stage_buffer()
        res_in = self._res
        res_out = None
        if res_in is not None:
            if getattr(self, "_res_alt", None) is None or self._res_alt.shape != res_in.shape:
                self._res_alt = torch.empty_like(res_in)
            res_out = self._res_alt
        ledger = TrafficLedger()
        est, est_host, input_bits, stats, bad = self._engine.run_streamed(
            host_rows, stage, res_in, res_out, round_index, ledger, nmse=self.compute_nmse)
        torch.cuda.current_stream().synchronize()   # a host caller reads the host estimate next
        if self.validate and int(bad.item()):
            raise ValueError("gradients must be finite")
        if res_in is not None:
            self._res, self._res_alt = res_out, res_in
        result = RoundResult(self.scheme, round_index, est, self.dim, ledger, input_bits, stats)
        result._est_host = est_host
        return result

    def _checked(self, worker_grads) -> torch.Tensor:
        """pipelines.py:184-197: one finite 1-d gradient of length dim per worker -> [n, d] device."""
        n, d = self.group.size, self.dim
        if torch.is_tensor(worker_grads) and worker_grads.dim() == 2:
            if worker_grads.shape[0] != n:
                raise ValueError("need exactly one gradient per worker")
            if worker_grads.shape[1] != d:
                raise ValueError("gradient length does not match the pipeline dim")
            g = worker_grads
            if g.dtype != torch.float32:
                raise ValueError("gradients must be float32")
            if g.device != self.device or not g.is_contiguous():
                g = self._staged(g)
        else:
            if len(worker_grads) != n:
                raise ValueError("need exactly one gradient per worker")
            stage = self._stage_buffer()
            for i, x in enumerate(worker_grads):
                if isinstance(x, GradientVector):
                    x = x.tensor if x.tensor is not None else x.logical
                t = x if torch.is_tensor(x) else torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32))
                if t.dim() != 1 or t.numel() != d:
                    raise ValueError("gradient length does not match the pipeline dim")
                stage[i].copy_(t.to(torch.float32), non_blocking=True)
            g = stage
        if self.validate:
            bad = torch.zeros(1, dtype=torch.int64, device=self.device)
            _native.call("gc_check_finite", n, g.data_ptr(), g.stride(0), d, bad.data_ptr(), _stream_ptr())
            self._engine.launches += 1
            if int(bad.item()):
                raise ValueError("gradients must be finite")
        return g

    def _stage_buffer(self) -> torch.Tensor:
        if self._stage is None:
            self._stage = torch.empty(self.group.size, self.dim, dtype=torch.float32, device=self.device)
        return self._stage

    def _staged(self, g: torch.Tensor) -> torch.Tensor:
        stage = self._stage_buffer()
        stage.copy_(g, non_blocking=True)
        return stage


def make_pipeline(config, num_workers, dim, seeds, error_feedback=None, **kw) -> GradientPipeline:
    """pipelines.py:418-425."""
    return GradientPipeline(config, num_workers, dim, seeds, error_feedback, **kw)


def _one_shot(config, worker_grads, seeds, round_index, residuals, error_feedback=None):
    """pipelines.py:428-440."""
    dim = int(np.asarray(worker_grads[0]).size) if not torch.is_tensor(worker_grads[0]) else worker_grads[0].numel()
    if residuals is not None and error_feedback is None:
        error_feedback = True
    pipe = GradientPipeline(config, len(worker_grads), dim, seeds, error_feedback)
    if residuals is not None:
        if len(residuals) != len(worker_grads):
            raise ValueError("need one residual per worker")
        pipe.residuals = residuals
    result = pipe.run_round(worker_grads, round_index)
    if residuals is not None:
        residuals[:] = pipe.residuals
    return result


def run_topk_round(worker_grads, k, seeds, *, round_index=0, residuals=None):
    return _one_shot(TopKConfig(k), worker_grads, seeds, round_index, residuals)


def run_chunked_topk_round(worker_grads, chunk_size, chunks_selected, seeds, *, round_index=0, residuals=None,
                           permute=False):
    return _one_shot(ChunkedTopKConfig(chunk_size, chunks_selected, permute), worker_grads, seeds, round_index,
                     residuals)


def run_rotated_quant_round(worker_grads, config: RotatedQuantConfig, seeds, *, round_index=0, residuals=None):
    return _one_shot(config, worker_grads, seeds, round_index, residuals)


def run_powersgd_round(worker_grads, config: PowerSgdConfig, seeds, *, round_index=0, residuals=None):
    return _one_shot(config, worker_grads, seeds, round_index, residuals)


def run_dense_round(worker_grads, bits, seeds, *, round_index=0):
    return _one_shot(DenseConfig(bits), worker_grads, seeds, round_index, None, error_feedback=False)
