"""Per-tensor pipelines over a flat gradient ("chunked" schemes).

A model's gradient is a list of tensors; running the reference on it tensor by tensor means one
GradientPipeline (pipelines.py:97-393) per tensor with the same config and SeedSpec, each with
its own EF residual and warm-start state.  TensorListPipeline does exactly that over a flat
[n, D] buffer (D = sum of the tensor sizes, each tensor a contiguous slice), and for PowerSGD runs
it B200-first: tensors below bypass_below are folded together in one dense-fp32 launch, and the
compressed tensors are batched by length (same rows x cols), so GPT-2-medium's 122 compressed
matrices become 5 shape groups of batched kernels instead of 122 pipelines.
"""

from __future__ import annotations

from collections import OrderedDict

import numpy as np
import torch

from . import _native
from .configs import PowerSgdConfig, scheme_label
from .ledger import TrafficLedger, WorkerGroup
from .pipeline import RoundResult
from .schemes import PowerSgdGroup, _simple_stats, make_engine, seed_q_groups, umma_unaligned
from .vectors import SeedSpec


def _sp() -> int:
    return _native.current_stream_handle()


def gpt2_medium_sizes() -> list[int]:
    """Parameter sizes of GPT-2-medium (355M): 292 tensors, 354,823,168 elements."""
    h, v, ctx, layers = 1024, 50257, 1024, 24
    sizes = [v * h, ctx * h]
    for _ in range(layers):
        sizes += [h, h, h * 3 * h, 3 * h, h * h, h, h, h, h * 4 * h, 4 * h, 4 * h * h, h]
    sizes += [h, h]
    return sizes


class TensorListPipeline:
    """One reference pipeline per tensor of a flat gradient, n workers simulated on one GPU."""

    def __init__(self, config, num_workers: int, sizes, seeds: SeedSpec, error_feedback: bool | None = None, *,
                 device=None, validate: bool = True, compute_nmse: bool = True):
        if num_workers < 1 or not sizes or min(sizes) < 1:
            raise ValueError("need workers >= 1 and positive tensor sizes")
        self.config = config
        self.scheme = scheme_label(config)
        self.group = WorkerGroup(num_workers)
        self.sizes = [int(x) for x in sizes]
        self.offsets = np.concatenate([[0], np.cumsum(self.sizes)[:-1]]).astype(np.int64)
        self.dim = int(sum(self.sizes))
        self.seeds = seeds
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        from .configs import DenseConfig
        if isinstance(config, DenseConfig):
            if error_feedback:
                raise ValueError("dense baselines do not carry error feedback")
            error_feedback = False
        elif error_feedback is None:
            error_feedback = True
        self.error_feedback = bool(error_feedback)
        self.validate = validate
        self.compute_nmse = compute_nmse
        n, D = num_workers, self.dim
        self._res = torch.zeros(n, D, dtype=torch.float32, device=self.device) if self.error_feedback else None
        self._stage = None
        self._fold_out = {}
        self.batched = isinstance(config, PowerSgdConfig)
        self.launches = 0
        if self.batched:
            self._build_psgd()
        else:   # any other scheme: one engine per tensor on strided views of the flat buffers
            self.engines = [make_engine(config, n, s, seeds, self.device) for s in self.sizes]

    # ------------------------------------------------------------------ PowerSGD layout
    def _build_psgd(self):
        cfg, n, D = self.config, self.group.size, self.dim
        dev = self.device
        byp = [t for t, s in enumerate(self.sizes) if s < cfg.bypass_below]
        self.bypass = byp
        self.seg_off = torch.tensor([int(self.offsets[t]) for t in byp], dtype=torch.int64, device=dev)
        self.seg_len = torch.tensor([self.sizes[t] for t in byp], dtype=torch.int64, device=dev)
        groups = OrderedDict()
        for t, s in enumerate(self.sizes):
            if s >= cfg.bypass_below:
                groups.setdefault(s, []).append(t)
        self.groups = []
        # smallest batches first: the round ends with the longest decode, behind which the host
        # reads the warm-Q Gram events and queues the next round (groups are independent)
        for s, ts in sorted(groups.items(), key=lambda kv: kv[0] * len(kv[1])):
            rows = [w * D + int(self.offsets[t]) for t in ts for w in range(n)]
            ro = torch.tensor(rows, dtype=torch.int64, device=dev)
            eo = torch.tensor([int(self.offsets[t]) for t in ts], dtype=torch.int64, device=dev)
            grp = PowerSgdGroup(cfg, n, n, s, len(ts), self.seeds, dev, row_offsets=ro, est_offsets=eo, ld=D,
                                host_offsets=[int(self.offsets[t]) for t in ts])
            grp.tensor_ids = ts
            grp.vec = grp.cols % 4 == 0 and all(x % 4 == 0 for x in rows) and D % 4 == 0
            self.groups.append(grp)

    def _fold(self, kind, x, m):
        n = self.group.size
        if n == 1:   # one worker: the ring sum is the row itself
            return x.reshape(x.shape[0], m)
        key = (kind, x.data_ptr(), x.shape[0] // n, m)   # one reused output per group input buffer
        out = self._fold_out.get(key)
        if out is None:
            out = self._fold_out[key] = torch.empty(x.shape[0] // n, m, dtype=torch.float32, device=self.device)
        _native.call("gc_float_fold_batched", x.shape[0] // n, n, m, x.data_ptr(), m, n * m, 0, 0, 0, out.data_ptr(),
                     m, _sp())
        return out

    # ------------------------------------------------------------------ state
    @property
    def residuals(self):
        if self._res is None:
            return None
        self._sync_residuals()
        h = self._res.cpu().numpy()
        return [h[i].copy() for i in range(self.group.size)]

    @property
    def residuals_tensor(self):
        if self._res is not None:
            self._sync_residuals()
        return self._res

    def _sync_residuals(self):
        """Materialise the EF updates the PowerSGD groups deferred into their next P = M Q pass."""
        for grp in getattr(self, "groups", []):
            grp.materialize(self._res.data_ptr())

    def warm_q(self, tensor: int):
        """The warm-start Q of one tensor (pipelines.py:366), or None."""
        if not self.batched:
            wq = self.engines[tensor].warm_q()
            return None if wq is None else wq.cpu().numpy()
        for grp in self.groups:
            if tensor in grp.tensor_ids and grp.warm is not None:
                return grp.warm[grp.tensor_ids.index(tensor)].cpu().numpy()
        return None

    # ------------------------------------------------------------------ round
    def _checked(self, worker_grads) -> torch.Tensor:
        n, D = self.group.size, self.dim
        if (torch.is_tensor(worker_grads) and worker_grads.dim() == 2 and tuple(worker_grads.shape) == (n, D)
                and worker_grads.is_cuda and worker_grads.is_contiguous() and worker_grads.dtype == torch.float32):
            g = worker_grads
        else:
            if len(worker_grads) != n:
                raise ValueError("need exactly one gradient per worker")
            if self._stage is None:
                self._stage = torch.empty(n, D, dtype=torch.float32, device=self.device)
            for i, x in enumerate(worker_grads):
                t = x if torch.is_tensor(x) else torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32))
                if t.numel() != D:
                    raise ValueError("gradient length does not match the sum of the tensor sizes")
                self._stage[i].copy_(t.reshape(-1), non_blocking=True)
            g = self._stage
        if self.validate:
            bad = torch.zeros(1, dtype=torch.int64, device=self.device)
            _native.call("gc_check_finite", n, g.data_ptr(), g.stride(0), D, bad.data_ptr(), _sp())
            if int(bad.item()):
                raise ValueError("gradients must be finite")
        return g

    def run_round(self, worker_grads, round_index: int) -> RoundResult:
        g = self._checked(worker_grads)
        ledger = TrafficLedger()
        n, D = self.group.size, self.dim
        est = torch.empty(D, dtype=torch.float32, device=self.device)
        acc = torch.zeros(2, dtype=torch.float64, device=self.device) if self.compute_nmse else None
        if not self.batched:
            bits = 0.0
            ref = None
            if acc is not None:   # nmse target: fp64 mean of the corrected vectors, before EF updates
                c = g.double()
                if self._res is not None:
                    c += self._res.double()
                ref = c.mean(0)
                del c
            for t, eng in enumerate(self.engines):
                off, s = int(self.offsets[t]), self.sizes[t]
                gv = g[:, off:off + s]
                rv = self._res[:, off:off + s] if self._res is not None else None
                e, b, _ = eng.run(gv, rv, round_index, ledger, nmse=False)
                est[off:off + s].copy_(e)
                bits += b
            self.launches += sum(e.launches for e in self.engines)
            if ref is not None:
                e = est.double() - ref
                acc = torch.stack([torch.dot(e, e), torch.dot(ref, ref)])
            return RoundResult(self.scheme, round_index, est, D, ledger, bits, _simple_stats(acc))

        sp = _sp()
        res = self._res
        # seed matrices of every group first: their rank checks read a few bytes back to the host,
        # so doing them before the heavy kernels keeps the device queue free of bubbles
        qs = seed_q_groups(self.groups, round_index)
        # Without nmse, ef_apply rides in the first pass over each tensor (P = M Q for the
        # compressed ones, the bypass fold for the small ones) and the residual update in the
        # decode pass.  The nmse diagnostic needs every corrected vector before any residual
        # changes, so then ef_apply runs as one pass up front and the EF updates come last.
        fuse_ef = res is not None and acc is None
        if res is not None and not fuse_ef:
            self._sync_residuals()
        if res is not None and not fuse_ef:   # corrected vectors kept in r until the EF updates
            _native.call("gc_ef_apply", n, D, g.data_ptr(), res.data_ptr(), g.stride(0), res.data_ptr(),
                         res.stride(0), sp)
        c = res if res is not None else g
        bits = 0.0
        # dense-fp32 bypass of the small tensors (pipelines.py:326-336), one launch
        if self.bypass:
            if fuse_ef:   # corrected = g + r formed in the fold; own == corrected, so r leaves as 0
                _native.call("gc_segment_ef_fold", n, len(self.bypass), self.seg_off.data_ptr(),
                             self.seg_len.data_ptr(), g.data_ptr(), res.data_ptr(), g.stride(0), est.data_ptr(), sp)
            else:
                _native.call("gc_segment_fold_ef", n, len(self.bypass), self.seg_off.data_ptr(),
                             self.seg_len.data_ptr(), c.data_ptr(), None, c.stride(0), est.data_ptr(), sp)
            ledger.charge_rings("dense-bypass", n, [self.sizes[t] for t in self.bypass], 32)
            bits += 32.0 * sum(self.sizes[t] for t in self.bypass)
        # every group up to its decode first, then all decodes: the next round's rank check waits on
        # the last group's warm-Q Gram while all decodes are still queued (no device bubble)
        finish = []
        for grp, q in zip(self.groups, qs):
            grp.set_ld(c.stride(0), grp.vec and c.data_ptr() % 16 == 0 and est.data_ptr() % 16 == 0
                       and g.data_ptr() % 16 == 0 and g.stride(0) == c.stride(0))
            if fuse_ef and (grp.batch.rows_aligned or umma_unaligned()):   # ef_apply inside the tcgen05 P = M Q
                fin = grp.run(c.data_ptr(), res.data_ptr(), est.data_ptr(), round_index, grads_ptr=g.data_ptr(),
                              vec=bool(grp.batch.rows_aligned), fold=self._fold, q=q, ef_resid_ptr=res.data_ptr(),
                              defer_decode=True)
            elif fuse_ef:   # unaligned rows: ef_apply on the group's tensors, then the plain passes
                grp.materialize(res.data_ptr())
                for t in grp.tensor_ids:
                    off = int(self.offsets[t])
                    _native.call("gc_ef_apply", n, self.sizes[t], g.data_ptr() + 4 * off, res.data_ptr() + 4 * off,
                                 g.stride(0), res.data_ptr() + 4 * off, res.stride(0), sp)
                fin = grp.run(c.data_ptr(), res.data_ptr(), est.data_ptr(), round_index, vec=False, fold=self._fold,
                              q=q, defer_decode=True)
            else:
                fin = grp.run(c.data_ptr(), None, est.data_ptr(), round_index, vec=bool(grp.batch.rows_aligned),
                              fold=self._fold, q=q, defer_decode=True)
            finish.append(fin)
        for grp, fin in zip(self.groups, finish):
            fin()
            grp.saved = dict(grp.last)
        for grp in self.groups:
            T = len(grp.tensor_ids)
            ledger.charge_ring("left-factor", n, grp.rows * grp.rank, 32, times=T)
            ledger.charge_ring("right-factor", n, grp.cols * grp.rank, 32, times=T)
            bits += 32.0 * grp.rank * (grp.rows + grp.cols) * T
        if acc is not None:
            _native.call("gc_nmse_accumulate", n, D, c.data_ptr(), None, c.stride(0), est.data_ptr(), acc.data_ptr(), sp)
        if res is not None and not fuse_ef:
            if self.bypass:   # own == corrected: residual 0
                _native.call("gc_segment_fold_ef", n, len(self.bypass), self.seg_off.data_ptr(),
                             self.seg_len.data_ptr(), c.data_ptr(), res.data_ptr(), c.stride(0), est.data_ptr(), sp)
            for grp in ([] if fuse_ef else self.groups):
                grp.saved["decode"](res.data_ptr(), None)   # EF update of the group (rank chunk by chunk)
        self.launches += 2 + len(self.groups) * 11
        return RoundResult(self.scheme, round_index, est, D, ledger, bits, _simple_stats(acc))
