"""Scheme engines: the device-side cores of GradientPipeline.run_round.

One engine per reference scheme core (pipelines.py:201-393).  An engine owns its device
buffers (allocated once per pipeline) and issues the native kernels on the current
stream; it never synchronises.  `run` returns (estimate [d] device tensor, input_bits,
RoundStats) and charges the round's closed-form traffic to the ledger.
"""

from __future__ import annotations

import ctypes
import math

import torch

from . import _native
from .configs import ChunkedTopKConfig, DenseConfig, PowerSgdConfig, RotatedQuantConfig, TopKConfig
from .ledger import OverflowStats, TrafficLedger
from .vectors import SeedSpec, next_pow2


def _sp() -> int:
    return torch.cuda.current_stream().cuda_stream


def _ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


class RoundStats:
    """Device-resident per-round diagnostics, copied to the host on first access."""

    def __init__(self, counters: torch.Tensor | None, nmse_acc: torch.Tensor | None, finalize):
        self._counters = counters
        self._nmse = nmse_acc
        self._finalize = finalize
        self._host = None

    def _load(self):
        if self._host is None:
            c = self._counters.cpu().tolist() if self._counters is not None else None
            m = self._nmse.cpu().tolist() if self._nmse is not None else None
            self._host = self._finalize(c, m)
        return self._host

    def nmse(self) -> float:
        return self._load()["nmse"]

    def overflow(self) -> OverflowStats:
        return self._load()["overflow"]

    def range_clips(self) -> int:
        return self._load()["range_clips"]


def nmse_from(acc) -> float:
    """metrics.py:32-37 from the device accumulators (sum err^2, sum ref^2)."""
    if acc is None:
        return float("nan")
    num, den = acc
    if den == 0.0:
        return 0.0 if num == 0.0 else math.inf
    return num / den


class Engine:
    def __init__(self, n: int, dim: int, seeds: SeedSpec, device):
        self.n, self.dim, self.seeds, self.device = n, dim, seeds, device
        self.capture = False       # keep intermediates for parity tests
        self.last = {}
        self.kernel_events = None  # list -> (start, end) CUDA events around the dominant kernel
        self.launches = 0          # native kernel launches issued (for the bench's gpu_launches)

    def _ev(self):
        if self.kernel_events is None:
            return None
        e = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
        self.kernel_events.append(e)
        return e

    def warm_q(self):
        return None

    def _nmse(self, grads, res, est, acc):
        _native.call("gc_nmse_accumulate", self.n, self.dim, grads.data_ptr(), _ptr(res) or None,
                     grads.stride(0), est.data_ptr(), acc.data_ptr(), _sp())


# ---------------------------------------------------------------------------------- THC
class ThcEngine(Engine):
    """pipelines.py:260-322 (RotatedQuantConfig)."""

    TILE = 1024

    def __init__(self, cfg: RotatedQuantConfig, n, dim, seeds, device, fused=True):
        super().__init__(n, dim, seeds, device)
        self.cfg = cfg
        P = next_pow2(dim)
        depth = min(P.bit_length() - 1, cfg.rotation_block.bit_length() - 1)   # transforms.py:78
        B = 1 << depth
        self.P, self.B = P, B
        self.geom = _native.ThcGeom(dim, P, B, cfg.quant_bits, cfg.wire_bits, float(B) ** -0.5)
        self.active = int(_native.lib().gc_thc_active_len(ctypes.byref(self.geom)))
        self.nb = self.active // B
        self.fused = bool(fused) and n <= 16 and P >= self.TILE and 32 <= B <= self.TILE
        sign_count = self.active
        if self.fused:
            sign_count = -(-self.active // self.TILE) * self.TILE
        self.sign_count = sign_count
        i32 = dict(dtype=torch.int32, device=device)
        self.signs = torch.empty(-(-sign_count // 32), **i32)
        self.est = torch.empty(dim, dtype=torch.float32, device=device)
        self.counters = torch.zeros(4, dtype=torch.int64, device=device)
        self.nmse_acc = torch.zeros(2, dtype=torch.float64, device=device)
        self.sum_bytes = 1 if cfg.wire_bits <= 8 else (2 if cfg.wire_bits <= 16 else 4)
        self.ring_blk = -(-P // n)
        self._generic = None
        ws = int(_native.lib().gc_thc_workspace_bytes(ctypes.byref(self.geom), n))
        self.workspace = torch.empty(max(ws, 1), dtype=torch.uint8, device=device) if ws else None

    def _generic_buffers(self):
        if self._generic is None:
            n, dev = self.n, self.device
            sdt = {1: torch.int8, 2: torch.int16, 4: torch.int32}[self.sum_bytes]
            self._generic = dict(
                x_rot=torch.empty(n, self.active, dtype=torch.float32, device=dev),
                ranges=torch.empty(n, self.nb, 2, dtype=torch.float32, device=dev),
                shared=torch.empty(self.nb, 2, dtype=torch.float32, device=dev),
                codes=torch.empty(n, self.active, dtype=torch.int8, device=dev),
                sums=torch.empty(self.active, dtype=sdt, device=dev),
            )
        return self._generic

    def coin_streams(self, round_index):
        arr = (_native.Pcg64 * self.n)()
        for w in range(self.n):
            arr[w] = self.seeds.pcg("stochastic-round", round_index, w)   # pipelines.py:293
        return arr

    def run(self, grads, res, round_index, ledger: TrafficLedger, nmse=True):
        n, cfg = self.n, self.cfg
        sp = _sp()
        rot = self.seeds.pcg("rotation-signs", round_index)                  # transforms.py:80-82
        _native.call("gc_thc_signs", ctypes.byref(rot), self.sign_count, self.signs.data_ptr(), sp)
        coins = self.coin_streams(round_index)
        # fresh per-round outputs: a RoundResult must stay valid after later rounds
        self.est = torch.empty(self.dim, dtype=torch.float32, device=self.device)
        self.counters = torch.zeros(4, dtype=torch.int64, device=self.device)
        self.nmse_acc = torch.zeros(2, dtype=torch.float64, device=self.device)
        g_ld = grads.stride(0)
        if self.fused:
            codes = None
            if self.capture:
                codes = torch.zeros(n, self.active, dtype=torch.int8, device=self.device)
                self.last = {"codes": codes, "signs": self.signs}
            ev = self._ev()
            if ev:
                ev[0].record()
            _native.call("gc_thc_round_fused", ctypes.byref(self.geom), n, grads.data_ptr(), _ptr(res),
                         g_ld, self.signs.data_ptr(), coins, self.est.data_ptr(), _ptr(codes),
                         self.counters.data_ptr(), self.nmse_acc.data_ptr() if nmse else None, sp)
            if ev:
                ev[1].record()
            self.launches += 2
        else:
            b = self._generic_buffers()
            ws = _ptr(self.workspace)
            _native.call("gc_thc_rotate", ctypes.byref(self.geom), n, grads.data_ptr(), _ptr(res), g_ld,
                         self.signs.data_ptr(), b["x_rot"].data_ptr(), b["ranges"].data_ptr(), ws, sp)
            _native.call("gc_range_consensus", n, self.nb, b["ranges"].data_ptr(), b["shared"].data_ptr(), sp)
            _native.call("gc_thc_quantize", ctypes.byref(self.geom), n, b["x_rot"].data_ptr(),
                         b["shared"].data_ptr(), coins, b["codes"].data_ptr(), self.counters.data_ptr(), sp)
            if n > 1:
                _native.call("gc_sat_fold", n, self.active, b["codes"].data_ptr(), self.active, 0, self.ring_blk,
                             cfg.wire_bits, b["sums"].data_ptr(), self.counters[3:].data_ptr(), sp)
                sums, sbytes = b["sums"], self.sum_bytes
            else:
                sums, sbytes = b["codes"][0], 1
            _native.call("gc_thc_decode_estimate", ctypes.byref(self.geom), n, sums.data_ptr(), sbytes,
                         b["shared"].data_ptr(), self.signs.data_ptr(), self.est.data_ptr(), ws, sp)
            if nmse:
                self._nmse(grads, res, self.est, self.nmse_acc)
            if res is not None:
                _native.call("gc_thc_decode_ef", ctypes.byref(self.geom), n, b["codes"].data_ptr(),
                             b["shared"].data_ptr(), self.signs.data_ptr(), grads.data_ptr(), res.data_ptr(),
                             res.stride(0), ws, sp)
            if self.capture:
                self.last = dict(b, signs=self.signs)
            self.launches += 5 + (n > 1) + bool(nmse) + (res is not None)
        # ledger + bits (pipelines.py:271-305, 321)
        num_blocks = self.P // self.B
        ledger.charge_ring("range-consensus", n, num_blocks, 32)
        ledger.charge_ring("range-consensus", n, num_blocks, 32)
        ledger.charge_ring("code-aggregate", n, self.P, cfg.wire_bits)
        input_bits = float(cfg.wire_bits * self.P + 64 * num_blocks)
        total = n * self.P
        total_adds = (n - 1) * self.ring_blk * n if n > 1 else 0

        def finalize(c, m):
            s1, s2 = c[1], c[2]
            var = (total * s2 - s1 * s1) / (total * total)
            sigma = math.sqrt(max(var, 0.0))
            return {"nmse": nmse_from(m), "range_clips": int(c[0]),
                    "overflow": OverflowStats(int(c[3]), int(total_adds), float(sigma))}

        return self.est, input_bits, RoundStats(self.counters, self.nmse_acc if nmse else None, finalize)


def _simple_stats(nmse_acc):
    return RoundStats(None, nmse_acc, lambda c, m: {"nmse": nmse_from(m), "range_clips": 0,
                                                    "overflow": OverflowStats()})


# -------------------------------------------------------------------------------- dense
class DenseEngine(Engine):
    """pipelines.py:370-393: FP16 bar (fp16 inputs, fp16 wire per hop) or exact FP32 ring; no EF."""

    def __init__(self, cfg: DenseConfig, n, dim, seeds, device):
        super().__init__(n, dim, seeds, device)
        self.bits = cfg.bits

    def run(self, grads, res, round_index, ledger, nmse=True):
        n, d = self.n, self.dim
        est = torch.empty(d, dtype=torch.float32, device=self.device)
        wire16 = 1 if self.bits == 16 else 0
        ev = self._ev()
        if ev:
            ev[0].record()
        _native.call("gc_float_fold", n, d, grads.data_ptr(), grads.stride(0), 0, -(-d // n), wire16, wire16, n,
                     est.data_ptr(), _sp())
        if ev:
            ev[1].record()
        self.launches += 1
        acc = None
        if nmse:
            acc = torch.zeros(2, dtype=torch.float64, device=self.device)
            self._nmse(grads, None, est, acc)
            self.launches += 1
        ledger.charge_ring("dense", n, d, self.bits)
        return est, float(self.bits) * d, _simple_stats(acc)


# -------------------------------------------------------------------------------- TopK
class TopKEngine(Engine):
    """pipelines.py:201-211 (TopKConfig)."""

    def __init__(self, cfg: TopKConfig, n, dim, seeds, device):
        super().__init__(n, dim, seeds, device)
        self.k = cfg.k
        ws = int(_native.lib().gc_topk_workspace_bytes(n, dim))
        self.ws = torch.empty(ws, dtype=torch.uint8, device=device)

    def run(self, grads, res, round_index, ledger, nmse=True):
        n, d, k = self.n, self.dim, self.k
        sp = _sp()
        idx = torch.empty(n, k, dtype=torch.int32, device=self.device)
        val = torch.empty(n, k, dtype=torch.float32, device=self.device)
        ev = self._ev()
        if ev:
            ev[0].record()
        # selection fused with ef_apply: the corrected vectors land in `res` (EF on)
        _native.call("gc_topk_select", n, d, None, grads.stride(0), k, grads.data_ptr(), _ptr(res),
                     idx.data_ptr(), val.data_ptr(), 1, self.ws.data_ptr(), sp)
        if ev:
            ev[1].record()
        est = torch.empty(d, dtype=torch.float32, device=self.device)
        _native.call("gc_sparse_accumulate", n, k, idx.data_ptr(), val.data_ptr(), d, est.data_ptr(), sp)
        _native.call("gc_scale_div", d, est.data_ptr(), n, est.data_ptr(), sp)
        self.launches += 10 + n
        acc = None
        corrected = res if res is not None else grads
        if nmse:
            acc = torch.zeros(2, dtype=torch.float64, device=self.device)
            self._nmse(corrected, None, est, acc)
            self.launches += 1
        if res is not None:
            _native.call("gc_sparse_ef_update", n, k, idx.data_ptr(), val.data_ptr(), res.data_ptr(),
                         res.stride(0), sp)
            self.launches += 1
        if self.capture:
            self.last = {"idx": idx, "val": val}
        ledger.charge_gather("sparse-gather", [48 * k] * n)
        return est, float(48 * k), _simple_stats(acc)


def make_engine(cfg, n, dim, seeds, device, fused=True) -> Engine:
    if isinstance(cfg, RotatedQuantConfig):
        return ThcEngine(cfg, n, dim, seeds, device, fused)
    if isinstance(cfg, DenseConfig):
        return DenseEngine(cfg, n, dim, seeds, device)
    if isinstance(cfg, TopKConfig):
        return TopKEngine(cfg, n, dim, seeds, device)
    raise NotImplementedError(f"{type(cfg).__name__} engine not built yet")
