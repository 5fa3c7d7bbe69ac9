"""Scheme engines: the device-side cores of GradientPipeline.run_round.

One engine per reference scheme core (pipelines.py:201-393).  An engine owns its device
buffers (allocated once per pipeline) and issues the native kernels on the current
stream; it never synchronises.  `run` returns (estimate [d] device tensor, input_bits,
RoundStats) and charges the round's closed-form traffic to the ledger.
"""

from __future__ import annotations

import ctypes
import os
import math

import torch

from . import _native
from .configs import (ChunkedTopKConfig, DenseConfig, PowerSgdConfig, RotatedQuantConfig, TopKConfig,
                      matrix_shape_for)
from .ledger import OverflowStats, TrafficLedger
from .vectors import SeedSpec, next_pow2


def _sp() -> int:
    return _native.current_stream_handle()


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

    def sync_residuals(self, res):
        """Materialise any error-feedback update the engine deferred into the next round (PowerSGD)."""

    def drop_deferred(self):
        """Forget a deferred EF update (the caller replaced the residual buffer)."""

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
        return self._round_meta(ledger, nmse)


    def run_streamed(self, host_rows, stage, res_in, res_out, round_index, ledger: TrafficLedger, nmse=True,
                     segments=None):
        """Host-fed fused round (gc_thc_round_fused_range): segment s of every worker's gradient is
        copied host -> device on one stream while segment s-1 is validated and runs its tiles on the
        compute stream and segment s-2's estimate is copied device -> host on a third, so PCIe in,
        the kernel and PCIe out overlap.  The residual is read from res_in and written to res_out;
        the caller keeps res_in until the round validated (pipelines.py:184-197 raises first).
        Returns (estimate_dev, estimate_host, input_bits, stats, nonfinite_count_dev)."""
        n, d, T = self.n, self.dim, -(-self.active // self.TILE)
        cur = torch.cuda.current_stream()
        if getattr(self, "_h2d", None) is None:
            self._h2d, self._d2h = torch.cuda.Stream(self.device), torch.cuda.Stream(self.device)
        h2d, d2h = self._h2d, self._d2h
        sp = cur.cuda_stream
        rot = self.seeds.pcg("rotation-signs", round_index)
        _native.call("gc_thc_signs", ctypes.byref(rot), self.sign_count, self.signs.data_ptr(), sp)
        coins = self.coin_streams(round_index)
        self.est = torch.empty(d, dtype=torch.float32, device=self.device)
        est_host = torch.empty(d, dtype=torch.float32, pin_memory=True)
        self.counters = torch.zeros(4, dtype=torch.int64, device=self.device)
        self.nmse_acc = torch.zeros(2, dtype=torch.float64, device=self.device)
        bad = torch.zeros(1, dtype=torch.int64, device=self.device)
        h2d.wait_stream(cur)   # the stage buffer may still be read by the previous round
        if segments is None:
            # measured on B200: one strided copy per segment ([n, d] block) overlaps best at 16
            # segments; per-row copies pay a launch per row and segment, so 8 fewer-larger ones win
            env = os.environ.get("GC_THC_SEGMENTS")
            segments = int(env) if env else (16 if torch.is_tensor(host_rows) else 8)
        segments = max(1, min(segments, T))
        ld = stage.stride(0)
        ev = self._ev()
        for s in range(segments):
            tb, te = T * s // segments, T * (s + 1) // segments
            a, b = tb * self.TILE, min(te * self.TILE, d)
            if a >= b:
                continue
            with torch.cuda.stream(h2d):
                if torch.is_tensor(host_rows):   # [n, d] host block: one strided copy per segment
                    _native.call("gc_copy_rows_async", stage[0, a:].data_ptr(), stage.stride(0) * 4,
                                 host_rows[0, a:].data_ptr(), host_rows.stride(0) * 4, (b - a) * 4, n,
                                 h2d.cuda_stream)
                else:
                    for w in range(n):
                        stage[w, a:b].copy_(host_rows[w][a:b], non_blocking=True)
            cur.wait_stream(h2d)
            if ev and s == 0:
                ev[0].record()
            _native.call("gc_check_finite", n, stage[:, a:].data_ptr(), ld, b - a, bad.data_ptr(), sp)
            _native.call("gc_thc_round_fused_range", ctypes.byref(self.geom), n, stage.data_ptr(), _ptr(res_in),
                         _ptr(res_out), ld, tb, te, self.signs.data_ptr(), coins, self.est.data_ptr(), None,
                         self.counters.data_ptr(), self.nmse_acc.data_ptr() if nmse else None, sp)
            if ev and s == segments - 1:
                ev[1].record()
            d2h.wait_stream(cur)
            with torch.cuda.stream(d2h):
                est_host[a:b].copy_(self.est[a:b], non_blocking=True)
            self.launches += 2
        cur.wait_stream(d2h)
        self.est.record_stream(d2h)
        stage.record_stream(h2d)
        est, bits, stats = self._round_meta(ledger, nmse)
        return est, est_host, bits, stats, bad

    def _round_meta(self, ledger, nmse):
        n, cfg = self.n, self.cfg
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
        self.ws = torch.zeros(ws, dtype=torch.uint8, device=device)   # zeroed: no threshold hint yet
        mws = int(_native.lib().gc_sparse_mean_workspace_bytes(n, dim))
        self.mean_ws = torch.empty(mws, dtype=torch.uint8, device=device)

    def run(self, grads, res, round_index, ledger, nmse=True):
        n, d, k = self.n, self.dim, self.k
        sp = _sp()
        idx = torch.empty(n, k, dtype=torch.int32, device=self.device)
        val = torch.empty(n, k, dtype=torch.float32, device=self.device)
        ev = self._ev()
        if ev:
            ev[0].record()
        # selection fused with ef_apply: the corrected vectors land in `res` (EF on); without the
        # nmse diagnostic (which reads the corrected vectors) ef_update is fused in as well
        fuse_ef = res is not None and not nmse
        flags = _native.TOPK_FP16_VALUES | (_native.TOPK_EF_UPDATE if fuse_ef else 0)
        _native.call("gc_topk_select", n, d, None, grads.stride(0), k, grads.data_ptr(), _ptr(res),
                     idx.data_ptr(), val.data_ptr(), flags, self.ws.data_ptr(), sp)
        if ev:
            ev[1].record()
        est = torch.empty(d, dtype=torch.float32, device=self.device)
        _native.call("gc_sparse_mean", n, k, idx.data_ptr(), val.data_ptr(), d, n, est.data_ptr(),
                     self.mean_ws.data_ptr(), sp)
        self.launches += 10 + n
        acc = None
        corrected = res if res is not None else grads
        if nmse:
            acc = torch.zeros(2, dtype=torch.float64, device=self.device)
            self._nmse(corrected, None, est, acc)
            self.launches += 1
        if res is not None and not fuse_ef:
            _native.call("gc_sparse_ef_update", n, k, idx.data_ptr(), val.data_ptr(), res.data_ptr(),
                         res.stride(0), sp)
            self.launches += 1
        if self.capture:
            self.last = {"idx": idx, "val": val}
        ledger.charge_gather("sparse-gather", [48 * k] * n)
        return est, float(48 * k), _simple_stats(acc)


# ------------------------------------------------------------------------- TopK-Chunked
class ChunkedEngine(Engine):
    """pipelines.py:213-258 (ChunkedTopKConfig), incl. the permutation ablation."""

    def __init__(self, cfg: ChunkedTopKConfig, n, dim, seeds, device):
        super().__init__(n, dim, seeds, device)
        self.cfg = cfg
        self.C = cfg.chunk_size
        self.J = cfg.chunks_selected
        self.nc = -(-dim // self.C)
        ws = int(_native.lib().gc_topk_workspace_bytes(1, self.nc))
        self.ws = torch.zeros(ws, dtype=torch.uint8, device=device)   # zeroed: no threshold hint yet
        self._work = None

    def _perm(self, round_index):
        """coordinate_permutation (transforms.py:129-133): host numpy draw, uploaded."""
        p = self.seeds.rng("coordinate-permutation", round_index).permutation(self.dim)
        return torch.from_numpy(p.astype("int64")).to(self.device, non_blocking=True)

    def run(self, grads, res, round_index, ledger, nmse=True):
        n, d, C, J, nc = self.n, self.dim, self.C, self.J, self.nc
        sp = _sp()
        dev = self.device
        perm = self._perm(round_index) if self.cfg.permute else None
        pp = _ptr(perm)
        fuse = perm is None and C % 8 == 0 and C <= 128 and (res is None or res.stride(0) == grads.stride(0))
        if res is not None and not fuse:   # corrected = g + r, kept in r until the EF update
            _native.call("gc_ef_apply", n, d, grads.data_ptr(), res.data_ptr(), grads.stride(0), res.data_ptr(),
                         res.stride(0), sp)
        work = res if res is not None else grads
        norms = torch.empty(n, nc, dtype=torch.float32, device=dev)
        ev = self._ev()
        if ev:
            ev[0].record()
        if fuse:   # ef_apply fused into the chunk energies
            _native.call("gc_chunk_norms_ef", n, d, C, grads.data_ptr(), _ptr(res), grads.stride(0), norms.data_ptr(),
                         sp)
        else:
            _native.call("gc_chunk_norms", n, d, C, work.data_ptr(), work.stride(0), pp, norms.data_ptr(), sp)
        energy = torch.empty(nc, dtype=torch.float32, device=dev)
        _native.call("gc_float_fold", n, nc, norms.data_ptr(), nc, 0, -(-nc // n), 1, 0, 0, energy.data_ptr(), sp)
        sel = torch.empty(J, dtype=torch.int32, device=dev)
        _native.call("gc_topk_select", 1, nc, energy.data_ptr(), nc, J, None, None, sel.data_ptr(), None, 0,
                     self.ws.data_ptr(), sp)
        L = J * C
        packs = torch.empty(n, L, dtype=torch.float32, device=dev)
        _native.call("gc_chunk_pack", n, d, C, J, sel.data_ptr(), work.data_ptr(), work.stride(0), pp,
                     packs.data_ptr(), sp)
        summed = torch.empty(L, dtype=torch.float32, device=dev)
        _native.call("gc_float_fold", n, L, packs.data_ptr(), L, 0, -(-L // n), 1, 0, 0, summed.data_ptr(), sp)
        est = torch.empty(d, dtype=torch.float32, device=dev)
        _native.call("gc_chunk_scatter", d, C, J, sel.data_ptr(), summed.data_ptr(), n, pp, est.data_ptr(), sp)
        if ev:
            ev[1].record()
        self.launches += 14 + (res is not None)
        acc = None
        if nmse:
            acc = torch.zeros(2, dtype=torch.float64, device=dev)
            self._nmse(work, None, est, acc)
            self.launches += 1
        if res is not None:
            _native.call("gc_chunk_ef_update", n, d, C, J, sel.data_ptr(), packs.data_ptr(), pp, res.data_ptr(),
                         res.stride(0), sp)
            self.launches += 1
        if self.capture:
            self.last = {"norms": norms, "energy": energy, "selected": sel, "summed": summed}
        ledger.charge_ring("norm-consensus", n, nc, 16)
        ledger.charge_ring("chunk-aggregate", n, L, 16)
        return est, 16.0 * (nc + J * C), _simple_stats(acc)


# ----------------------------------------------------------------------------- PowerSGD
def _rank_ok_many(groups, host_grams, q_devs):
    """PowerSgdGroup._rank_ok_host for several groups of the same rank with one eigvalsh call:
    per tensor np.linalg.matrix_rank(q) == rank (compressors.py:599) from the fp64 Gram eigenvalues,
    the exact numpy call on a host copy near numpy's tolerance."""
    import numpy as np
    if not groups:
        return []
    r = groups[0].rank
    sig = np.sqrt(np.clip(np.linalg.eigvalsh(np.concatenate(host_grams).reshape(-1, r, r)), 0.0, None))
    width = np.concatenate([np.full(hg.shape[0], max(grp.cols, r), dtype=np.float64)
                            for grp, hg in zip(groups, host_grams)])
    tol = sig.max(axis=1) * width * np.finfo(np.float32).eps
    clear = np.all((sig > 2 * tol[:, None]) | (sig < 0.5 * tol[:, None]), axis=1)
    ok = np.count_nonzero(sig > tol[:, None], axis=1) == r
    out, off = [], 0
    for grp, hg, q in zip(groups, host_grams, q_devs):
        t_n = hg.shape[0]
        o = [bool(x) for x in ok[off:off + t_n]]
        for t in np.nonzero(~clear[off:off + t_n])[0]:
            o[t] = int(np.linalg.matrix_rank(q[t].cpu().numpy())) == r
        out.append(o)
        off += t_n
    return out


def seed_q_groups(groups, round_index):
    """Seed matrices of several PowerSGD groups with one device -> host round trip: all Gram
    matrices are computed, copied back together and decided with batched eigvalsh; only the
    (rare) rejected tensors loop through ensure_full_rank's redraws (compressors.py:591-603)."""
    from .configs import DegenerateMatrixError
    state = [grp.seed_start(round_index) for grp in groups]
    pending = list(range(len(groups)))
    for attempt in range(4):
        # warm Q of the previous round: its Gram is already on the host once that event fired
        ready = {}
        if attempt == 0:
            for i in pending:
                grp = groups[i]
                pg = grp._pending_gram
                if pg is not None and pg[0] is grp.warm and grp.cfg.warm_start:
                    pg[1].synchronize()
                    ready[i] = grp._gram_host.numpy()
        todo = [i for i in pending if i not in ready]
        grams = [groups[i]._gram(state[i][0]) for i in todo]
        host = torch.cat([x.reshape(-1) for x in grams]).cpu().numpy() if grams else None   # one sync
        off, hgs = 0, []
        for i in pending:
            if i in ready:
                hgs.append(ready[i])
            else:
                gm = grams[todo.index(i)]
                hgs.append(host[off:off + gm.numel()].reshape(gm.shape))
                off += gm.numel()
        # one batched eigvalsh over every pending group's Gram matrices (the host step between the
        # previous round's factor exchange and this round's first launch)
        oks = _rank_ok_many([groups[i] for i in pending], hgs, [state[i][0] for i in pending])
        still = []
        for i, ok in zip(pending, oks):
            grp = groups[i]
            if not all(ok):
                if attempt == 3:
                    raise DegenerateMatrixError("seed matrix rank-deficient after redraws")
                grp.seed_redraw(state[i][0], ok, state[i][1], round_index)
                still.append(i)
        if not still:
            break
        pending = still
    return [q for q, _ in state]


def _finish_steps(steps):
    """Resume a run_steps generator paused at its decode phase and run it to the end."""
    try:
        steps.send(None)
    except StopIteration as stop:
        return stop.value
    raise RuntimeError("PowerSGD round generator yielded after its decode phase")


def umma_unaligned() -> bool:
    """P = M Q for unaligned rows on the tcgen05 kernel (masked scalar producer, ef_apply fused)
    rather than ef_apply + the fp64 CUDA-core kernel; GC_PSGD_MQ_UNALIGNED=cores selects the latter."""
    return os.environ.get("GC_PSGD_MQ_UNALIGNED", "umma") != "cores"


class PowerSgdGroup:
    """T independent PowerSGD pipelines of the same length d (hence the same rows x cols),
    L workers each, run as one batch of kernels (pipelines.py:338-368 per tensor).

    The single-matrix reference path is T = 1 with rows at w * ld; the chunked mode of
    cfg4(b) passes per-(tensor, worker) row offsets into the flat per-worker gradients."""

    RANKS = (1, 2, 3, 4, 5, 6, 7, 8, 16)   # ranks the factor kernels are compiled for
    MAX_RANK = 1024                         # orthonormalization / Gram limit (kMaxOrthRank)

    @staticmethod
    def rank_chunks(r: int) -> list[int]:
        """Compiled ranks whose sum is r (16s, then 8, then the rest): a rank outside RANKS runs
        its factor passes chunk by chunk (P, Q and the decode are column-separable; the
        orthonormalization and the rank check see all r columns)."""
        out = []
        while r >= 16:
            out.append(16)
            r -= 16
        if r > 8:
            out.append(8)
            r -= 8
        if r:
            out.append(r)
        return out

    def __init__(self, cfg: PowerSgdConfig, n: int, L: int, d: int, T: int, seeds: SeedSpec, device,
                 row_offsets=None, est_offsets=None, ld: int = 0, host_offsets=None):
        self.cfg, self.n, self.L, self.d, self.T = cfg, n, L, d, T
        self.seeds, self.device = seeds, device
        self.rows, self.cols = matrix_shape_for(d)
        self.rank = cfg.rank
        if self.rank > self.MAX_RANK:
            raise NotImplementedError(f"PowerSGD rank {self.rank} > {self.MAX_RANK} is not supported")
        if self.rows < self.rank:
            raise ValueError("need a tall matrix (rows >= cols)")
        self.chunks = [self.rank] if self.rank in self.RANKS else self.rank_chunks(self.rank)
        self.row_offsets, self.est_offsets = row_offsets, est_offsets
        self.host_offsets = host_offsets   # [T] tensor offsets within a worker row (batched layout)
        self.batch = _native.PsgdBatch(T, L, _ptr(row_offsets), ld, _ptr(est_offsets), 0, 0)
        ws = int(_native.lib().gc_psgd_workspace_bytes(T * L, self.rows, self.cols, self.rank))
        self.ws = torch.empty(ws, dtype=torch.uint8, device=device)
        self.mgs_ws = torch.empty(int(_native.lib().gc_psgd_orth_workspace_bytes(T, self.rows, self.rank)),
                                  dtype=torch.uint8, device=device)
        self.gram_ws = torch.empty(int(_native.lib().gc_psgd_gram_workspace_bytes(T, self.rank)) // 8,
                                   dtype=torch.float64, device=device)
        self.warm = None          # [T][cols][r]
        self.last = {}
        self._gram_host = None    # pinned [T][r][r]: Gram of the warm Q, filled behind an event
        self._pending_gram = None
        self._bufs = {}           # per-round device buffers, allocated once (no allocator traffic)
        # deferred EF: (residual buffer ptr, P_hat, Q_w) of the last round when that buffer still holds
        # the round's corrected matrices (r = c - P_hat Q_w^T not yet materialised, see materialize)
        self.pending = None
        self.defer = os.environ.get("GC_PSGD_DEFER", "1") != "0"

    def _buf(self, name, shape, dtype=torch.float32):
        b = self._bufs.get(name)
        if b is None or tuple(b.shape) != tuple(shape) or b.dtype != dtype:
            b = self._bufs[name] = torch.empty(shape, dtype=dtype, device=self.device)
        return b

    def set_ld(self, ld: int, aligned: bool = False):
        self.batch.ld = ld
        self.batch.rows_aligned = 1 if aligned else 0

    def _gram(self, q_dev):
        gram = torch.empty(self.T, self.rank, self.rank, dtype=torch.float64, device=self.device)
        _native.call("gc_psgd_gram", self.T, self.cols, self.rank, q_dev.data_ptr(), gram.data_ptr(),
                     self.gram_ws.data_ptr(), _sp())
        return gram

    def _rank_ok_host(self, host_gram, q_dev):
        """Per tensor: np.linalg.matrix_rank(q) == rank (compressors.py:599), decided from the fp64
        Gram eigenvalues (one batched eigvalsh for all T tensors); near numpy's tolerance the exact
        numpy call on a host copy decides."""
        import numpy as np
        r, cols = self.rank, self.cols
        sig = np.sqrt(np.clip(np.linalg.eigvalsh(host_gram), 0.0, None))           # [T, r]
        tol = sig.max(axis=1, keepdims=True) * max(cols, r) * np.finfo(np.float32).eps
        clear = np.all((sig > 2 * tol) | (sig < 0.5 * tol), axis=1)
        ok = np.count_nonzero(sig > tol, axis=1) == r
        for t in np.nonzero(~clear)[0]:
            ok[t] = int(np.linalg.matrix_rank(q_dev[t].cpu().numpy())) == r
        return [bool(x) for x in ok]

    def _rank_ok(self, q_dev):
        return self._rank_ok_host(self._gram(q_dev).cpu().numpy(), q_dev)

    def seed_start(self, round_index):
        """The round's candidate seed matrices (warm Q or the first draw) and the draw counts."""
        import numpy as np
        T, cols, r = self.T, self.cols, self.rank
        if self.cfg.warm_start and self.warm is not None:
            return self.warm.clone(), [0] * T
        first = self.seeds.rng("lowrank-seed", round_index).standard_normal((cols, r)).astype(np.float32)
        return torch.from_numpy(first).to(self.device).unsqueeze(0).repeat(T, 1, 1).contiguous(), [1] * T

    def seed_redraw(self, q, ok, draws, round_index):
        """ensure_full_rank's redraw of every rejected tensor from its own rng stream."""
        import numpy as np
        cols, r = self.cols, self.rank
        for t in range(self.T):
            if not ok[t]:   # continue this tensor's own rng stream
                rng = self.seeds.rng("lowrank-seed", round_index)
                for _ in range(draws[t]):
                    rng.standard_normal((cols, r))
                q[t] = torch.from_numpy(rng.standard_normal((cols, r)).astype(np.float32)).to(self.device)
                draws[t] += 1

    def seed_q(self, round_index):
        """Seed matrices with ensure_full_rank's redraws, one reference rng per tensor
        (pipelines.py:341-346, compressors.py:591-603)."""
        return seed_q_groups([self], round_index)[0]

    def host_offsets_arg(self):
        """ctypes array of the batch's tensor offsets (element offset of tensor t in a worker row), or
        None for the single-matrix layout -- the TMA pass builds one tensor map per tensor."""
        if self.host_offsets is None:
            return None
        if getattr(self, "_hoffs", None) is None:
            self._hoffs = (ctypes.c_int64 * len(self.host_offsets))(*[int(x) for x in self.host_offsets])
        return self._hoffs

    def materialize(self, resid_ptr):
        """Write the deferred residuals r = c - P_hat Q_w^T (pipelines.py:357-361, ef_update) into the
        buffer that holds the last round's corrected matrices -- before anything but the next round's
        TMA P = M Q pass reads them.  A no-op when nothing is deferred."""
        if self.pending is None:
            return
        rp, ph, qw = self.pending
        self.pending = None
        if resid_ptr is None or rp != resid_ptr:   # the caller replaced the EF state
            return
        _native.call("gc_psgd_decode", ctypes.byref(self.batch), self.n, self.d, self.rows, self.cols, self.rank,
                     ph.data_ptr(), qw.data_ptr(), qw.data_ptr(), resid_ptr, None, _sp())

    def _mtp_ef_ok(self):
        # opt-in (GC_PSGD_MTP_EF=1): the fused pass moves exactly the algorithmic bytes but its
        # 128-byte column-strip segments run at ~1.7 TB/s, slower than mtp + decode
        if getattr(self, "_mtp_ef_cache", None) is None:
            self._mtp_ef_cache = os.environ.get("GC_PSGD_MTP_EF", "0") == "1"
        return self._mtp_ef_cache and bool(
            _native.lib().gc_psgd_mtp_ef_supported(self.rows, self.cols, self.rank, self.batch.rows_aligned))

    def run(self, c_ptr: int, resid_ptr, est_ptr: int, round_index: int, grads_ptr=None, vec=False, fold=None,
            before_ef=None, q=None, ef_resid_ptr=None, defer_decode=False):
        """One round for the batch (run_steps driven with `fold` at its two factor all-reduces).
        defer_decode: stop before the decode and return a callable that finishes the round (and
        returns warm Q), so a caller can queue the decodes of several groups after all their warm-Q
        Gram copies -- the next round's rank check then waits on the last Gram while every decode
        is still queued on the device."""
        steps = self.run_steps(c_ptr, resid_ptr, est_ptr, round_index, grads_ptr=grads_ptr, vec=vec,
                               before_ef=before_ef, q=q, ef_resid_ptr=ef_resid_ptr, decode_phase=defer_decode)
        req = next(steps)
        try:
            while True:
                if req[0] == "decode":
                    return lambda: _finish_steps(steps)
                req = steps.send(fold(*req))
        except StopIteration as stop:
            return stop.value

    def run_steps(self, c_ptr: int, resid_ptr, est_ptr: int, round_index: int, grads_ptr=None, vec=False,
                  before_ef=None, q=None, ef_resid_ptr=None, decode_phase=False):
        """One round for the batch as a generator: it yields each factor all-reduce as
        (kind, x [T*L][m], m) and resumes with its [T][m] sums in the reference ring order
        (simulated: local fold; distributed: exchange), so a caller can exchange the factors of
        several groups in one collective.  c_ptr: corrected matrices (or raw gradients when
        grads_ptr is given together with vec: ef_apply fused into P = M Q, corrected written over
        resid).  before_ef() runs after the estimate, before the residuals change (the nmse hook).
        ef_resid_ptr (with grads_ptr and vec): ef_apply fused into P = M Q, corrected written there
        (c_ptr must then point at it).  decode_phase: also yield ("decode", None, 0) once warm Q and
        its Gram copy are queued, before the decode (resume with None).  Returns warm Q [T][cols][r]."""
        sp = _sp()
        T, L, n, d, rows, cols, r = self.T, self.L, self.n, self.d, self.rows, self.cols, self.rank
        bref = ctypes.byref(self.batch)
        if q is None:
            q = self.seed_q(round_index)
        # rank chunks: (first column, width); one chunk = the compiled rank itself
        spans, c0 = [], 0
        for rc in self.chunks:
            spans.append((c0, rc))
            c0 += rc
        multi = len(spans) > 1

        def cols_of(x, c0, rc, name):
            if not multi:
                return x
            out = self._buf(name, x.shape[:-1] + (rc,))
            out.copy_(x[..., c0:c0 + rc])
            return out

        p = self._buf("p", (T * L, rows, r))
        # P = M Q on tcgen05 with the previous round's EF update riding along (deferred EF): TMA-fed
        # when a tensor map describes the rows, cp.async-fed otherwise (gc_psgd_mq_deferred_batched).
        # GC_PSGD_TMA=0: the register-fed pass (float4 producer for aligned rows, masked scalars
        # otherwise) with eager EF
        umma = vec or umma_unaligned()
        rp = ef_resid_ptr if ef_resid_ptr is not None else resid_ptr
        hoffs = self.host_offsets_arg()
        tma = (not multi and grads_ptr is not None and rp is not None and os.environ.get("GC_PSGD_TMA", "1") != "0"
               and bool(_native.lib().gc_psgd_mq_deferred_supported(bref, hoffs, d, rows, cols, r, grads_ptr, rp)))
        if self.pending is not None and not (tma and self.pending[0] == rp):
            self.materialize(rp)
        if tma:
            pend, self.pending = self.pending, None
            _native.call("gc_psgd_mq_deferred_batched", bref, hoffs, d, rows, cols, r, grads_ptr, rp, q.data_ptr(),
                         pend[1].data_ptr() if pend else None, pend[2].data_ptr() if pend else None, p.data_ptr(),
                         self.ws.data_ptr(), sp)
        for k, (c0, rc) in enumerate(spans):
            if tma:
                break
            q_c = cols_of(q, c0, rc, f"q_c{k}")
            p_c = self._buf(f"p_c{k}", (T * L, rows, rc)) if multi else p
            if umma and k == 0 and ef_resid_ptr is not None:
                _native.call("gc_psgd_mq_fused", bref, d, rows, cols, rc, grads_ptr, ef_resid_ptr, q_c.data_ptr(),
                             p_c.data_ptr(), self.ws.data_ptr(), sp)
            elif umma and k == 0 and grads_ptr is not None:
                _native.call("gc_psgd_mq_fused", bref, d, rows, cols, rc, grads_ptr, resid_ptr, q_c.data_ptr(),
                             p_c.data_ptr(), self.ws.data_ptr(), sp)
            elif umma:   # later chunks read the corrected matrices the first chunk left in c_ptr
                _native.call("gc_psgd_mq_fused", bref, d, rows, cols, rc, c_ptr, None, q_c.data_ptr(), p_c.data_ptr(),
                             self.ws.data_ptr(), sp)
            else:
                _native.call("gc_psgd_mq", bref, d, rows, cols, rc, c_ptr, q_c.data_ptr(), p_c.data_ptr(), sp)
            if multi:
                p[..., c0:c0 + rc].copy_(p_c)
        p_sum = (yield ("left-factor", p, rows * r)).reshape(T, rows, r)
        p_hat = self._buf("p_hat", (T, rows, r))
        status = self._buf("status", (T,), torch.int32).zero_()
        _native.call("gc_psgd_orthonormalize", T, rows, r, p_sum.data_ptr(), p_hat.data_ptr(), self.mgs_ws.data_ptr(),
                     status.data_ptr(), sp)
        qw = self._buf("qw", (T * L, cols, r))
        # Q_w and the EF update in one pass over M when nothing reads the corrected matrices
        # between them (no nmse hook; corrected held in resid); the estimate stays in decode
        mtp_ef = (not multi and before_ef is None and resid_ptr is not None and c_ptr == resid_ptr
                  and self._mtp_ef_ok())
        ph_chunks, qw_chunks = [], []
        for k, (c0, rc) in enumerate(spans):
            ph_c = cols_of(p_hat, c0, rc, f"ph_c{k}")
            qw_c = self._buf(f"qw_c{k}", (T * L, cols, rc)) if multi else qw
            if mtp_ef:
                _native.call("gc_psgd_mtp_ef", bref, d, rows, cols, rc, resid_ptr, ph_c.data_ptr(), qw_c.data_ptr(), sp)
            else:
                _native.call("gc_psgd_mtp_batched", bref, hoffs, d, rows, cols, rc, c_ptr, ph_c.data_ptr(),
                             qw_c.data_ptr(), self.ws.data_ptr(), sp)
            if multi:
                qw[..., c0:c0 + rc].copy_(qw_c)
            ph_chunks.append(ph_c)
            qw_chunks.append(qw_c)
        q_sum = (yield ("right-factor", qw, cols * r)).reshape(T, cols, r)
        # warm Q (pipelines.py:366) before the decode, and its Gram copied to pinned host memory
        # behind an event: the next round's rank check (ensure_full_rank) then reads it without
        # draining the device, so that round's kernels queue while this round's decode runs
        warm = self._buf("warm", (T, cols, r))   # the next round clones it before overwriting
        _native.call("gc_scale_div", T * cols * r, q_sum.data_ptr(), n, warm.data_ptr(), sp)
        self.warm = warm
        if self.cfg.warm_start:
            if self._gram_host is None:
                self._gram_host = torch.empty(T, r, r, dtype=torch.float64, pin_memory=True)
            self._gram_host.copy_(self._gram(warm), non_blocking=True)
            ev = torch.cuda.Event()
            ev.record()
            self._pending_gram = (warm, ev)
        if decode_phase:
            yield ("decode", None, 0)
        qs_chunks = [cols_of(q_sum, c0, rc, f"qs_c{k}") for k, (c0, rc) in enumerate(spans)]

        def decode(resid, est):
            # own = P_hat Q_w^T and the estimate are sums over the rank: chunk k > 0 subtracts its
            # part from the residual in place and adds its part to the estimate
            for k, (c0, rc) in enumerate(spans):
                self.batch.est_accumulate = 1 if (k > 0 and est is not None) else 0
                _native.call("gc_psgd_decode", bref, n, d, rows, cols, rc, ph_chunks[k].data_ptr(),
                             qw_chunks[k].data_ptr(), qs_chunks[k].data_ptr(), resid, est, sp)
            self.batch.est_accumulate = 0

        if mtp_ef:
            decode(None, est_ptr)
        elif tma and self.defer and resid_ptr is not None and rp == resid_ptr:
            # deferred EF: the estimate only; r = c - P_hat Q_w^T is folded into the next round's
            # P = M Q pass (or materialised when the residuals are read first)
            decode(None, est_ptr)
            if before_ef is not None:
                before_ef()
            self.pending = (rp, p_hat, qw)
        elif before_ef is None and resid_ptr is not None:   # EF update and estimate in one pass
            decode(resid_ptr, est_ptr)
        else:
            decode(None, est_ptr)
            if before_ef is not None:
                before_ef()
            if resid_ptr is not None:
                decode(resid_ptr, None)
        self.last = {"p_hat": p_hat, "q_sum": q_sum, "seed_q": q, "status": status, "qw": qw, "decode": decode}
        return warm


class PowerSgdEngine(Engine):
    """pipelines.py:324-368 (PowerSgdConfig), warm start and dense bypass included."""

    def __init__(self, cfg: PowerSgdConfig, n, dim, seeds, device):
        super().__init__(n, dim, seeds, device)
        self.cfg = cfg
        self.bypass = dim < cfg.bypass_below
        self.group = None if self.bypass else PowerSgdGroup(cfg, n, n, dim, 1, seeds, device)

    def warm_q(self):
        return None if self.group is None or self.group.warm is None else self.group.warm[0]

    def sync_residuals(self, res):
        if self.group is not None:
            self.group.materialize(_ptr(res))

    def drop_deferred(self):
        if self.group is not None:
            self.group.pending = None

    def _fold(self, kind, x, m):
        n = self.n
        if n == 1:   # one worker: the ring sum is the row itself
            return x.reshape(x.shape[0], m)
        out = torch.empty(x.shape[0] // n, m, dtype=torch.float32, device=self.device)
        _native.call("gc_float_fold_batched", x.shape[0] // n, n, m, x.data_ptr(), m, n * m, 0, 0, 0, out.data_ptr(),
                     m, _sp())
        return out

    def run(self, grads, res, round_index, ledger, nmse=True):
        n, d = self.n, self.dim
        sp = _sp()
        dev = self.device
        est = torch.empty(d, dtype=torch.float32, device=dev)
        acc = torch.zeros(2, dtype=torch.float64, device=dev) if nmse else None
        if self.bypass:   # dense fp32 ring (pipelines.py:326-336); own = corrected -> r_new = 0
            if res is not None:
                _native.call("gc_ef_apply", n, d, grads.data_ptr(), res.data_ptr(), grads.stride(0), res.data_ptr(),
                             res.stride(0), sp)
            c = res if res is not None else grads
            _native.call("gc_float_fold", n, d, c.data_ptr(), c.stride(0), 0, -(-d // n), 0, 0, n, est.data_ptr(), sp)
            if nmse:
                self._nmse(c, None, est, acc)
            if res is not None:
                _native.call("gc_fill_zero", res.data_ptr(), res.numel() * 4, sp)
            self.launches += 4
            ledger.charge_ring("dense-bypass", n, d, 32)
            return est, 32.0 * d, _simple_stats(acc)

        grp = self.group
        lib = _native.lib()
        fuse_ef = bool(res is not None and grads.stride(0) == res.stride(0) and
                       (umma_unaligned() or
                        lib.gc_psgd_vectorizable(grp.cols, grads.data_ptr(), res.data_ptr(), grads.stride(0))))
        if fuse_ef:   # ef_apply fused into P = M Q
            c, gptr = res, grads.data_ptr()
        else:
            grp.materialize(_ptr(res))
            if res is not None:
                _native.call("gc_ef_apply", n, d, grads.data_ptr(), res.data_ptr(), grads.stride(0), res.data_ptr(),
                             res.stride(0), sp)
                self.launches += 1
            c, gptr = (res if res is not None else grads), None
        vec = bool(lib.gc_psgd_vectorizable(grp.cols, c.data_ptr(), est.data_ptr(), c.stride(0)))
        grp.set_ld(c.stride(0), vec)
        ev = self._ev()
        if ev:
            ev[0].record()
        before = (lambda: self._nmse(c, None, est, acc)) if nmse else None
        grp.run(c.data_ptr(), _ptr(res), est.data_ptr(), round_index, grads_ptr=gptr, vec=vec, fold=self._fold,
                before_ef=before)
        if ev:
            ev[1].record()
        self.launches += 10
        if self.capture:
            self.last = {k: (v[0] if k not in ("status", "qw") else v) for k, v in grp.last.items() if not callable(v)}
        ledger.charge_ring("left-factor", n, grp.rows * grp.rank, 32)
        ledger.charge_ring("right-factor", n, grp.cols * grp.rank, 32)
        return est, 32.0 * grp.rank * (grp.rows + grp.cols), _simple_stats(acc)


def make_engine(cfg, n, dim, seeds, device, fused=True) -> Engine:
    if isinstance(cfg, PowerSgdConfig):
        return PowerSgdEngine(cfg, n, dim, seeds, device)
    if isinstance(cfg, ChunkedTopKConfig):
        return ChunkedEngine(cfg, n, dim, seeds, device)
    if isinstance(cfg, RotatedQuantConfig):
        return ThcEngine(cfg, n, dim, seeds, device, fused)
    if isinstance(cfg, DenseConfig):
        return DenseEngine(cfg, n, dim, seeds, device)
    if isinstance(cfg, TopKConfig):
        return TopKEngine(cfg, n, dim, seeds, device)
    raise NotImplementedError(f"{type(cfg).__name__} engine not built yet")
