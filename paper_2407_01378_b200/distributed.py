"""Multi-GPU GradientPipeline: one process per GPU, n logical workers split over the ranks.

Reference semantics are those of the simulated ring (pipelines.py:201-393,
collectives.py:177-263): worker w of the reference is global worker w = rank * L + l here
(L = n / world local workers per rank, all sharing one GPU's kernels).  The exchange steps
are the ones SURVEY.md §8(e) derives from the reference:

* THC: range consensus = all-reduce MAX of (-lo, hi) (min/max are order-free, exact);
  saturating code sums = all-to-all of 1/world slices of the codes -> ring-ordered
  saturating fold of the slice (gc_sat_fold, start worker floor(i / ceil(P/n)) as in the
  reference's padded ring partition) -> all-gather of the summed slices.  NCCL's wrapping
  int8 sum cannot reproduce the clamp-per-hop order, so it is not used for codes.
* TopK: all-gather of the (index, value) payloads, ordered scatter-add (worker-id order).
* TopK-Chunked: all-gather of the fp16 chunk energies and of the chunk packs, then the
  fp16-wire ring fold locally (bit-exact selection and sums).
* PowerSGD: all-gather of the P and Q factors (rows*r and cols*r floats) and the fp32 ring
  fold locally, so P_hat / Q_sum are bit-identical on every rank and to the reference order.
* Dense FP16 / FP32 (the utility bar): NCCL all-reduce in half / float (tolerance-level
  agreement; this is the baseline the compressed schemes are measured against).

Collectives go through `Comm`, a thin layer over torch.distributed: NCCL with CUDA tensors,
or gloo with host staging (used by the CPU tests of the exchange plan and by the
two-process single-GPU tests).
"""

from __future__ import annotations

import ctypes
import math
import os

import numpy as np
import torch
import torch.distributed as dist

from . import _native
from .configs import (
    ChunkedTopKConfig, DenseConfig, PowerSgdConfig, RotatedQuantConfig, TopKConfig, scheme_label,
)
from .ledger import OverflowStats, TrafficLedger, WorkerGroup
from .pipeline import RoundResult
from .schemes import RoundStats, _simple_stats, nmse_from
from .vectors import ChunkGeometry, GradientVector, SeedSpec, next_pow2


def _sp() -> int:
    return _native.current_stream_handle()


def _ptr(t):
    return None if t is None else t.data_ptr()


class Comm:
    """Collectives used by the exchange plan (NCCL on CUDA tensors, gloo with host staging).

    `sent` counts, per ledger phase, the payload bytes this rank delivers to the other ranks:
    (world-1) x own bytes for an all-gather, the off-rank chunks of an all-to-all, and
    2 (world-1) / world x bytes for an all-reduce (the ring's reduce-scatter + all-gather) --
    the quantities the reference's TrafficLedger meters per worker (collectives.py:209-262)."""

    def __init__(self, group=None):
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.stage = dist.get_backend(group) != "nccl"
        # a one-rank gloo group needs no transport; a one-rank NCCL group still issues every
        # collective (local copies), so the per-rank NCCL path runs as it does at N ranks
        self.local_only = self.world == 1 and self.stage
        self.sent: dict[str, int] = {}

    def _count(self, phase, nbytes):
        if phase is not None and self.world > 1:
            self.sent[phase] = self.sent.get(phase, 0) + int(nbytes)

    def _run(self, fn, out, *ins):
        if self.stage and out.is_cuda:
            h_out = torch.empty(out.shape, dtype=out.dtype)
            fn(h_out, *[x.cpu() for x in ins])
            out.copy_(h_out)
        else:
            fn(out, *ins)
        return out

    def all_gather_rows(self, x: torch.Tensor, phase: str | None = None) -> torch.Tensor:
        """[L, ...] per rank -> [world * L, ...] in rank order (global worker order).

        Pure data movement, done on a byte view (int16 sums are not an NCCL / gloo type)."""
        x = x.contiguous()
        self._count(phase, (self.world - 1) * x.numel() * x.element_size())
        out = torch.empty((self.world * x.shape[0],) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
        if self.local_only:
            out.copy_(x)
            return out
        self._run(lambda o, i: dist.all_gather_into_tensor(o, i, group=self.group),
                  out.view(-1).view(torch.uint8), x.view(-1).view(torch.uint8))
        return out

    def all_to_all(self, send: torch.Tensor, phase: str | None = None) -> torch.Tensor:
        """send [world, ...]: chunk r goes to rank r; returns recv [world, ...], chunk r from rank r."""
        send = send.contiguous()
        self._count(phase, (self.world - 1) * (send.numel() // self.world) * send.element_size())
        recv = torch.empty_like(send)
        if self.local_only:
            recv.copy_(send)
            return recv
        self._run(lambda o, i: dist.all_to_all_single(o, i, group=self.group),
                  recv.view(-1).view(torch.uint8), send.view(-1).view(torch.uint8))
        return recv

    def _count_ring(self, phase, t: torch.Tensor, rings: int):
        # what `rings` reference ring all-reduces of numel / rings elements send per worker:
        # 2 (W - 1) ceil(len / W) elements each (collectives.py:209-233)
        per = t.numel() // rings
        self._count(phase, rings * 2 * (self.world - 1) * -(-per // self.world) * t.element_size())

    def all_reduce_async(self, t: torch.Tensor, op, phase: str | None = None, rings: int = 1):
        """In-place all-reduce of a contiguous tensor; returns a work handle to wait() on before
        the result is used (NCCL: the current stream waits), or None when already complete.
        `rings`: the tensor stands for that many equal reference rings (for the wire accounting)."""
        self._count_ring(phase, t, rings)
        if self.local_only or t.numel() == 0:
            return None
        if self.stage and t.is_cuda:
            h = t.cpu()
            dist.all_reduce(h, op=op, group=self.group)
            t.copy_(h)
            return None
        return dist.all_reduce(t, op=op, group=self.group, async_op=True)

    def all_reduce(self, t: torch.Tensor, op, phase: str | None = None, rings: int = 1) -> torch.Tensor:
        self._count_ring(phase, t, rings)
        if self.local_only:
            return t
        if self.stage and t.is_cuda:
            h = t.cpu()
            dist.all_reduce(h, op=op, group=self.group)
            t.copy_(h)
        else:
            dist.all_reduce(t, op=op, group=self.group)
        return t


def fold_slices(active: int, world: int, align: int = 256) -> int:
    """Length of the equal per-rank slices of the code vector for the all-to-all fold."""
    s = -(-active // world)
    s = -(-s // align) * align
    return s


def _nibbles(x: torch.Tensor, pack: bool) -> torch.Tensor:
    """int8 [.., 2m] <-> uint8 [.., m] nibble pairs on the device (gc_pack_nibbles)."""
    x = x.contiguous()
    if pack:
        out = torch.empty(x.shape[:-1] + (x.shape[-1] // 2,), dtype=torch.uint8, device=x.device)
        _native.call("gc_pack_nibbles", x.numel(), x.data_ptr(), out.data_ptr(), _sp())
    else:
        out = torch.empty(x.shape[:-1] + (x.shape[-1] * 2,), dtype=torch.int8, device=x.device)
        _native.call("gc_unpack_nibbles", out.numel(), x.data_ptr(), out.data_ptr(), _sp())
    return out


def exchange_sums(send: torch.Tensor, comm: Comm, n: int, active: int, slice_len: int, fold_fn, out_dtype,
                  phase: str | None = None, nibble: bool = False) -> torch.Tensor:
    """The code exchange for a send buffer already in the all-to-all layout [W][L][S] (int8, or
    packed nibbles [W][L][S/2] when nibble): all-to-all, ordered saturating fold of this rank's
    slice over the n worker rows, all-gather of the summed slices (collectives.py:215-235)."""
    recv = comm.all_to_all(send, phase)
    if nibble:
        recv = _nibbles(recv, False)
    recv = recv.reshape(n, slice_len)
    s0 = comm.rank * slice_len
    my_len = max(0, min(slice_len, active - s0))
    if n == 1 and out_dtype == recv.dtype:   # one worker: its codes are the sums (tail already zero)
        sums = recv[0]
    else:
        sums = torch.empty(slice_len, dtype=out_dtype, device=send.device)
        if my_len < slice_len:
            sums[my_len:].zero_()
        if my_len:
            fold_fn(recv, my_len, s0, sums)
    if nibble:
        return _nibbles(comm.all_gather_rows(_nibbles(sums.reshape(1, -1), True), phase), False).reshape(-1)
    return comm.all_gather_rows(sums.reshape(1, -1), phase).reshape(-1)


def exchange_fold(codes: torch.Tensor, comm: Comm, n: int, active: int, slice_len: int, fold_fn, out_dtype,
                  send: torch.Tensor | None = None, phase: str | None = None, nibble: bool = False) -> torch.Tensor:
    """Saturating code sums over all n workers, reference ring order (collectives.py:215-235).

    codes: this rank's [L, active] int8 codes (global workers rank*L .. rank*L+L-1).  Slice
    r = [r*S, (r+1)*S) of every worker goes to rank r (all-to-all); rank r folds its slice
    over the n worker rows with fold_fn(rows [n, S], length, offset) -> sums [S]; the summed
    slices are all-gathered.  Returns sums [world*S] (entries >= active are zero)."""
    W, L = comm.world, codes.shape[0]
    if send is None:
        send = torch.zeros(W, L, slice_len, dtype=codes.dtype, device=codes.device)
    for dst in range(W):
        lo, hi = dst * slice_len, min(active, (dst + 1) * slice_len)
        if hi > lo:
            send[dst, :, : hi - lo].copy_(codes[:, lo:hi])
    if nibble:   # wire_bits <= 4: codes and sums travel as packed nibbles (the ledger's b bits)
        recv = _nibbles(comm.all_to_all(_nibbles(send, True), phase), False).reshape(n, slice_len)
    else:
        recv = comm.all_to_all(send, phase).reshape(n, slice_len)
    s0 = comm.rank * slice_len
    my_len = max(0, min(slice_len, active - s0))
    sums = torch.zeros(slice_len, dtype=out_dtype, device=codes.device)
    if my_len:
        fold_fn(recv, my_len, s0, sums)
    if nibble:
        return _nibbles(comm.all_gather_rows(_nibbles(sums.reshape(1, -1), True), phase), False).reshape(-1)
    return comm.all_gather_rows(sums.reshape(1, -1), phase).reshape(-1)


def exchange_float(x: torch.Tensor, comm: Comm, n: int, phase: str | None, wire16: bool) -> torch.Tensor:
    """FloatSum ring all-reduce (collectives.py:112-120, 177-236) of [L, m] float32 rows per rank,
    exact in the reference's ring order and with the ring's wire volume: slice r of every row goes to
    rank r (all-to-all), rank r folds its slice over the n worker rows in ring order (gc_float_fold:
    element i starts at worker floor(i / ceil(m/n)), fp16 wire per hop when wire16), and the folded
    slices are all-gathered -- 2 (W-1) ceil(m/W) elements per rank, the ledger's 2 (n-1) ceil(m/n)
    when every rank holds one worker.  Rows are fp16-valued when wire16 (they travel as binary16).
    Returns the [m] sums on every rank."""
    W, L, m = comm.world, x.shape[0], x.shape[1]
    S = -(-m // W)
    wdt = torch.float16 if wire16 else torch.float32
    send = torch.empty(W, L, S, dtype=wdt, device=x.device)
    for r in range(W):
        lo, hi = r * S, min(m, (r + 1) * S)
        if hi > lo:
            send[r, :, : hi - lo].copy_(x[:, lo:hi])
        if hi - lo < S:   # the padded tail of the last slices (never folded; zero on the wire)
            send[r, :, max(0, hi - lo):].zero_()
    recv = comm.all_to_all(send, phase).reshape(n, S).float()
    s0 = comm.rank * S
    my_len = max(0, min(S, m - s0))
    out = torch.empty(1, S, dtype=torch.float32, device=x.device)
    if my_len < S:
        out[:, my_len:].zero_()
    if my_len:
        _native.call("gc_float_fold", n, my_len, recv.data_ptr(), S, s0, -(-m // n), int(wire16), 0, 0,
                     out.data_ptr(), _sp())
    return comm.all_gather_rows(out.to(wdt), phase).reshape(-1)[:m].float()


class DistributedGradientPipeline:
    """GradientPipeline (pipelines.py:97-393) over torch.distributed ranks.

    num_workers is the global n; each rank passes its L = n / world local gradients to
    run_round (a [L, d] tensor or a list); the returned estimate is identical on every rank.
    Local residuals (`residuals`) belong to the rank's own workers.
    """

    def __init__(self, config, num_workers: int, dim: int, seeds: SeedSpec, error_feedback: bool | None = None, *,
                 group=None, device=None, validate: bool = True, compute_nmse: bool = False):
        """compute_nmse=True fills RoundResult.nmse as the reference does (an fp64 all-reduce of the
        corrected gradients per round); off by default, in which case nmse is NaN."""
        if num_workers < 1:
            raise ValueError("num_workers must be positive")
        if dim < 1:
            raise ValueError("dim must be positive")
        self.comm = Comm(group)
        if num_workers % self.comm.world:
            raise ValueError("num_workers must be a multiple of the number of ranks")
        self.config = config
        self.scheme = scheme_label(config)
        self.group = WorkerGroup(num_workers)
        self.dim = dim
        self.seeds = seeds
        self.L = num_workers // self.comm.world
        self.w0 = self.comm.rank * self.L
        if isinstance(config, DenseConfig):
            if error_feedback:
                raise ValueError("dense baselines do not carry error feedback")
            error_feedback = False
        elif error_feedback is None:
            error_feedback = True
        self.error_feedback = bool(error_feedback)
        if isinstance(config, TopKConfig) and config.k > dim:
            raise ValueError("k exceeds the dimension")
        if isinstance(config, ChunkedTopKConfig):
            if config.chunks_selected > ChunkGeometry.for_dim(dim, config.chunk_size).num_chunks:
                raise ValueError("chunks_selected exceeds the chunk count")
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.validate = validate
        self.compute_nmse = compute_nmse
        self._res = (torch.zeros(self.L, dim, dtype=torch.float32, device=self.device) if self.error_feedback
                     else None)
        self._stage = None
        self._engine = _make(config, self)

    # state --------------------------------------------------------------------------
    @property
    def residuals(self):
        if self._res is None:
            return None
        self._engine.sync_residuals(self._res)
        h = self._res.cpu().numpy()
        return [h[i].copy() for i in range(self.L)]

    @property
    def residuals_tensor(self):
        if self._res is not None:
            self._engine.sync_residuals(self._res)
        return self._res

    @property
    def _warm_q(self):
        wq = getattr(self._engine, "warm", None)
        return None if wq is None else wq.cpu().numpy()

    # round ---------------------------------------------------------------------------
    def run_round(self, local_grads, round_index: int) -> RoundResult:
        g = self._checked(local_grads)
        ledger = TrafficLedger()
        self.comm.sent = {}
        ref = self._nmse_reference(g) if self.compute_nmse else None
        est, bits, stats = self._engine.run(g, self._res, round_index, ledger, self.compute_nmse)
        if ref is not None:
            stats = _NmseStats(stats, self._nmse_acc(est, ref))
        res = RoundResult(self.scheme, round_index, est, self.dim, ledger, bits, stats)
        res.wire_bytes = dict(self.comm.sent)   # bytes this rank sent per ledger phase
        return res

    def _nmse_reference(self, g) -> torch.Tensor:
        """The reference's nmse target (pipelines.py:176-181): the fp64 mean of every worker's
        corrected gradient, summed over the ranks (an fp64 all-reduce of d values: the opt-in
        diagnostic's cost).  Taken before the round overwrites the residuals."""
        c = g.double()
        if self._res is not None:
            self._engine.sync_residuals(self._res)
            c += self._res.double()
        total = c.sum(0)
        self.comm.all_reduce(total, dist.ReduceOp.SUM)
        return total / self.group.size

    def _nmse_acc(self, est, ref) -> torch.Tensor:
        """[sum (est - ref)^2, sum ref^2] in fp64 (metrics.py:32-37)."""
        e = est.double() - ref
        return torch.stack([torch.dot(e, e), torch.dot(ref, ref)])

    def _checked(self, local_grads) -> torch.Tensor:
        L, d = self.L, self.dim
        if torch.is_tensor(local_grads) and local_grads.dim() == 2:
            if tuple(local_grads.shape) != (L, d):
                raise ValueError("need [local_workers, dim] gradients")
            g = local_grads
            if g.device != self.device or not g.is_contiguous() or g.dtype != torch.float32:
                g = self._buf().copy_(g, non_blocking=True)
        else:
            if len(local_grads) != L:
                raise ValueError("need exactly one gradient per local worker")
            g = self._buf()
            for i, x in enumerate(local_grads):
                if isinstance(x, GradientVector):
                    x = x.tensor if x.tensor is not None else x.logical
                t = x if torch.is_tensor(x) else torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32))
                if t.dim() != 1 or t.numel() != d:
                    raise ValueError("gradient length does not match the pipeline dim")
                g[i].copy_(t, non_blocking=True)
        if self.validate:
            bad = torch.zeros(1, dtype=torch.int64, device=self.device)
            _native.call("gc_check_finite", L, g.data_ptr(), g.stride(0), d, bad.data_ptr(), _sp())
            self.comm.all_reduce(bad, dist.ReduceOp.SUM)
            self._engine.launches += 1
            if int(bad.item()):
                raise ValueError("gradients must be finite")
        return g

    def _buf(self):
        if self._stage is None:
            self._stage = torch.empty(self.L, self.dim, dtype=torch.float32, device=self.device)
        return self._stage


class _NmseStats:
    """An engine's RoundStats with the nmse taken from the distributed fp64 accumulators."""

    def __init__(self, stats, acc):
        self._s, self._acc, self._nmse = stats, acc, None

    def nmse(self) -> float:
        if self._nmse is None:
            self._nmse = nmse_from(self._acc.cpu().tolist())
        return self._nmse

    def overflow(self):
        return self._s.overflow()

    def range_clips(self) -> int:
        return self._s.range_clips()


# ======================================================================================
class _Base:
    def __init__(self, pipe: DistributedGradientPipeline):
        self.p = pipe
        self.n, self.L, self.w0, self.dim = pipe.group.size, pipe.L, pipe.w0, pipe.dim
        self.comm, self.dev, self.seeds = pipe.comm, pipe.device, pipe.seeds
        self.launches = 0
        self.kernel_events = None

    def _ev(self):
        if self.kernel_events is None:
            return None
        e = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
        self.kernel_events.append(e)
        return e

    def sync_residuals(self, res):
        """Materialise an EF update deferred into the next round (PowerSGD)."""

    def drop_deferred(self):
        pass


class _Thc(_Base):
    """RotatedQuantConfig round (pipelines.py:260-322) for this rank's L workers.

    Rotation blocks 32..1024 (the paper's settings) run the fused per-rank kernels of
    gc_thc_rank.cu over L2-sized segments of tiles:

        K1(s)  ranges of segment s                       (reads g, r; they stay in L2)
        AR(s)  NCCL MAX all-reduce of segment s's (-lo, hi) pairs, async -- K1(s+1) runs meanwhile
        K2(s)  quantize + codes into the all-to-all send buffer + own decode + EF (g, r from L2)

    then one all-to-all of the codes, the ring-ordered saturating fold of this rank's slice, one
    all-gather of the sums and K3, the estimate decode.  Other block sizes use the generic
    multi-kernel path (gc_thc_rotate / quantize / decode)."""

    SEG_TILES = 32768   # tiles (of 1024 coordinates) per segment across ranks
    DEPTH = 2           # segments whose K1 and range all-reduce are in flight before K2 runs

    def __init__(self, cfg: RotatedQuantConfig, pipe):
        super().__init__(pipe)
        self.cfg = cfg
        d = self.dim
        P = next_pow2(d)
        B = 1 << min(P.bit_length() - 1, cfg.rotation_block.bit_length() - 1)
        self.P, self.B = P, B
        self.geom = _native.ThcGeom(d, P, B, cfg.quant_bits, cfg.wire_bits, float(B) ** -0.5)
        self.active = int(_native.lib().gc_thc_active_len(ctypes.byref(self.geom)))
        self.nb = self.active // B
        self.ring_blk = -(-P // self.n)
        self.sum_bytes = 1 if cfg.wire_bits <= 8 else (2 if cfg.wire_bits <= 16 else 4)
        self.sum_dtype = {1: torch.int8, 2: torch.int16, 4: torch.int32}[self.sum_bytes]
        self.nibble = cfg.wire_bits <= 4
        L, W = self.L, self.comm.world
        self.fused = P >= 1024 and 32 <= B <= 1024 and L <= 16
        self.k1_signs = os.environ.get("GC_THC_K1_SIGNS", "1") != "0"   # signs drawn inside K1
        i32 = dict(dtype=torch.int32, device=self.dev)
        self.counters = torch.zeros(4, dtype=torch.int64, device=self.dev)
        if self.fused:
            self.tiles = -(-self.active // 1024)
            self.S = fold_slices(self.active, W, align=1024)
            self.signs = torch.empty(self.tiles * 32, **i32)
            self.neg = torch.empty(L, self.nb, 2, dtype=torch.float32, device=self.dev)
            self.shared = self.neg[0] if L == 1 else torch.empty(self.nb, 2, dtype=torch.float32, device=self.dev)
            if self.nibble:
                self.send = torch.zeros(W, L, self.S // 2, dtype=torch.uint8, device=self.dev)
            else:
                self.send = torch.zeros(W, L, self.S, dtype=torch.int8, device=self.dev)
            # one segment on a one-rank group (nothing to overlap); across ranks segments of
            # SEG_TILES so the range all-reduce of one overlaps the next one's K1
            env = os.environ.get("GC_THC_RANK_SEG_TILES")
            self.seg_tiles = max(1, int(env)) if env else (self.tiles if W == 1 else self.SEG_TILES)
            # bench roofline: the whole per-rank round, algorithmic bytes per SURVEY §8(d) (g, r in,
            # r_new and codes out, summed codes in, estimate out)
            w = 0.5 if self.nibble else 1
            self.timed_kernel = "thc per-rank round (K1 + K2 + exchange + K3)"
            self.timed_kernel_bytes = int((12 * L + 4 + w * (L + 1)) * d)
        else:
            self.S = fold_slices(self.active, W)
            ws = int(_native.lib().gc_thc_workspace_bytes(ctypes.byref(self.geom), L))
            self.ws = torch.empty(max(ws, 1), dtype=torch.uint8, device=self.dev) if ws else None
            self.signs = torch.empty(-(-self.active // 32), **i32)
            self.x_rot = torch.empty(L, self.active, dtype=torch.float32, device=self.dev)
            self.ranges = torch.empty(L, self.nb, 2, dtype=torch.float32, device=self.dev)
            self.codes = torch.empty(L, self.active, dtype=torch.int8, device=self.dev)
            self.send = torch.zeros(W, L, self.S, dtype=torch.int8, device=self.dev)

    def _coins(self, r):
        coins = (_native.Pcg64 * self.L)()
        for l in range(self.L):
            coins[l] = self.seeds.pcg("stochastic-round", r, self.w0 + l)   # pipelines.py:293
        return coins

    def _fold(self, counters):
        cfg, n = self.cfg, self.n

        def fold(rows, length, offset, out):
            if n > 1:
                _native.call("gc_sat_fold", n, length, rows.data_ptr(), rows.stride(0), offset, self.ring_blk,
                             cfg.wire_bits, out.data_ptr(), counters[3:].data_ptr(), _sp())
            else:
                out[:length].copy_(rows[0, :length])
        return fold

    def run(self, g, res, r, ledger, nmse):
        n, L, cfg, comm = self.n, self.L, self.cfg, self.comm
        sp = _sp()
        geom = ctypes.byref(self.geom)
        rot = self.seeds.pcg("rotation-signs", r)                            # transforms.py:80-82
        # the fused path draws the signs inside K1 (gc_thc_rank_ranges_signs): K1 streams g and r, so
        # the PCG64 work rides in its spare issue slots instead of a separate pass
        self._rot = rot if (self.fused and self.k1_signs) else None
        if self._rot is None:
            _native.call("gc_thc_signs", ctypes.byref(rot), self.signs.numel() * 32, self.signs.data_ptr(), sp)
        coins = self._coins(r)
        counters = self.counters = torch.zeros(4, dtype=torch.int64, device=self.dev)
        ev = self._ev()
        if ev:
            ev[0].record()
        if self.fused:
            sums = self._run_fused(g, res, coins, counters, geom, sp)
            shared = self.shared
        else:
            sums, shared = self._run_generic(g, res, coins, counters, geom, sp)
        est = torch.empty(self.dim, dtype=torch.float32, device=self.dev)
        if self.fused:
            _native.call("gc_thc_rank_decode", geom, n, sums.data_ptr(), self.sum_bytes, shared.data_ptr(),
                         self.signs.data_ptr(), est.data_ptr(), sp)
        else:
            _native.call("gc_thc_decode_estimate", geom, n, sums.data_ptr(), self.sum_bytes, shared.data_ptr(),
                         self.signs.data_ptr(), est.data_ptr(), _ptr(self.ws), sp)
            if res is not None:
                _native.call("gc_thc_decode_ef", geom, L, self.codes.data_ptr(), shared.data_ptr(),
                             self.signs.data_ptr(), g.data_ptr(), res.data_ptr(), res.stride(0), _ptr(self.ws), sp)
        if ev:
            ev[1].record()
        comm.all_reduce(counters, dist.ReduceOp.SUM)   # clamp count, sum z, sum z^2, clips
        num_blocks = self.P // self.B
        ledger.charge_ring("range-consensus", n, num_blocks, 32)
        ledger.charge_ring("range-consensus", n, num_blocks, 32)
        ledger.charge_ring("code-aggregate", n, self.P, cfg.wire_bits)
        total = n * self.P
        total_adds = (n - 1) * self.ring_blk * n if n > 1 else 0

        def finalize(c, m):
            var = (total * c[2] - c[1] * c[1]) / (total * total)
            return {"nmse": float("nan"), "range_clips": int(c[0]),
                    "overflow": OverflowStats(int(c[3]), int(total_adds), math.sqrt(max(var, 0.0)))}

        return est, float(cfg.wire_bits * self.P + 64 * num_blocks), RoundStats(counters, None, finalize)

    def _run_fused(self, g, res, coins, counters, geom, sp):
        L, comm, B = self.L, self.comm, self.B
        seg = self.seg_tiles
        bounds = [(t, min(t + seg, self.tiles)) for t in range(0, self.tiles, seg)]
        pending = []

        def k2(tb, te, work):
            if work is not None:
                work.wait()
            _native.call("gc_thc_rank_quant", geom, L, g.data_ptr(), _ptr(res), _ptr(res), g.stride(0), tb, te,
                         self.signs.data_ptr(), self.shared.data_ptr(), coins, self.send.data_ptr(), self.S,
                         int(self.nibble), counters.data_ptr(), sp)
            self.launches += 1

        for tb, te in bounds:
            if self._rot is not None:
                _native.call("gc_thc_rank_ranges_signs", geom, L, g.data_ptr(), _ptr(res), g.stride(0), tb, te,
                             ctypes.byref(self._rot), self.signs.data_ptr(), self.neg.data_ptr(), sp)
            else:
                _native.call("gc_thc_rank_ranges", geom, L, g.data_ptr(), _ptr(res), g.stride(0), tb, te,
                             self.signs.data_ptr(), self.neg.data_ptr(), sp)
            b0, b1 = tb * 1024 // B, min(te * 1024 // B, self.nb)
            if L > 1:   # this rank's L tables -> one, rows b0..b1
                part = self.neg[:, b0:b1].contiguous()
                _native.call("gc_thc_merge_ranges", L, b1 - b0, part.data_ptr(), self.shared[b0:b1].data_ptr(), sp)
            self.launches += 1 + (L > 1)
            # ElemMin / ElemMax ring (pipelines.py:271-288) as one MAX all-reduce of (-lo, hi)
            work = comm.all_reduce_async(self.shared[b0:b1], dist.ReduceOp.MAX, "range-consensus", rings=2)
            pending.append((tb, te, work))
            if len(pending) > self.DEPTH:
                k2(*pending.pop(0))
        while pending:
            k2(*pending.pop(0))
        return exchange_sums(self.send, comm, self.n, self.active, self.S, self._fold(counters), self.sum_dtype,
                             "code-aggregate", nibble=self.nibble)

    def _run_generic(self, g, res, coins, counters, geom, sp):
        L, comm, cfg = self.L, self.comm, self.cfg
        _native.call("gc_thc_rotate", geom, L, g.data_ptr(), _ptr(res), g.stride(0), self.signs.data_ptr(),
                     self.x_rot.data_ptr(), self.ranges.data_ptr(), _ptr(self.ws), sp)
        shared = torch.empty(self.nb, 2, dtype=torch.float32, device=self.dev)
        _native.call("gc_range_consensus", L, self.nb, self.ranges.data_ptr(), shared.data_ptr(), sp)
        shared[:, 0].neg_()
        comm.all_reduce(shared, dist.ReduceOp.MAX, "range-consensus", rings=2)
        shared[:, 0].neg_()
        _native.call("gc_thc_quantize", geom, L, self.x_rot.data_ptr(), shared.data_ptr(), coins,
                     self.codes.data_ptr(), counters.data_ptr(), sp)
        sums = exchange_fold(self.codes, comm, self.n, self.active, self.S, self._fold(counters), self.sum_dtype,
                             self.send, "code-aggregate", nibble=cfg.wire_bits <= 4)
        self.launches += 7
        return sums, shared


class _TopK(_Base):
    def __init__(self, cfg: TopKConfig, pipe):
        super().__init__(pipe)
        self.k = cfg.k
        ws = int(_native.lib().gc_topk_workspace_bytes(self.L, self.dim))
        self.ws = torch.zeros(ws, dtype=torch.uint8, device=self.dev)   # zeroed: no threshold hint yet
        mws = int(_native.lib().gc_sparse_mean_workspace_bytes(self.n, self.dim))
        self.mean_ws = torch.empty(mws, dtype=torch.uint8, device=self.dev)

    def run(self, g, res, r, ledger, nmse):
        L, k, d, n = self.L, self.k, self.dim, self.n
        sp = _sp()
        idx = torch.empty(L, k, dtype=torch.int32, device=self.dev)
        val = torch.empty(L, k, dtype=torch.float32, device=self.dev)
        # ef_update fused into the select (own payload = the fp16 values at idx)
        flags = _native.TOPK_FP16_VALUES | (_native.TOPK_EF_UPDATE if res is not None else 0)
        _native.call("gc_topk_select", L, d, None, g.stride(0), k, g.data_ptr(), _ptr(res), idx.data_ptr(),
                     val.data_ptr(), flags, self.ws.data_ptr(), sp)
        # all_gather (collectives.py:239-263) of the SparsePayload wire: int32 indices + fp16 values
        all_idx = self.comm.all_gather_rows(idx, "sparse-gather")
        all_val = self.comm.all_gather_rows(val.half(), "sparse-gather").float()
        est = torch.empty(d, dtype=torch.float32, device=self.dev)
        _native.call("gc_sparse_mean", n, k, all_idx.data_ptr(), all_val.data_ptr(), d, n, est.data_ptr(),
                     self.mean_ws.data_ptr(), sp)
        self.launches += 11 + n
        ledger.charge_gather("sparse-gather", [48 * k] * n)
        return est, float(48 * k), _simple_stats(None)


class _Chunked(_Base):
    def __init__(self, cfg: ChunkedTopKConfig, pipe):
        super().__init__(pipe)
        self.cfg = cfg
        self.C, self.J = cfg.chunk_size, cfg.chunks_selected
        self.nc = -(-self.dim // self.C)
        ws = int(_native.lib().gc_topk_workspace_bytes(1, self.nc))
        self.ws = torch.zeros(ws, dtype=torch.uint8, device=self.dev)   # zeroed: no threshold hint yet

    def run(self, g, res, r, ledger, nmse):
        L, n, d, C, J, nc = self.L, self.n, self.dim, self.C, self.J, self.nc
        sp = _sp()
        if res is not None:
            _native.call("gc_ef_apply", L, d, g.data_ptr(), res.data_ptr(), g.stride(0), res.data_ptr(),
                         res.stride(0), sp)
            work = res
        else:
            work = g
        perm = None
        if self.cfg.permute:
            p = self.seeds.rng("coordinate-permutation", r).permutation(d)
            perm = torch.from_numpy(p.astype(np.int64)).to(self.dev)
        pp = _ptr(perm)
        norms = torch.empty(L, nc, dtype=torch.float32, device=self.dev)
        _native.call("gc_chunk_norms", L, d, C, work.data_ptr(), work.stride(0), pp, norms.data_ptr(), sp)
        # norm consensus: fp16-wire FloatSum ring (pipelines.py:224-232), ring volume, reference order
        energy = exchange_float(norms, self.comm, n, "norm-consensus", wire16=True)
        sel = torch.empty(J, dtype=torch.int32, device=self.dev)
        _native.call("gc_topk_select", 1, nc, energy.data_ptr(), nc, J, None, None, sel.data_ptr(), None, 0,
                     self.ws.data_ptr(), sp)
        Lc = J * C
        packs = torch.empty(L, Lc, dtype=torch.float32, device=self.dev)
        _native.call("gc_chunk_pack", L, d, C, J, sel.data_ptr(), work.data_ptr(), work.stride(0), pp,
                     packs.data_ptr(), sp)
        summed = exchange_float(packs, self.comm, n, "chunk-aggregate", wire16=True)   # pipelines.py:235-251
        est = torch.empty(d, dtype=torch.float32, device=self.dev)
        _native.call("gc_chunk_scatter", d, C, J, sel.data_ptr(), summed.data_ptr(), n, pp, est.data_ptr(), sp)
        if res is not None:
            _native.call("gc_chunk_ef_update", L, d, C, J, sel.data_ptr(), packs.data_ptr(), pp, res.data_ptr(),
                         res.stride(0), sp)
        self.launches += 16
        ledger.charge_ring("norm-consensus", n, nc, 16)
        ledger.charge_ring("chunk-aggregate", n, Lc, 16)
        return est, 16.0 * (nc + J * C), _simple_stats(None)


class _PowerSgd(_Base):
    def __init__(self, cfg: PowerSgdConfig, pipe):
        super().__init__(pipe)
        from .schemes import PowerSgdGroup
        self.cfg = cfg
        self.bypass = self.dim < cfg.bypass_below
        self.grp = None if self.bypass else PowerSgdGroup(cfg, self.n, self.L, self.dim, 1, self.seeds, self.dev)

    @property
    def warm(self):
        return None if self.grp is None or self.grp.warm is None else self.grp.warm[0]

    def sync_residuals(self, res):
        if self.grp is not None:
            self.grp.materialize(_ptr(res))

    def drop_deferred(self):
        if self.grp is not None:
            self.grp.pending = None

    def _fold(self, kind, x, m):
        """The factor all-reduce (pipelines.py:349-351, 362-364): exact fp32 FloatSum ring order,
        ring wire volume (exchange_float)."""
        return exchange_float(x.reshape(self.L, m), self.comm, self.n, kind, wire16=False).reshape(1, m)

    def run(self, g, res, r, ledger, nmse):
        L, n, d = self.L, self.n, self.dim
        sp = _sp()
        est = torch.empty(d, dtype=torch.float32, device=self.dev)
        grp = self.grp
        if grp is not None and res is not None and g.stride(0) == res.stride(0):
            # ef_apply (and the previous round's deferred EF update) fused into P = M Q when the
            # TMA pass takes this layout (pipelines.py:338-368 with ef_apply / ef_update)
            vec = bool(_native.lib().gc_psgd_vectorizable(grp.cols, g.data_ptr(), res.data_ptr(), g.stride(0)))
            grp.set_ld(g.stride(0), vec)
            if _native.lib().gc_psgd_mq_deferred_supported(ctypes.byref(grp.batch), None, d, grp.rows, grp.cols,
                                                           grp.rank, g.data_ptr(), res.data_ptr()):
                grp.run(res.data_ptr(), res.data_ptr(), est.data_ptr(), r, grads_ptr=g.data_ptr(), vec=vec,
                        fold=self._fold)
                self.launches += 6
                ledger.charge_ring("left-factor", n, grp.rows * grp.rank, 32)
                ledger.charge_ring("right-factor", n, grp.cols * grp.rank, 32)
                return est, 32.0 * grp.rank * (grp.rows + grp.cols), _simple_stats(None)
        if grp is not None:
            grp.materialize(_ptr(res))
        if res is not None:
            _native.call("gc_ef_apply", L, d, g.data_ptr(), res.data_ptr(), g.stride(0), res.data_ptr(),
                         res.stride(0), sp)
        c = res if res is not None else g
        if self.bypass:
            all_c = self.comm.all_gather_rows(c, "dense-bypass")
            _native.call("gc_float_fold", n, d, all_c.data_ptr(), d, 0, -(-d // n), 0, 0, n, est.data_ptr(), sp)
            if res is not None:
                _native.call("gc_fill_zero", res.data_ptr(), res.numel() * 4, sp)
            ledger.charge_ring("dense-bypass", n, d, 32)
            return est, 32.0 * d, _simple_stats(None)
        vec = bool(_native.lib().gc_psgd_vectorizable(grp.cols, c.data_ptr(), est.data_ptr(), c.stride(0)))
        grp.set_ld(c.stride(0), vec)
        grp.run(c.data_ptr(), _ptr(res), est.data_ptr(), r, vec=vec, fold=self._fold)
        self.launches += 11
        ledger.charge_ring("left-factor", n, grp.rows * grp.rank, 32)
        ledger.charge_ring("right-factor", n, grp.cols * grp.rank, 32)
        return est, 32.0 * grp.rank * (grp.rows + grp.cols), _simple_stats(None)


class _Dense(_Base):
    """The FP16 / FP32 NCCL all-reduce utility bar (pipelines.py:370-393 up to summation order)."""

    def __init__(self, cfg: DenseConfig, pipe):
        super().__init__(pipe)
        self.bits = cfg.bits
        self._wire = None

    def run(self, g, res, r, ledger, nmse):
        L, n, d = self.L, self.n, self.dim
        sp = _sp()
        est = torch.empty(d, dtype=torch.float32, device=self.dev)
        if self.bits == 16:
            # local workers folded with fp16 inputs / wire straight into binary16, NCCL half sum,
            # then f32 mean with the fp16 wire's +-65504 saturation (no eager casts)
            if self._wire is None:
                self._wire = torch.empty(d, dtype=torch.float16, device=self.dev)
            _native.call("gc_fold_to_half", L, d, g.data_ptr(), g.stride(0), self._wire.data_ptr(), sp)
            self.comm.all_reduce(self._wire, dist.ReduceOp.SUM, "dense")
            _native.call("gc_half_mean_sat", d, self._wire.data_ptr(), n, est.data_ptr(), sp)
        else:
            local = torch.empty(d, dtype=torch.float32, device=self.dev)
            _native.call("gc_float_fold", L, d, g.data_ptr(), g.stride(0), 0, d, 0, 0, 0, local.data_ptr(), sp)
            total = self.comm.all_reduce(local, dist.ReduceOp.SUM, "dense")
            _native.call("gc_scale_div", d, total.data_ptr(), n, est.data_ptr(), sp)
        self.launches += 2
        ledger.charge_ring("dense", n, d, self.bits)
        return est, float(self.bits) * d, _simple_stats(None)


def _make(cfg, pipe):
    if isinstance(cfg, RotatedQuantConfig):
        return _Thc(cfg, pipe)
    if isinstance(cfg, TopKConfig):
        return _TopK(cfg, pipe)
    if isinstance(cfg, ChunkedTopKConfig):
        return _Chunked(cfg, pipe)
    if isinstance(cfg, PowerSgdConfig):
        return _PowerSgd(cfg, pipe)
    if isinstance(cfg, DenseConfig):
        return _Dense(cfg, pipe)
    raise TypeError(f"unknown config type {type(cfg).__name__}")


def exchange_float_groups(phase: str | None, reqs, comm: Comm, n: int, L: int) -> list:
    """exchange_float_batched for several groups at once: reqs = [(x [T_g * L, m_g], T_g, m_g)] ->
    [[T_g, m_g]] sums, each tensor in its own reference ring order, with ONE all-to-all and ONE
    all-gather for all of them (a round's factor phase costs two collectives, not two per group).
    The send buffer per destination rank is the concatenation of every group's [T_g][L][S_g]
    slice block (S_g = ceil(m_g / W))."""
    W = comm.world
    S = [-(-m // W) for _, _, m in reqs]
    blocks = []
    for (x, T, m), Sg in zip(reqs, S):
        xv = x.reshape(T, L, m)
        if W * Sg != m:
            xp = torch.zeros(T, L, W * Sg, dtype=torch.float32, device=x.device)
            xp[:, :, :m].copy_(xv)
            xv = xp
        blocks.append(xv.reshape(T, L, W, Sg).permute(2, 0, 1, 3).reshape(W, T * L * Sg))
    send = torch.cat(blocks, dim=1).contiguous()                       # [W][sum_g T_g L S_g]
    recv = comm.all_to_all(send, phase)                                # [W][...]: every rank's workers
    outs, col = [], 0
    for (x, T, m), Sg in zip(reqs, S):
        width = T * L * Sg
        blk = recv[:, col:col + width].reshape(W, T, L, Sg)
        col += width
        if L == 1:
            rows, ld, stride = blk, recv.stride(0), Sg
        else:
            rows, ld, stride = blk.permute(1, 0, 2, 3).reshape(T, n, Sg).contiguous(), Sg, n * Sg
        s0 = comm.rank * Sg
        my_len = max(0, min(Sg, m - s0))
        out = torch.empty(T, Sg, dtype=torch.float32, device=x.device)
        if my_len < Sg:
            out[:, my_len:].zero_()
        if my_len:
            _native.call("gc_float_fold_batched_slice", T, n, my_len, rows.data_ptr(), ld, stride, s0, -(-m // n), 0,
                         0, 0, out.data_ptr(), Sg, _sp())
        outs.append(out.reshape(T * Sg))
    gathered = comm.all_gather_rows(torch.cat(outs).reshape(1, -1), phase)   # [W][sum_g T_g S_g]
    res, col = [], 0
    for (x, T, m), Sg in zip(reqs, S):
        blk = gathered[:, col:col + T * Sg]
        col += T * Sg
        if W == 1:
            res.append(blk.reshape(T, Sg))
        else:
            res.append(blk.reshape(W, T, Sg).permute(1, 0, 2).reshape(T, W * Sg)[:, :m].contiguous())
    return res


def exchange_float_batched(x: torch.Tensor, comm: Comm, n: int, T: int, m: int, phase: str | None) -> torch.Tensor:
    """T independent fp32 FloatSum rings of length m at once (one per tensor of a shape group):
    x [T * L, m] (row t * L + l = tensor t, local worker l) -> [T, m] sums in the reference ring
    order of each tensor (collectives.py:177-236), one all-to-all + one all-gather."""
    return exchange_float_groups(phase, [(x, T, m)], comm, n, x.shape[0] // T)[0]


class DistributedTensorListPipeline:
    """Chunked PowerSGD across ranks: one reference pipeline per tensor of a flat gradient
    (pipelines.py:324-368 per tensor), this rank's L = n / world workers.

    The tensors below bypass_below go through the dense-fp32 ring (pipelines.py:326-336): their
    corrected values are gathered from all ranks and folded per tensor in ring order
    (gc_segment_fold_ef), residual 0.  The compressed tensors are batched by shape as in
    TensorListPipeline (tcgen05 P = M Q with the deferred EF update); the groups run in lock step
    (PowerSgdGroup.run_steps) and each factor phase of ALL groups is one exchange_float_groups
    (all-to-all + per-tensor ring-order fold + all-gather): a round issues 4 collectives for the
    factors plus one all-gather for the bypass tensors, whatever the number of tensors and shapes."""

    def __init__(self, config: PowerSgdConfig, num_workers: int, sizes, seeds: SeedSpec,
                 error_feedback: bool | None = None, *, group=None, device=None, validate: bool = True):
        from collections import OrderedDict
        from .schemes import PowerSgdGroup
        if not isinstance(config, PowerSgdConfig):
            raise TypeError("DistributedTensorListPipeline runs PowerSGD (chunked); use DistributedGradientPipeline")
        self.comm = Comm(group)
        W = self.comm.world
        if num_workers < 1 or num_workers % W:
            raise ValueError("num_workers must be a positive multiple of the world size")
        if not sizes or min(sizes) < 1:
            raise ValueError("need positive tensor sizes")
        self.config, self.scheme = config, scheme_label(config)
        self.group = WorkerGroup(num_workers)
        self.L = num_workers // W
        self.sizes = [int(x) for x in sizes]
        self.offsets = np.concatenate([[0], np.cumsum(self.sizes)[:-1]]).astype(np.int64)
        self.dim = D = int(sum(self.sizes))
        self.seeds, self.validate = seeds, validate
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.error_feedback = True if error_feedback is None else bool(error_feedback)
        dev, L, n = self.device, self.L, num_workers
        self._res = torch.zeros(L, D, dtype=torch.float32, device=dev) if self.error_feedback else None
        self.bypass = [t for t, s in enumerate(self.sizes) if s < config.bypass_below]
        if self.bypass:
            idx = np.concatenate([np.arange(self.offsets[t], self.offsets[t] + self.sizes[t]) for t in self.bypass])
            self.byp_idx = torch.from_numpy(idx.astype(np.int64)).to(dev)
            lens = [self.sizes[t] for t in self.bypass]
            self.byp_off = torch.tensor(np.concatenate([[0], np.cumsum(lens)[:-1]]), dtype=torch.int64, device=dev)
            self.byp_len = torch.tensor(lens, dtype=torch.int64, device=dev)
        groups = OrderedDict()
        for t, s in enumerate(self.sizes):
            if s >= config.bypass_below:
                groups.setdefault(s, []).append(t)
        self.groups = []
        for s, ts in sorted(groups.items(), key=lambda kv: kv[0] * len(kv[1])):
            rows = [l * D + int(self.offsets[t]) for t in ts for l in range(L)]
            ro = torch.tensor(rows, dtype=torch.int64, device=dev)
            eo = torch.tensor([int(self.offsets[t]) for t in ts], dtype=torch.int64, device=dev)
            grp = PowerSgdGroup(config, n, L, s, len(ts), seeds, dev, row_offsets=ro, est_offsets=eo, ld=D,
                                host_offsets=[int(self.offsets[t]) for t in ts])
            grp.tensor_ids = ts
            grp.vec = grp.cols % 4 == 0 and all(x % 4 == 0 for x in rows) and D % 4 == 0
            self.groups.append(grp)
        self.launches = 0

    @property
    def residuals(self):
        if self._res is None:
            return None
        self._sync()
        h = self._res.cpu().numpy()
        return [h[i].copy() for i in range(self.L)]

    @property
    def residuals_tensor(self):
        if self._res is not None:
            self._sync()
        return self._res

    def _sync(self):
        for grp in self.groups:
            grp.materialize(self._res.data_ptr())

    def run_round(self, local_grads, round_index: int) -> RoundResult:
        from .schemes import seed_q_groups, umma_unaligned
        L, D, n = self.L, self.dim, self.group.size
        if not (torch.is_tensor(local_grads) and tuple(local_grads.shape) == (L, D)):
            raise ValueError("need [local_workers, dim] gradients")
        g = local_grads if (local_grads.is_cuda and local_grads.is_contiguous()
                            and local_grads.dtype == torch.float32) else local_grads.to(self.device, torch.float32).contiguous()
        if self.validate:
            bad = torch.zeros(1, dtype=torch.int64, device=self.device)
            _native.call("gc_check_finite", L, g.data_ptr(), g.stride(0), D, bad.data_ptr(), _sp())
            self.comm.all_reduce(bad, dist.ReduceOp.SUM)
            if int(bad.item()):
                raise ValueError("gradients must be finite")
        sp = _sp()
        res = self._res
        ledger = TrafficLedger()
        est = torch.empty(D, dtype=torch.float32, device=self.device)
        bits = 0.0
        qs = seed_q_groups(self.groups, round_index)
        if self.bypass:   # dense fp32 ring per small tensor (pipelines.py:326-336): own = corrected, r -> 0
            c = g.index_select(1, self.byp_idx)
            if res is not None:
                c += res.index_select(1, self.byp_idx)
                res.index_fill_(1, self.byp_idx, 0.0)
            allc = self.comm.all_gather_rows(c, "dense-bypass")            # [n, Dbyp], worker order
            packed = torch.empty(allc.shape[1], dtype=torch.float32, device=self.device)
            _native.call("gc_segment_fold_ef", n, len(self.bypass), self.byp_off.data_ptr(), self.byp_len.data_ptr(),
                         allc.data_ptr(), None, allc.stride(0), packed.data_ptr(), sp)
            est.index_copy_(0, self.byp_idx, packed)
            ledger.charge_rings("dense-bypass", n, [self.sizes[t] for t in self.bypass], 32)
            bits += 32.0 * sum(self.sizes[t] for t in self.bypass)
        # every group's round as a generator (PowerSgdGroup.run_steps): the groups advance in lock
        # step and each factor phase of all groups is ONE exchange (one all-to-all + one all-gather)
        steps = []
        for grp, q in zip(self.groups, qs):
            aligned = grp.vec and g.data_ptr() % 16 == 0 and est.data_ptr() % 16 == 0
            if res is not None:
                grp.set_ld(D, aligned and res.data_ptr() % 16 == 0)
                if grp.batch.rows_aligned or umma_unaligned():   # ef_apply inside the tcgen05 P = M Q
                    steps.append(grp.run_steps(res.data_ptr(), res.data_ptr(), est.data_ptr(), round_index,
                                               grads_ptr=g.data_ptr(), vec=bool(grp.batch.rows_aligned), q=q,
                                               ef_resid_ptr=res.data_ptr(), decode_phase=True))
                else:
                    grp.materialize(res.data_ptr())
                    for t in grp.tensor_ids:
                        off = int(self.offsets[t])
                        _native.call("gc_ef_apply", L, self.sizes[t], g.data_ptr() + 4 * off, res.data_ptr() + 4 * off,
                                     D, res.data_ptr() + 4 * off, D, sp)
                    steps.append(grp.run_steps(res.data_ptr(), res.data_ptr(), est.data_ptr(), round_index, vec=False,
                                               q=q, decode_phase=True))
            else:
                grp.set_ld(D, aligned)
                steps.append(grp.run_steps(g.data_ptr(), None, est.data_ptr(), round_index,
                                           vec=bool(grp.batch.rows_aligned), q=q, decode_phase=True))
            T = len(grp.tensor_ids)
            ledger.charge_ring("left-factor", n, grp.rows * grp.rank, 32, times=T)
            ledger.charge_ring("right-factor", n, grp.cols * grp.rank, 32, times=T)
            bits += 32.0 * grp.rank * (grp.rows + grp.cols) * T
        reqs = [st.send(None) for st in steps]
        while steps:
            kind = reqs[0][0]
            if kind == "decode":   # every group's warm-Q Gram is queued: now all decodes
                sums = [None] * len(steps)
            else:
                sums = exchange_float_groups(kind, [(x, x.shape[0] // L, m) for _, x, m in reqs], self.comm, n, L)
            nxt_steps, nxt_reqs = [], []
            for st, sm in zip(steps, sums):
                try:
                    nxt_reqs.append(st.send(sm))
                    nxt_steps.append(st)
                except StopIteration:
                    pass
            steps, reqs = nxt_steps, nxt_reqs
        self.launches += 4 + len(self.groups) * 11
        result = RoundResult(self.scheme, round_index, est, D, ledger, bits, _simple_stats(None))
        result.wire_bytes = dict(self.comm.sent)
        self.comm.sent = {}
        return result
