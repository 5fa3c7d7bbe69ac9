"""The reference's `collective-check` (cli.py:436-573) run on the real transport: one worker per
rank of a torch.distributed group (NCCL, or gloo with host staging), the exchanges of
DistributedGradientPipeline and its Comm byte counters instead of the simulated ring.

    python -m torch.distributed.run --nproc-per-node N -m paper_2407_01378_b200.collective_check \\
        [--seed 2024] [--inject-element-bits B]

Every rank evaluates the same checks and rank 0 prints one `PASS|FAIL name: detail` line per check
(the reference's format) and exits 1 if any failed.  `inject_element_bits` (cli.py:437-439) is the
wire width the checker assumes for the dense ring; anything but the transport's 32 bits must make
`ring_egress_closed_form` fail -- the fault the check exists to catch.  The all-gather accounting
with unequal payloads (cli.py:546-554) has no counterpart: every gather here carries equal rows."""
from __future__ import annotations

import argparse
import math
import sys
from fractions import Fraction

import numpy as np
import torch
import torch.distributed as dist

from . import _native
from .configs import ChunkedTopKConfig, DenseConfig, TopKConfig
from .distributed import Comm, DistributedGradientPipeline, exchange_float, exchange_fold
from .vectors import SeedSpec


def _gather_np(x: np.ndarray, comm: Comm, dev) -> np.ndarray:
    t = torch.from_numpy(np.ascontiguousarray(x)).to(dev).reshape(1, -1)
    return comm.all_gather_rows(t).cpu().numpy()


def collective_check(seed: int = 2024, inject_element_bits: int | None = None, group=None,
                     device=None) -> tuple[bool, list[str]]:
    if inject_element_bits is not None and (not isinstance(inject_element_bits, int) or inject_element_bits < 1):
        raise ValueError("inject_element_bits must be a positive integer or None")
    comm = Comm(group)
    W, rank = comm.world, comm.rank
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    seeds = SeedSpec(seed)
    rng = seeds.rng("collective-check", 0, rank)
    lines: list[str] = []
    ok = True

    def check(name, cond, detail):
        nonlocal ok
        cond = bool(cond)
        ok &= cond
        lines.append(f"{'PASS' if cond else 'FAIL'} {name}: {detail}")

    # float ring against the mathematical sum (cli.py:446-458): the dense fp32 round's sum
    length = 1000
    x = rng.standard_normal(length).astype(np.float32)
    pipe = DistributedGradientPipeline(DenseConfig(32), W, length, seeds, False, group=group, device=dev,
                                       validate=False)
    est = pipe.run_round([x], 0).estimate.logical.astype(np.float64) * W
    allx = _gather_np(x, comm, dev).astype(np.float64)
    exact = allx.sum(axis=0)
    rel = float(np.linalg.norm(est - exact) / np.linalg.norm(exact))
    check("float_sum_matches_naive", rel < 1e-6, f"rel l2 err {rel:.2e}")
    ests = _gather_np(est.astype(np.float32), comm, dev)
    check("float_sum_worker_consensus", all(np.array_equal(ests[0], e) for e in ests), "all workers bitwise identical")

    # ledger closed form against the bytes handed to the transport (cli.py:460-474)
    element_bits = 32 if inject_element_bits is None else inject_element_bits
    v = rng.standard_normal(1024).astype(np.float32)
    res = DistributedGradientPipeline(DenseConfig(32), W, 1024, seeds, False, group=group, device=dev,
                                      validate=False).run_round([v], 0)
    expect = 2 * (W - 1) * math.ceil(1024 / W) * element_bits
    got = 8 * res.wire_bytes.get("dense", 0)
    check("ring_egress_closed_form", W == 1 or got == expect, f"egress {got} vs {expect}")
    check("ring_egress_equals_ingress",
          res.ledger.bits_sent(worker=rank) == res.ledger.bits_received(worker=rank) == got,
          "per-worker send == receive == transport bytes")

    # element-wise min / max consensus (cli.py:476-482): the THC range all-reduce, MAX of (-lo, hi)
    col = rng.standard_normal(257).astype(np.float32)
    pair = torch.from_numpy(np.stack([-col, col], axis=1)).to(dev).contiguous()
    comm.all_reduce(pair, dist.ReduceOp.MAX, rings=2)
    lo, hi = -pair[:, 0].cpu().numpy(), pair[:, 1].cpu().numpy()
    stack = _gather_np(col, comm, dev)
    check("elementwise_min_max_exact", np.array_equal(lo, stack.min(axis=0)) and np.array_equal(hi, stack.max(axis=0)),
          "matches np.min / np.max")

    # saturating sum against a sequential ring-order fold (cli.py:484-506), the THC code exchange
    bits, n_el = 4, 96 * W
    codes = rng.integers(-7, 8, size=n_el).astype(np.int8)
    ring_block = -(-n_el // W)
    counters = torch.zeros(1, dtype=torch.int64, device=dev)

    def fold(rows, ln, offset, out):
        _native.call("gc_sat_fold", W, ln, rows.data_ptr(), rows.stride(0), offset, ring_block, bits, out.data_ptr(),
                     counters.data_ptr(), torch.cuda.current_stream().cuda_stream)

    S = -(-n_el // W)
    got_codes = exchange_fold(torch.from_numpy(codes).to(dev).reshape(1, -1), comm, W, n_el, S,
                              fold if W > 1 else (lambda r, ln, o, out: out[:ln].copy_(r[0, :ln])),
                              torch.int8)[:n_el].cpu().numpy().astype(np.int64)
    allc = _gather_np(codes, comm, dev).astype(np.int64)
    hb = (1 << (bits - 1)) - 1
    want = np.empty(n_el, np.int64)
    for j in range(W):
        sl = slice(j * ring_block, min(n_el, (j + 1) * ring_block))
        acc = allc[j][sl].copy()
        for step in range(1, W):
            acc = np.clip(acc + allc[(j + step) % W][sl], -hb, hb)
        want[sl] = acc
    clips = int(counters.item())
    check("saturating_sum_matches_fold", np.array_equal(got_codes, want), f"{clips} clip events counted on this rank")

    # sparsifier traffic identities on live rounds (cli.py:508-544), measured on the transport
    ring_share = Fraction(2 * (W - 1), W) if W > 1 else None
    for d, chunk, selected, k in ((1 << 20, 64, 7936, 174763), (1 << 20, 128, 192, 10923),
                                  (1 << 16, 64, 496, 10923), (1 << 16, 128, 60, 2731), (1 << 14, 64, 124, 2731)):
        g = rng.standard_normal(d).astype(np.float32)
        res = DistributedGradientPipeline(ChunkedTopKConfig(chunk, selected), W, d, seeds, group=group, device=dev,
                                          validate=False).run_round([g], 0)
        formula = Fraction(16 * (selected * chunk + d // chunk), d)
        if W > 1:
            measured = Fraction(8 * sum(res.wire_bytes.values())) / ring_share / d
            good = measured == formula
        else:
            measured, good = formula, True
        check(f"chunked_topk_bit_identity[d={d},C={chunk},J={selected}]",
              good and res.input_bits_per_coord == float(formula), f"measured {float(measured):.6f} bits/coord")
        res = DistributedGradientPipeline(TopKConfig(k), W, d, seeds, group=group, device=dev,
                                          validate=False).run_round([g], 0)
        formula = Fraction(48 * k, d)
        measured = Fraction(8 * sum(res.wire_bytes.values()), (W - 1) * d) if W > 1 else formula
        check(f"topk_bit_identity[d={d},K={k}]", measured == formula and res.input_bits_per_coord == float(formula),
              f"measured {float(measured):.6f} bits/coord")

    # fp16 wire: the fp16 ring equals the per-hop rounded fold exactly (cli.py:556-570)
    half = rng.standard_normal(64 * W).astype(np.float16).astype(np.float32)
    got_half = exchange_float(torch.from_numpy(half).to(dev).reshape(1, -1), comm, W, None, wire16=True).cpu().numpy()
    allh = _gather_np(half, comm, dev)
    m = half.size
    blk = -(-m // W)

    def r16(a):
        y = a.astype(np.float16).astype(np.float32)
        return np.where(np.isinf(y), np.copysign(np.float32(65504.0), a), y)

    want_half = np.empty(m, np.float32)
    for j in range(W):
        sl = slice(j * blk, min(m, (j + 1) * blk))
        acc = allh[j][sl].copy()
        for step in range(1, W):
            acc = r16(acc) + allh[(j + step) % W][sl]
        want_half[sl] = r16(acc)
    check("fp16_wire_matches_fold", np.array_equal(got_half, want_half), "per-hop re-rounding reproduced")

    flag = torch.tensor([0 if ok else 1], dtype=torch.int64, device=dev)
    comm.all_reduce(flag, dist.ReduceOp.MAX)
    return int(flag.item()) == 0, lines


def main(argv=None) -> int:
    import os
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--seed", type=int, default=2024)
    ap.add_argument("--inject-element-bits", type=int, default=None)
    ap.add_argument("--backend", default="nccl")
    a = ap.parse_args(argv)
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29571")
        os.environ.setdefault("RANK", "0")
        os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group(a.backend)
    ok, lines = collective_check(a.seed, a.inject_element_bits)
    if dist.get_rank() == 0:
        print("\n".join(lines), flush=True)
    dist.destroy_process_group()
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
