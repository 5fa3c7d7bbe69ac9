"""World-size-2 gloo tests (CPU) of the multi-GPU exchange plan: the all-to-all + ordered
saturating fold + all-gather reproduces the reference ring's saturated sums and clip counts,
and the gather-then-fold pattern keeps the reference's float ring order."""
import numpy as np
import pytest

from tests.dist_util import run_world


def _ring_fold_slice(rows, length, offset, ring_blk, bits):
    """Test-side fold of one slice in the reference ring order (collectives.py:215-226)."""
    hi = (1 << (bits - 1)) - 1
    n = rows.shape[0]
    out = np.zeros(length, dtype=np.int64)
    clips = 0
    for e in range(length):
        s = (offset + e) // ring_blk
        acc = int(rows[s, e])
        for k in range(1, n):
            acc += int(rows[(s + k) % n, e])
            c = max(-hi, min(hi, acc))
            clips += c != acc
            acc = c
        out[e] = acc
    return out, clips


def _thc_plan(rank, world, n, active, padded, bits, seed):
    import torch
    from paper_2407_01378_b200.distributed import Comm, exchange_fold, fold_slices
    comm = Comm()
    L = n // world
    rng = np.random.default_rng(seed)
    q_bound = (1 << (min(bits, 8) - 1)) - 1
    all_codes = rng.integers(-q_bound, q_bound + 1, size=(n, active)).astype(np.int8)
    mine = torch.from_numpy(all_codes[rank * L:(rank + 1) * L].copy())
    S = fold_slices(active, world, align=64)
    ring_blk = -(-padded // n)
    clips = [0]

    def fold(rows, length, offset, out):
        v, c = _ring_fold_slice(rows.numpy(), length, offset, ring_blk, bits)
        out[:length] = torch.from_numpy(v)
        clips[0] += c

    sums = exchange_fold(mine, comm, n, active, S, fold, torch.int64)
    return sums.numpy()[:active], clips[0], all_codes


@pytest.mark.parametrize("n,active,padded,bits", [(4, 5000, 8192, 4), (4, 1024, 1024, 8), (2, 777, 1024, 3),
                                                  (6, 3000, 4096, 5)])
def test_exchange_fold_matches_reference_ring(n, active, padded, bits):
    from oracle import gradcomp_oracle as orc
    res = run_world(_thc_plan, 2, (n, active, padded, bits, 17))
    (s0, c0, codes), (s1, c1, _) = res
    assert np.array_equal(s0, s1)
    sat = orc.SatCounter(bits)
    full = [np.concatenate([c.astype(np.int64), np.zeros(padded - active, np.int64)]) for c in codes]
    ref = orc.ring_fold(full, sat, dtype=np.int64)[:active]
    assert np.array_equal(s0, ref)
    assert c0 + c1 == sat.clip_events


def _gather_plan(rank, world):
    import torch
    from paper_2407_01378_b200.distributed import Comm
    comm = Comm()
    x = torch.arange(6, dtype=torch.float32).reshape(2, 3) + 100 * rank
    rows = comm.all_gather_rows(x)
    t = torch.tensor([float(rank), -float(rank)])
    from torch.distributed import ReduceOp
    comm.all_reduce(t, ReduceOp.MAX)
    return rows.numpy(), t.numpy()


def test_gather_rows_are_in_global_worker_order():
    res = run_world(_gather_plan, 2)
    rows, t = res[0]
    assert rows.tolist() == [[0, 1, 2], [3, 4, 5], [100, 101, 102], [103, 104, 105]]
    assert np.array_equal(rows, res[1][0])
    assert t.tolist() == [1.0, 0.0]
