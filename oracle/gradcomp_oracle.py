"""CPU oracle for the compress -> aggregate -> decompress path (TEST INFRASTRUCTURE ONLY).

This module is a NumPy restatement of the reference package `gradcomp`
(/root/reference/pkg/src/gradcomp, v0.1.0).  It exists to check the CUDA path:
only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
leg may import it, and never as the thing measured or shipped.  The product path
(paper_2407_01378_b200) must never import it.

Parity pinning: tests/test_oracle_golden.py checks every function here against
golden vectors produced by the reference itself (tests/golden/make_golden.py,
run in the container that holds /root/reference).

Third-party algorithms used by the reference and restated / reused here:
  * numpy 2.3.5 PCG64 + SeedSequence (`np.random.PCG64(seed)`), Generator.random,
    Generator.integers(0, 2) (Lemire on buffered u32 halves), Generator.standard_normal
    (ziggurat) -- used through numpy itself, plus the pure-integer restatement
    `pcg64_state_from_seed` / `pcg64_next` pinned against numpy in the tests;
  * numpy pairwise float64 summation (chunk energies), stable argsort (top-k), IEEE
    binary16 casts (fp16 wire), OpenBLAS sgemm (PowerSGD; pinned to tolerance only).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# ----------------------------------------------------------------------------
# seeding (vectors.py:17-76)

MASK64 = (1 << 64) - 1
MASK128 = (1 << 128) - 1
HALF_MAX = 65504.0                       # vectors.py:19
PCG_MULT = 0x2360ED051FC65DA44385DF649FCCF645


def splitmix64(value: int) -> int:
    """vectors.py:26-31."""
    z = (value + 0x9E3779B97F4A7C15) & MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def fnv1a64(text: str) -> int:
    """vectors.py:34-39."""
    h = 0xCBF29CE484222325
    for byte in text.encode("utf-8"):
        h = ((h ^ byte) * 0x100000001B3) & MASK64
    return h


def stream_seed(experiment_seed: int, tag: str, round_index: int = 0, worker: int | None = None) -> int:
    """SeedSpec.stream_seed, vectors.py:64-73."""
    h = splitmix64((experiment_seed ^ fnv1a64(tag)) & MASK64)
    h = splitmix64(h ^ round_index)
    if worker is not None:
        h = splitmix64(h ^ ((worker + 0x517CC1B727220A95) & MASK64))
    return h


def stream_rng(experiment_seed: int, tag: str, round_index: int = 0, worker: int | None = None):
    """SeedSpec.rng, vectors.py:75-76."""
    return np.random.Generator(np.random.PCG64(stream_seed(experiment_seed, tag, round_index, worker)))


def pcg64_state_from_seed(seed: int) -> tuple[int, int]:
    """Integer restatement of numpy's SeedSequence(seed) -> PCG64 seeding (numpy 2.3)."""
    m32 = 0xFFFFFFFF
    words = [0] if seed == 0 else []
    while seed:
        words.append(seed & m32)
        seed >>= 32
    hash_const = [0x43B0D7E5]

    def hashmix(v):
        v = (v ^ hash_const[0]) & m32
        hash_const[0] = (hash_const[0] * 0x931E8875) & m32
        v = (v * hash_const[0]) & m32
        return v ^ (v >> 16)

    def mix(x, y):
        r = (0xCA01F9DD * x - 0x4973F715 * y) & m32
        return r ^ (r >> 16)

    pool = [hashmix(words[i] if i < len(words) else 0) for i in range(4)]
    for s in range(4):
        for d in range(4):
            if s != d:
                pool[d] = mix(pool[d], hashmix(pool[s]))
    hb = 0x8B51F9DD
    out = []
    for i in range(8):
        v = (pool[i % 4] ^ hb) & m32
        hb = (hb * 0x58F38DED) & m32
        v = (v * hb) & m32
        out.append(v ^ (v >> 16))
    w = [out[2 * i] | (out[2 * i + 1] << 32) for i in range(4)]
    initstate, initseq = (w[0] << 64) | w[1], (w[2] << 64) | w[3]
    inc = ((initseq << 1) | 1) & MASK128
    state = inc                                   # step from 0
    state = (state + initstate) & MASK128
    state = (state * PCG_MULT + inc) & MASK128
    return state, inc


def pcg64_next(state: int, inc: int) -> tuple[int, int]:
    """One numpy pcg64_next64: step then XSL-RR output."""
    state = (state * PCG_MULT + inc) & MASK128
    hi, lo = state >> 64, state & MASK64
    x, rot = hi ^ lo, hi >> 58
    return state, ((x >> rot) | (x << ((64 - rot) & 63))) & MASK64


# ----------------------------------------------------------------------------
# elementary codecs

def next_pow2(n: int) -> int:
    """vectors.py:79-80 / pipelines.py:400-401."""
    return 1 << (n - 1).bit_length()


def fp16_round_trip(x) -> np.ndarray:
    """vectors.py:136-152: RNE to binary16, overflow saturates to +-65504."""
    arr = np.asarray(x, dtype=np.float32)
    with np.errstate(over="ignore"):
        out = arr.astype(np.float16).astype(np.float32)
    inf = np.isinf(out)
    if inf.any():
        out = np.where(inf, np.copysign(np.float32(HALF_MAX), arr), out)
    return out


def rotation_signs(experiment_seed: int, round_index: int, padded: int) -> np.ndarray:
    """RotationSpec.for_round signs, transforms.py:80-82 (+1 / -1 as float32)."""
    rng = stream_rng(experiment_seed, "rotation-signs", round_index)
    return rng.integers(0, 2, size=padded).astype(np.float32) * 2.0 - 1.0


def rotation_block(padded: int, max_block: int) -> int:
    """depth_used = min(depth_full, log2(max_block)), transforms.py:78-79."""
    return 1 << min(padded.bit_length() - 1, max_block.bit_length() - 1)


def wht_rows(rows: np.ndarray) -> np.ndarray:
    """Unnormalised Sylvester WHT along axis 1, stage width 1, 2, 4, ... (transforms.py:86-99)."""
    m, blk = rows.shape
    width = 1
    while width < blk:
        r = rows.reshape(m, blk // (2 * width), 2, width)
        rows = np.stack((r[:, :, 0] + r[:, :, 1], r[:, :, 0] - r[:, :, 1]), axis=2).reshape(m, blk)
        width *= 2
    return rows


def rht_forward(values: np.ndarray, signs: np.ndarray, block: int) -> np.ndarray:
    """transforms.py:107-117: f32(WHT_B(f64(v) * signs) * B^-0.5)."""
    work = np.asarray(values, dtype=np.float32).astype(np.float64) * signs.astype(np.float64)
    work = wht_rows(work.reshape(-1, block))
    work *= float(block) ** -0.5
    return work.reshape(-1).astype(np.float32)


def rht_inverse(values: np.ndarray, signs: np.ndarray, block: int) -> np.ndarray:
    """transforms.py:120-126: f32(WHT_B(f64(v)) * B^-0.5 * signs)."""
    work = wht_rows(np.asarray(values, dtype=np.float32).astype(np.float64).reshape(-1, block))
    work *= float(block) ** -0.5
    return (work.reshape(-1) * signs.astype(np.float64)).astype(np.float32)


def chunk_ranges(values: np.ndarray, block: int) -> np.ndarray:
    """compressors.py:447-453."""
    b = np.asarray(values, dtype=np.float32).reshape(-1, block)
    return np.stack([b.min(axis=1), b.max(axis=1)], axis=1)


def quantize_stochastic(values, ranges, quant_bits, rng):
    """compressors.py:456-498 -> (int8 codes, clamp count)."""
    v = np.asarray(values, dtype=np.float64)
    per = v.size // ranges.shape[0]
    lo = np.repeat(ranges[:, 0].astype(np.float64), per)
    hi = np.repeat(ranges[:, 1].astype(np.float64), per)
    bound = float((1 << (quant_bits - 1)) - 1)
    cl = np.clip(v, lo, hi)
    clamped = int(np.count_nonzero(cl != v))
    mid = (lo + hi) / 2.0
    step = (hi - lo) / float((1 << quant_bits) - 2)
    degenerate = step <= 0.0
    t = np.clip((cl - mid) / np.where(degenerate, 1.0, step), -bound, bound)
    low = np.floor(t)
    frac = t - low
    near_one = frac > 1.0 - 1e-9
    low[near_one] += 1.0
    frac = np.where((frac < 1e-9) | near_one, 0.0, frac)
    coins = rng.random(t.size)
    z = np.clip((low + (coins < frac)).astype(np.int64), -int(bound), int(bound))
    z[degenerate] = 0
    return z.astype(np.int8), clamped


def dequantize_sum(code_sums, ranges, quant_bits, addends) -> np.ndarray:
    """compressors.py:501-521: f32(n*mu + delta*z)."""
    s = np.asarray(code_sums, dtype=np.float64)
    per = s.size // ranges.shape[0]
    lo = np.repeat(ranges[:, 0].astype(np.float64), per)
    hi = np.repeat(ranges[:, 1].astype(np.float64), per)
    mid = (lo + hi) / 2.0
    step = np.where(hi > lo, (hi - lo) / float((1 << quant_bits) - 2), 0.0)
    return (addends * mid + step * s).astype(np.float32)


def topk_indices(values: np.ndarray, k: int) -> np.ndarray:
    """compressors.py:387-396: largest |x|, lower index on ties, ascending."""
    order = np.argsort(-np.abs(np.asarray(values)), kind="stable")
    return np.sort(order[:k])


def chunk_sq_norms(values: np.ndarray, chunk: int) -> np.ndarray:
    """vectors.py:180-192 (fp64, numpy pairwise summation per chunk)."""
    v = np.asarray(values, dtype=np.float32)
    nc = math.ceil(v.size / chunk)
    buf = np.zeros(nc * chunk, dtype=np.float64)
    buf[: v.size] = v
    return (buf.reshape(nc, chunk) ** 2).sum(axis=1)


def pairwise_sum(a) -> float:
    """Scalar restatement of numpy's float64 pairwise summation (used to pin the GPU order)."""
    n = len(a)
    if n < 8:
        res = 0.0
        for x in a:
            res += float(x)
        return res
    if n <= 128:
        r = [float(x) for x in a[:8]]
        i = 8
        while i < n - (n % 8):
            for j in range(8):
                r[j] += float(a[i + j])
            i += 8
        res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
        while i < n:
            res += float(a[i])
            i += 1
        return res
    n2 = n // 2
    n2 -= n2 % 8
    return pairwise_sum(a[:n2]) + pairwise_sum(a[n2:])


def matrix_shape_for(size: int) -> tuple[int, int]:
    """compressors.py:530-538."""
    rows = math.isqrt(size)
    if rows * rows < size:
        rows += 1
    return rows, math.ceil(size / rows)


def orthonormalize(mat: np.ndarray) -> np.ndarray:
    """fp64 modified Gram-Schmidt with canonical completion, compressors.py:555-588."""
    a = np.asarray(mat, dtype=np.float64).copy()
    rows, cols = a.shape
    scale = float(np.linalg.norm(a)) / max(1.0, math.sqrt(cols))
    floor = max(scale * 1e-8, 1e-300)
    for c in range(cols):
        col = a[:, c]
        for p in range(c):
            col -= (a[:, p] @ col) * a[:, p]
        nrm = float(np.linalg.norm(col))
        if nrm > floor:
            col /= nrm
            continue
        for basis in range(rows):
            cand = np.zeros(rows)
            cand[basis] = 1.0
            for p in range(c):
                cand -= (a[:, p] @ cand) * a[:, p]
            nrm = float(np.linalg.norm(cand))
            if nrm > 0.5:
                a[:, c] = cand / nrm
                break
        else:
            raise ValueError("could not complete an orthonormal basis")
    return a.astype(np.float32)


def ensure_full_rank(q, cols, rank, rng, attempts=3):
    """compressors.py:595-603."""
    cand = q
    for remaining in range(attempts, -1, -1):
        if np.linalg.matrix_rank(cand) == rank:
            return np.ascontiguousarray(cand, dtype=np.float32)
        if remaining:
            cand = rng.standard_normal((cols, rank)).astype(np.float32)
    raise ValueError("seed matrix rank-deficient after redraws")


# ----------------------------------------------------------------------------
# ring collective semantics (collectives.py:177-236)

def ring_fold(inputs, combine, wire=None, neutral=0, dtype=np.float32):
    """Block j of the (n-padded) vector starts at worker j and folds in ring order;
    `wire` rounds every transmitted partial and the final value (collectives.py:215-235)."""
    n = len(inputs)
    length = np.asarray(inputs[0]).size
    if n == 1:
        return np.array(inputs[0], dtype=dtype, copy=True)
    blk = -(-length // n)
    bufs = []
    for x in inputs:
        b = np.full(blk * n, neutral, dtype=dtype)
        b[:length] = x
        bufs.append(b)
    out = np.empty(blk * n, dtype=dtype)
    for j in range(n):
        sl = slice(j * blk, (j + 1) * blk)
        acc = bufs[j][sl].copy()
        for step in range(1, n):
            acc = combine(acc if wire is None else wire(acc), bufs[(j + step) % n][sl])
        out[sl] = acc if wire is None else wire(acc)
    return out[:length]


def float_sum(a, b):
    return (a + b).astype(np.float32)


class SatCounter:
    """SatIntSum (collectives.py:123-143) with clip / add counters."""

    def __init__(self, bits):
        self.hi = (1 << (bits - 1)) - 1
        self.clip_events = 0
        self.total_adds = 0

    def __call__(self, a, b):
        s = a + b
        c = np.clip(s, -self.hi, self.hi)
        self.clip_events += int(np.count_nonzero(c != s))
        self.total_adds += int(s.size)
        return c


# ----------------------------------------------------------------------------
# scheme rounds (pipelines.py:201-393); each returns a dict of outputs

@dataclass
class OracleState:
    """Cross-round state of GradientPipeline (pipelines.py:129-134)."""

    residuals: list | None
    warm_q: np.ndarray | None = None
    extras: dict = field(default_factory=dict)


def _padded(c, length):
    out = np.zeros(length, dtype=np.float32)
    out[: c.size] = c
    return out


def thc_round(corrected, seed, round_index, quant_bits, wire_bits, max_block):
    """pipelines.py:260-322."""
    n, d = len(corrected), corrected[0].size
    P = next_pow2(d)
    B = rotation_block(P, max_block)
    signs = rotation_signs(seed, round_index, P)
    rotated = [rht_forward(_padded(c, P), signs, B) for c in corrected]
    ranges = [chunk_ranges(r, B) for r in rotated]
    lo = ring_fold([r[:, 0] for r in ranges], np.minimum)
    hi = ring_fold([r[:, 1] for r in ranges], np.maximum)
    shared = np.stack([lo, hi], axis=1)
    codes, range_clips = [], 0
    for w, r in enumerate(rotated):
        z, k = quantize_stochastic(r, shared, quant_bits, stream_rng(seed, "stochastic-round", round_index, w))
        codes.append(z)
        range_clips += k
    sat = SatCounter(wire_bits)
    sums = ring_fold([z.astype(np.int64) for z in codes], sat, dtype=np.int64)
    agg = dequantize_sum(sums, shared, quant_bits, n)
    estimate = rht_inverse(agg, signs, B)[:d] / np.float32(n)
    own = [rht_inverse(dequantize_sum(z, shared, quant_bits, 1), signs, B)[:d] for z in codes]
    sigma = float(np.std(np.concatenate(codes).astype(np.float64)))
    return dict(estimate=estimate, own=own, input_bits=float(wire_bits * P + 64 * shared.shape[0]),
                clip_events=sat.clip_events, total_adds=sat.total_adds, code_sigma=sigma,
                range_clips=range_clips, signs=signs, rotated=rotated, ranges=ranges, shared=shared,
                codes=codes, sums=sums, block=B, padded=P)


def topk_round(corrected, k):
    """pipelines.py:201-211."""
    n, d = len(corrected), corrected[0].size
    payloads = []
    for c in corrected:
        idx = topk_indices(c, k).astype(np.int32)
        payloads.append((idx, fp16_round_trip(c[idx])))
    est = np.zeros(d, dtype=np.float32)
    for idx, val in payloads:
        np.add.at(est, idx, val)
    est /= np.float32(n)
    own = []
    for idx, val in payloads:
        o = np.zeros(d, dtype=np.float32)
        o[idx] = val
        own.append(o)
    return dict(estimate=est, own=own, input_bits=float(48 * k), payloads=payloads)


def chunked_round(corrected, chunk, num_selected, perm=None):
    """pipelines.py:213-258 (perm: optional shared coordinate permutation)."""
    n, d = len(corrected), corrected[0].size
    work = [c[perm] if perm is not None else c for c in corrected]
    nc = math.ceil(d / chunk)
    norms = [fp16_round_trip(chunk_sq_norms(w, chunk).astype(np.float32)) for w in work]
    energy = ring_fold(norms, float_sum, wire=fp16_round_trip)
    selected = topk_indices(energy, num_selected)
    packs = []
    for w in work:
        buf = np.zeros(nc * chunk, dtype=np.float32)
        buf[:d] = w
        packs.append(fp16_round_trip(buf.reshape(nc, chunk)[selected].reshape(-1)))
    summed = ring_fold(packs, float_sum, wire=fp16_round_trip)

    def scatter(vals):
        buf = np.zeros((nc, chunk), dtype=np.float32)
        buf[selected] = vals.reshape(-1, chunk)
        return buf.reshape(-1)[:d].copy()

    est = scatter(summed)
    est /= np.float32(n)
    own = [scatter(p) for p in packs]
    if perm is not None:
        def back(x):
            out = np.zeros_like(x)
            out[perm] = x
            return out
        est, own = back(est), [back(o) for o in own]
    return dict(estimate=est, own=own, input_bits=16.0 * (nc + num_selected * chunk), norms=norms,
                energy=energy, selected=selected, summed=summed)


def powersgd_round(corrected, seed, round_index, rank, warm_q, warm_start=True, bypass_below=4096):
    """pipelines.py:324-368; returns the new warm Q in 'warm_q'."""
    n, d = len(corrected), corrected[0].size
    if d < bypass_below:
        summed = ring_fold(list(corrected), float_sum)
        return dict(estimate=summed / np.float32(n), own=list(corrected), input_bits=32.0 * d,
                    warm_q=warm_q, bypass=True)
    rows, cols = matrix_shape_for(d)
    mats = [_padded(c, rows * cols).reshape(rows, cols) for c in corrected]
    rng = stream_rng(seed, "lowrank-seed", round_index)
    if warm_start and warm_q is not None:
        q = warm_q
    else:
        q = rng.standard_normal((cols, rank)).astype(np.float32)
    q = ensure_full_rank(q, cols, rank, rng)
    lefts = [(m @ q).reshape(-1) for m in mats]
    left_sum = ring_fold(lefts, float_sum)
    p_hat = orthonormalize(left_sum.reshape(rows, rank))
    rights = [m.T @ p_hat for m in mats]
    own = [(p_hat @ r.T).reshape(-1)[:d].copy() for r in rights]
    right_sum = ring_fold([r.reshape(-1) for r in rights], float_sum).reshape(cols, rank)
    est = (p_hat @ right_sum.T).reshape(-1)[:d] / np.float32(n)
    new_q = (right_sum / np.float32(n)).astype(np.float32)
    return dict(estimate=est, own=own, input_bits=32.0 * rank * (rows + cols), warm_q=new_q, seed_q=q,
                p_hat=p_hat, left_sum=left_sum, right_sum=right_sum, bypass=False)


def dense_round(corrected, bits):
    """pipelines.py:370-393."""
    n, d = len(corrected), corrected[0].size
    if bits == 16:
        summed = ring_fold([fp16_round_trip(c) for c in corrected], float_sum, wire=fp16_round_trip)
    else:
        summed = ring_fold(list(corrected), float_sum)
    return dict(estimate=summed / np.float32(n), own=list(corrected), input_bits=float(bits) * d)


def nmse(estimate, reference) -> float:
    """metrics.py:22-37."""
    est = np.asarray(estimate, dtype=np.float64)
    ref = np.asarray(reference, dtype=np.float64)
    den = float(ref @ ref)
    err = est - ref
    num = float(err @ err)
    if den == 0.0:
        return 0.0 if num == 0.0 else math.inf
    return num / den


def run_round(scheme: str, params: dict, state: OracleState, grads, seed: int, round_index: int) -> dict:
    """GradientPipeline.run_round (pipelines.py:147-182) for one scheme.

    scheme in {"rotated_quant", "topk", "chunked_topk", "powersgd", "dense"};
    params carry the config fields.  Residuals in `state` are updated in place."""
    grads = [np.asarray(g, dtype=np.float32) for g in grads]
    if state.residuals is not None:
        corrected = [(g + r).astype(np.float32) for g, r in zip(grads, state.residuals)]   # ef_apply
    else:
        corrected = grads
    if scheme == "rotated_quant":
        out = thc_round(corrected, seed, round_index, params["quant_bits"], params["wire_bits"],
                        params.get("rotation_block", 1024))
    elif scheme == "topk":
        out = topk_round(corrected, params["k"])
    elif scheme == "chunked_topk":
        perm = None
        if params.get("permute"):
            perm = stream_rng(seed, "coordinate-permutation", round_index).permutation(corrected[0].size)
        out = chunked_round(corrected, params["chunk_size"], params["chunks_selected"], perm)
    elif scheme == "powersgd":
        out = powersgd_round(corrected, seed, round_index, params["rank"], state.warm_q,
                             params.get("warm_start", True), params.get("bypass_below", 4096))
        if not out["bypass"]:
            state.warm_q = out["warm_q"]
    elif scheme == "dense":
        out = dense_round(corrected, params["bits"])
    else:
        raise ValueError(scheme)
    if state.residuals is not None:
        state.residuals = [(c - o).astype(np.float32) for c, o in zip(corrected, out["own"])]  # ef_update
    ref = np.mean(np.stack(corrected), axis=0, dtype=np.float64)
    out["nmse"] = nmse(out["estimate"], ref)
    out["corrected"] = corrected
    return out
