"""Reference-pinned fixtures at BASELINE.json sizes (run where /root/reference exists).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_large.py [case ...]

Runs the REFERENCE (`gradcomp` 0.1.0, `make_pipeline(...).run_round`, pipelines.py:418-425,
147-182) on the full-size configs of SURVEY.md §8(d) and stores, per round,

  * SHA-256 of the bytes of every exact output: the estimate (f32[d]) and the stacked EF
    residuals (f32[n, d]) for THC, TopK and TopK-Chunked (bit-exact contract);
  * for PowerSGD (1e-5 contract, BLAS order differs): the estimate / residuals at a fixed set of
    sampled coordinates, their full-vector fp64 sums of squares, and the warm-start Q;
  * the RoundResult scalars (nmse, input bits, clip events, total adds, code sigma, range clips);
  * SHA-256 of every worker's input gradient, so a box-side input generator mismatch is reported
    apart from a kernel mismatch.

Inputs are regenerated at test time without the reference:
  * Gaussian configs: `SeedSpec(2024).rng("grad-worker", r, w).standard_normal(d)` as f32
    (SURVEY §8(d) cfg1/cfg2/cfg4);
  * cfg3: `trainbench.synthetic_round(SyntheticGradSpec(dim=110_000_000), SeedSpec(2024), r, 8)`
    (trainbench.py:31-113), restated in `oracle/synthetic.py` and pinned by the input hashes.

Output: tests/golden/large/<case>.json (+ <case>.npz for the PowerSGD samples).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from gradcomp.compressors import (  # noqa: E402
    ChunkedTopKConfig, PowerSgdConfig, RotatedQuantConfig, TopKConfig,
)
from gradcomp.pipelines import make_pipeline  # noqa: E402
from gradcomp.trainbench import SyntheticGradSpec, synthetic_round  # noqa: E402
from gradcomp.vectors import SeedSpec  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "large")
SEED = 2024
N_SAMPLES = 16384


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def gaussian(d, n, r):
    s = SeedSpec(SEED)
    return [s.rng("grad-worker", r, w).standard_normal(d).astype(np.float32) for w in range(n)]


def sample_index(d: int) -> np.ndarray:
    """Fixed coordinates for float fixtures: the first/last 64 plus a seeded uniform draw."""
    rng = np.random.default_rng(99)
    idx = np.concatenate([np.arange(64), np.arange(d - 64, d), rng.integers(0, d, N_SAMPLES - 128)])
    return np.unique(idx)


def gpt2_medium_sizes():
    h, v, ctx, layers = 1024, 50257, 1024, 24
    sizes = [v * h, ctx * h]
    for _ in range(layers):
        sizes += [h, h, h * 3 * h, 3 * h, h * h, h, h, h, h * 4 * h, 4 * h, 4 * h * h, h]
    return sizes + [h, h]


def scalars(res):
    return {"scheme": res.scheme, "nmse": res.nmse, "input_bits_per_coord": res.input_bits_per_coord,
            "clip_events": res.overflow.clip_events, "total_adds": res.overflow.total_adds,
            "code_sigma": res.overflow.code_sigma, "range_clips": res.range_clips}


def exact_case(name, cfg, n, d, rounds, gen, gen_label):
    pipe = make_pipeline(cfg, n, d, SeedSpec(SEED))
    meta = {"name": name, "config": repr(cfg), "n": n, "d": d, "seed": SEED, "inputs": gen_label, "rounds": []}
    for r in range(rounds):
        t0 = time.time()
        grads = gen(d, n, r)
        t1 = time.time()
        res = pipe.run_round(grads, r)
        t2 = time.time()
        est = res.estimate.logical
        rec = {"round": r, "input_sha256": [sha(g) for g in grads], "estimate_sha256": sha(est),
               "residuals_sha256": sha(np.stack(pipe.residuals)),
               "estimate_head": [float(x) for x in est[:8]], "ref_seconds": t2 - t1, "gen_seconds": t1 - t0}
        rec.update(scalars(res))
        meta["rounds"].append(rec)
        print(name, "round", r, f"gen {t1 - t0:.1f}s ref {t2 - t1:.1f}s", flush=True)
        del grads, res
    with open(os.path.join(OUT, f"{name}.json"), "w") as f:
        json.dump(meta, f, indent=1)


def powersgd_case(name, n, sizes, rounds, rank=4):
    """One reference pipeline per tensor (the 'chunked' mode of SURVEY §8(d) cfg4(b)); a single
    size is cfg4(a).  Inputs: the flat Gaussian grad-worker vector of length sum(sizes), sliced."""
    D = int(sum(sizes))
    offs = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int64)
    pipes = [make_pipeline(PowerSgdConfig(rank), n, s, SeedSpec(SEED)) for s in sizes]
    idx = sample_index(D)
    meta = {"name": name, "config": repr(PowerSgdConfig(rank)), "n": n, "d": D, "sizes": [int(s) for s in sizes],
            "seed": SEED, "inputs": "gaussian grad-worker(r, w) over the flat vector, sliced per tensor",
            "rounds": []}
    arrs = {"index": idx}
    for r in range(rounds):
        t0 = time.time()
        grads = gaussian(D, n, r)
        t1 = time.time()
        est = np.empty(D, np.float32)
        res_all = np.empty((n, D), np.float32)
        nm = []
        for p, o, s in zip(pipes, offs, sizes):
            res = p.run_round([g[o:o + s] for g in grads], r)
            est[o:o + s] = res.estimate.logical
            for w in range(n):
                res_all[w, o:o + s] = p.residuals[w]
            nm.append(res.nmse)
        t2 = time.time()
        arrs[f"estimate_{r}"] = est[idx]
        arrs[f"residuals_{r}"] = res_all[:, idx]
        big = [t for t, s in enumerate(sizes) if s >= 4096]
        # warm Q of the largest tensor (and the first compressed one when different)
        for t in sorted({max(big, key=lambda t: sizes[t]), big[0]}):
            arrs[f"warm_q_{r}_t{t}"] = pipes[t]._warm_q.copy()
        rec = {"round": r, "input_sha256": [sha(g) for g in grads],
               "estimate_sq": float(np.dot(est.astype(np.float64), est.astype(np.float64))),
               "residuals_sq": [float(np.dot(x.astype(np.float64), x.astype(np.float64))) for x in res_all],
               "nmse_per_tensor": nm, "ref_seconds": t2 - t1, "gen_seconds": t1 - t0}
        if len(sizes) == 1:
            rec.update(scalars(res))
        meta["rounds"].append(rec)
        print(name, "round", r, f"gen {t1 - t0:.1f}s ref {t2 - t1:.1f}s", flush=True)
        del grads
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **arrs)
    with open(os.path.join(OUT, f"{name}.json"), "w") as f:
        json.dump(meta, f, indent=1)


def synthetic(d, n, r):
    return synthetic_round(SyntheticGradSpec(dim=d), SeedSpec(SEED), r, n)


CASES = {
    # BASELINE.json configs[1]: THC partial rotation + saturation, ResNet-50 sized, 8 workers
    "cfg2_thc_q4b8": lambda: exact_case("cfg2_thc_q4b8", RotatedQuantConfig(4, 8, 1024), 8, 25_557_032, 2,
                                        gaussian, "gaussian grad-worker(r, w)"),
    "cfg2_thc_q4b4": lambda: exact_case("cfg2_thc_q4b4", RotatedQuantConfig(4, 4, 1024), 8, 25_557_032, 2,
                                        gaussian, "gaussian grad-worker(r, w)"),
    # configs[2]: TopK 1 % and TopK-Chunked (1 % of coordinates) on SyntheticGradSpec inputs
    "cfg3_topk": lambda: exact_case("cfg3_topk", TopKConfig(1_100_000), 8, 110_000_000, 2, synthetic,
                                    "trainbench.synthetic_round(SyntheticGradSpec(dim=d), SeedSpec(2024), r, n)"),
    "cfg3_topkc": lambda: exact_case("cfg3_topkc", ChunkedTopKConfig(64, 17_187), 8, 110_000_000, 2, synthetic,
                                     "trainbench.synthetic_round(SyntheticGradSpec(dim=d), SeedSpec(2024), r, n)"),
    # configs[3]: PowerSGD rank 4 at 350M (one 18,709 x 18,708 matrix) and GPT-2-medium's tensors
    "cfg4_psgd": lambda: powersgd_case("cfg4_psgd", 2, [350_000_000], 2),
    "gpt2_psgd": lambda: powersgd_case("gpt2_psgd", 2, gpt2_medium_sizes(), 2),
}


def main():
    os.makedirs(OUT, exist_ok=True)
    names = sys.argv[1:] or list(CASES)
    for nm in names:
        CASES[nm]()


if __name__ == "__main__":
    main()
