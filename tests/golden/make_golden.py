"""Generate golden vectors from the REFERENCE implementation (run where /root/reference exists).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/*.npz and seeds.json.  Every array comes from the reference's own
public API (gradcomp 0.1.0): GradientPipeline.run_round for whole rounds, and the codec
functions it calls (RotationSpec.for_round, rht_forward, chunk_ranges, quantize_stochastic,
ring_all_reduce, ...) for THC intermediates.  These fixtures pin the oracle
(oracle/gradcomp_oracle.py) and the GPU path; nothing at test time reads /root/reference.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import gradcomp  # noqa: E402
from gradcomp import compressors as comp  # noqa: E402
from gradcomp.collectives import ElemMax, ElemMin, SatIntSum, WorkerGroup, ring_all_reduce  # noqa: E402
from gradcomp.compressors import (  # noqa: E402
    ChunkedTopKConfig, DenseConfig, PowerSgdConfig, RotatedQuantConfig, TopKConfig,
)
from gradcomp.pipelines import make_pipeline  # noqa: E402
from gradcomp.transforms import RotationSpec, rht_forward, rht_inverse  # noqa: E402
from gradcomp.vectors import GradientVector, SeedSpec, chunk_sq_norms, ChunkGeometry, fnv1a64, splitmix64  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def quarters(rng, n):
    return (rng.integers(-32, 33, n) / 4.0).astype(np.float32)


def run_case(name, cfg, n, d, seed, rounds, gen, error_feedback=None):
    seeds = SeedSpec(seed)
    pipe = make_pipeline(cfg, n, d, seeds, error_feedback)
    rng = np.random.default_rng(seed + 7)
    arrs = {}
    meta = {"name": name, "n": n, "d": d, "seed": seed, "rounds": rounds, "config": repr(cfg),
            "error_feedback": pipe.error_feedback}
    stats = []
    for r in range(rounds):
        grads = [gen(rng, d, w) for w in range(n)]
        arrs[f"grads_{r}"] = np.stack(grads)
        res = pipe.run_round(grads, r)
        arrs[f"estimate_{r}"] = res.estimate.logical.copy()
        arrs[f"estimate_padded_{r}"] = res.estimate.values.copy()
        if pipe.residuals is not None:
            arrs[f"residuals_{r}"] = np.stack(pipe.residuals)
        if pipe._warm_q is not None:
            arrs[f"warm_q_{r}"] = pipe._warm_q.copy()
        ledger = {ph: [[res.ledger.bits_sent(worker=w, phase=ph), res.ledger.bits_received(worker=w, phase=ph)]
                       for w in range(n)] for ph in res.ledger.phases()}
        stats.append({"round": r, "scheme": res.scheme, "nmse": res.nmse,
                      "input_bits_per_coord": res.input_bits_per_coord,
                      "clip_events": res.overflow.clip_events, "total_adds": res.overflow.total_adds,
                      "code_sigma": res.overflow.code_sigma, "range_clips": res.range_clips,
                      "ledger": ledger, "max_egress_bits": res.ledger.max_egress_bits()})
    meta["stats"] = stats
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), meta=json.dumps(meta), **arrs)
    print(name, "ok", [round(s["nmse"], 6) for s in stats])


def thc_intermediates(name, n, d, seed, r, q, b, max_block):
    """The _round_quant call sequence (pipelines.py:260-322) via the reference's functions."""
    seeds = SeedSpec(seed)
    rng = np.random.default_rng(seed + 11)
    corrected = [rng.standard_normal(d).astype(np.float32) for _ in range(n)]
    P = 1 << (d - 1).bit_length()
    spec = RotationSpec.for_round(seeds, r, P, max_block=max_block)
    group = WorkerGroup(n)
    rotated = []
    for c in corrected:
        buf = np.zeros(P, dtype=np.float32)
        buf[:d] = c
        rotated.append(rht_forward(GradientVector(buf, d), spec).values)
    ranges = [comp.chunk_ranges(x, spec.block_size) for x in rotated]
    lo = ring_all_reduce([x[:, 0] for x in ranges], ElemMin(), group)[0]
    hi = ring_all_reduce([x[:, 1] for x in ranges], ElemMax(), group)[0]
    shared = np.stack([lo, hi], axis=1)
    codes, clamps = [], []
    for i, x in enumerate(rotated):
        z, k = comp.quantize_stochastic(x, shared, q, seeds.rng("stochastic-round", r, i))
        codes.append(z)
        clamps.append(k)
    op = SatIntSum(b)
    sums = ring_all_reduce(codes, op, group, element_bits=b)[0]
    agg = comp.dequantize_sum(sums, shared, q, n)
    est = rht_inverse(GradientVector(agg, agg.size), spec).values[:d] / n
    own = [rht_inverse(GradientVector(comp.dequantize_sum(z, shared, q, 1), agg.size), spec).values[:d]
           for z in codes]
    np.savez_compressed(
        os.path.join(OUT, f"{name}.npz"),
        meta=json.dumps({"n": n, "d": d, "seed": seed, "round": r, "q": q, "b": b, "max_block": max_block,
                         "block": spec.block_size, "padded": P, "sign_seed": spec.sign_seed,
                         "clip_events": op.clip_events, "total_adds": op.total_adds, "clamps": clamps}),
        corrected=np.stack(corrected), signs=spec.signs, rotated=np.stack(rotated), ranges=np.stack(ranges),
        shared=shared, codes=np.stack(codes), sums=np.asarray(sums, dtype=np.int64), agg=agg,
        estimate=est, own=np.stack(own))
    print(name, "ok")


def seed_vectors():
    seeds = SeedSpec(2024)
    out = {"splitmix64": {str(v): splitmix64(v) for v in (0, 1, 12345, (1 << 64) - 1)},
           "fnv1a64": {t: fnv1a64(t) for t in ("", "a", "rotation-signs", "stochastic-round", "lowrank-seed")},
           "stream_seed": [], "pcg": []}
    for tag, r, w in (("rotation-signs", 0, None), ("rotation-signs", 7, None), ("stochastic-round", 3, 2),
                      ("lowrank-seed", 1, None), ("grad-worker", 0, 5)):
        s = seeds.stream_seed(tag, r, w)
        st = np.random.PCG64(s).state["state"]
        g = seeds.rng(tag, r, w)
        out["stream_seed"].append({"tag": tag, "round": r, "worker": w, "seed": s})
        out["pcg"].append({"seed": s, "state": st["state"], "inc": st["inc"],
                           "random5": [float(x) for x in g.random(5)],
                           "bits64": [int(x) for x in seeds.rng(tag, r, w).integers(0, 2, size=64)]})
    with open(os.path.join(OUT, "seeds.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("seeds ok")


def chunk_norm_vectors():
    rng = np.random.default_rng(77)
    out = {}
    for C in (1, 3, 8, 9, 64, 100, 129, 1000):
        v = (rng.standard_normal(C * 5 + 3) * rng.uniform(0.01, 100)).astype(np.float32)
        out[f"v_{C}"] = v
        out[f"norms_{C}"] = chunk_sq_norms(v, ChunkGeometry.for_dim(v.size, C))
    np.savez_compressed(os.path.join(OUT, "chunk_norms.npz"), **out)
    print("chunk norms ok")


def payload_vectors():
    """Reference encode_payload bytes (compressors.py:292-325) for one payload of every type,
    built with the reference codec functions on seeded data."""
    rng = np.random.default_rng(77)
    x = rng.standard_normal(5000).astype(np.float32)
    x[:3] = 1e6   # fp16 saturation in the sparse values
    sp = comp.topk_compress(x, 200)
    ids = comp.select_chunks(np.abs(x[:4992].reshape(-1, 64)).sum(axis=1).astype(np.float32), 5)
    cs = comp.chunk_values(x, 64, ids)
    xr = x[:4096].astype(np.float32)
    ranges = comp.chunk_ranges(xr, 1024)
    codes, _ = comp.quantize_stochastic(xr, ranges, 4, SeedSpec(1).rng("stochastic-round", 0, 0))
    qp = comp.QuantPayload(codes, ranges, 0xDEADBEEFCAFE, 4, 1024)
    lr = comp.LowRankPayload(rng.standard_normal((30, 3)).astype(np.float32),
                             rng.standard_normal((20, 3)).astype(np.float32), (30, 20))
    d16 = comp.DensePayload(x[:100], 16)
    d32 = comp.DensePayload(x[:100], 32)
    out = {}
    for name, pl in (("sparse", sp), ("chunkset", cs), ("quant", qp), ("lowrank", lr), ("dense16", d16),
                     ("dense32", d32)):
        out[f"{name}_bytes"] = np.frombuffer(comp.encode_payload(pl), dtype=np.uint8)
        out[f"{name}_bits"] = np.array(comp.payload_bits(pl), dtype=np.int64)
    out["sparse_idx"], out["sparse_val"] = sp.indices, sp.values
    out["chunk_ids"], out["chunk_vals"] = cs.chunk_ids, cs.values
    out["quant_codes"], out["quant_ranges"] = qp.codes, qp.ranges
    out["lr_left"], out["lr_right"] = lr.left, lr.right
    out["dense_vals"] = x[:100]
    np.savez_compressed(os.path.join(OUT, "payloads.npz"), **out)
    print("payloads ok")


def synthetic_vectors():
    """trainbench.synthetic_round (trainbench.py:31-113) at small sizes: pins oracle/synthetic.py."""
    from gradcomp.trainbench import SyntheticGradSpec, synthetic_round
    out, meta = {}, []
    for i, (d, kw, seed, r, n) in enumerate([(1000, {}, 2024, 0, 3), (4099, dict(rho=0.0), 5, 2, 2),
                                             (20000, dict(rho=0.5, spike_density=0.3, divergence=0.0), 9, 1, 2),
                                             (30000, {}, 2024, 3, 4)]):
        out[f"g_{i}"] = np.stack(synthetic_round(SyntheticGradSpec(dim=d, **kw), SeedSpec(seed), r, n))
        meta.append({"d": d, "kw": kw, "seed": seed, "round": r, "n": n})
    np.savez_compressed(os.path.join(OUT, "synthetic.npz"), meta=json.dumps(meta), **out)
    print("synthetic ok")


def main():
    gauss = lambda rng, d, w: rng.standard_normal(d).astype(np.float32)  # noqa: E731
    quart = lambda rng, d, w: quarters(rng, d)  # noqa: E731
    seed_vectors()
    synthetic_vectors()
    chunk_norm_vectors()
    payload_vectors()
    thc_intermediates("thc_steps_a", 3, 3000, 1234, 0, 4, 4, 256)
    thc_intermediates("thc_steps_b", 4, 4096, 99, 2, 4, 8, 1024)
    thc_intermediates("thc_steps_c", 5, 20000, 5, 1, 3, 6, 1 << 15)
    run_case("thc_a", RotatedQuantConfig(4, 4, 256), 3, 3000, 1234, 2, gauss)
    run_case("thc_b", RotatedQuantConfig(4, 8, 1024), 4, 4096, 2024, 2, gauss)
    run_case("thc_c", RotatedQuantConfig(3, 5, 1024), 2, 100, 7, 2, gauss)
    run_case("thc_d", RotatedQuantConfig(4, 4, 1 << 15), 4, 20000, 901, 1, gauss, error_feedback=False)
    run_case("thc_e", RotatedQuantConfig(8, 16, 64), 5, 777, 31, 2, gauss)
    run_case("thc_f", RotatedQuantConfig(2, 2, 2), 3, 50, 3, 2, gauss)
    run_case("topk_a", TopKConfig(50), 4, 5000, 1, 2, quart)
    run_case("topk_b", TopKConfig(7), 3, 1000, 2, 3, gauss)
    run_case("chunked_a", ChunkedTopKConfig(64, 10), 3, 5000, 3, 2, gauss)
    run_case("chunked_b", ChunkedTopKConfig(16, 20, permute=True), 2, 1000, 4, 2, gauss)
    run_case("chunked_c", ChunkedTopKConfig(7, 5), 5, 333, 5, 2, quart)
    run_case("psgd_a", PowerSgdConfig(4), 3, 10000, 6, 3, gauss)
    run_case("psgd_b", PowerSgdConfig(2), 2, 1000, 7, 2, gauss)
    run_case("psgd_c", PowerSgdConfig(2, warm_start=False), 2, 4096, 8, 2, gauss)
    run_case("dense16", DenseConfig(16), 4, 5000, 9, 1, gauss)
    run_case("dense32", DenseConfig(32), 3, 5000, 10, 1, gauss)
    print("gradcomp", gradcomp.__version__, "numpy", np.__version__)


if __name__ == "__main__":
    main()
