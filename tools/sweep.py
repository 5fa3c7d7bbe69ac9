"""Time every scheme at its SURVEY §8(d) config, n simulated workers on one B200.

python tools/sweep.py [--n 8] [--steps 10] [--only thc,topk,...] [--synthetic] [--nmse R]
Prints one JSON line per scheme: ms/round, Gelem/s (d / T), algorithmic HBM bytes and the
fraction of the measured HBM bandwidth those bytes imply.

--synthetic: SyntheticGradSpec-model gradients (paper_2407_01378_b200.synthetic, trainbench.py:31-113
structure), a fresh round for every warm-up and timed step (pre-generated outside the timed
region), so data-dependent paths (TopK's threshold hint) see real round-to-round drift.
--nmse R: the nmse sweep of cli.py:279-333 instead of timing: R rounds per scheme on synthetic
gradients with compute_nmse, one `round,scheme,nmse,bits_per_coord,overflow_rate` row per round and
a mean line per scheme (the reference's rounds.csv / nmse_summary.csv columns, minus the
TimeModel's simulated_ms)."""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2407_01378_b200 as gcb

HBM = 6539.2e9


def alg_bytes(name, n, d, cfg):
    # compulsory bytes: g, r read; r_new, estimate written
    if name.startswith("dense"):
        return (4 * n + 4) * d
    if name.startswith("topk_"):
        k = cfg.k
        return 12 * n * d + 4 * d + 6 * k * n * 2
    return 12 * n * d + 4 * d


def nmse_sweep(name, cfg, n, d, rounds, seed=2024):
    """cli.py:279-333: R rounds of one scheme on synthetic gradients, nmse per round."""
    from paper_2407_01378_b200.ledger import overflow_rate
    from paper_2407_01378_b200.synthetic import SyntheticGradients
    gen = SyntheticGradients(d, gcb.SeedSpec(seed))
    pipe = gcb.make_pipeline(cfg, n, d, gcb.SeedSpec(seed), validate=False, compute_nmse=True)
    nmses, rates = [], []
    for r in range(rounds):
        res = pipe.run_round(gen.round(r, n), r)
        nmses.append(res.nmse)
        rates.append(overflow_rate(res.overflow))
        print(f"{r},{name},{res.nmse!r},{res.input_bits_per_coord!r},{rates[-1]!r}", flush=True)
    print(json.dumps({"scheme": name, "n": n, "d": d, "rounds": rounds, "bits_per_coord": res.input_bits_per_coord,
                      "mean_nmse": sum(nmses) / rounds, "mean_overflow_rate": sum(rates) / rounds}), flush=True)
    del pipe, gen
    torch.cuda.empty_cache()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=8)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=12)
    ap.add_argument("--only", default="")
    ap.add_argument("--dims", default="", help="cfg5: comma list of d (e.g. 1048576,...,1e9); every scheme at each d")
    ap.add_argument("--synthetic", action="store_true", help="fresh SyntheticGradSpec-model gradients every round")
    ap.add_argument("--nmse", type=int, default=0, help="nmse sweep: R rounds per scheme, no timing")
    a = ap.parse_args()
    n = a.n
    if a.dims:
        dims = [int(float(x)) for x in a.dims.split(",")]
        cases = []
        for d in dims:
            cases += [(f"thc_q4b8_d{d}", gcb.RotatedQuantConfig(4, 8), d),
                      (f"thc_q4b4_d{d}", gcb.RotatedQuantConfig(4, 4), d),
                      (f"topk_1pct_d{d}", gcb.TopKConfig(max(1, d // 100)), d),
                      (f"topkc_1pct_d{d}", gcb.ChunkedTopKConfig(64, max(1, d // 6400)), d),
                      (f"powersgd_r4_d{d}", gcb.PowerSgdConfig(4), d),
                      (f"dense16_d{d}", gcb.DenseConfig(16), d),
                      (f"dense32_d{d}", gcb.DenseConfig(32), d)]
    else:
      cases = [
        ("thc_q4b8_cfg2", gcb.RotatedQuantConfig(4, 8), 25_557_032),
        ("thc_q4b4_cfg2", gcb.RotatedQuantConfig(4, 4), 25_557_032),
        ("topk_1pct_cfg3", gcb.TopKConfig(1_100_000), 110_000_000),
        ("topkc_1pct_cfg3", gcb.ChunkedTopKConfig(64, 17_187), 110_000_000),
        ("powersgd_r4_cfg4", gcb.PowerSgdConfig(4), 350_000_000),
        ("powersgd_r4_gpt2m_chunked", gcb.PowerSgdConfig(4), "gpt2m"),
        ("dense16_cfg2", gcb.DenseConfig(16), 25_557_032),
        ("dense16_cfg4", gcb.DenseConfig(16), 350_000_000),
        ("dense32_cfg4", gcb.DenseConfig(32), 350_000_000),
    ]
    only = set(a.only.split(",")) if a.only else None
    for name, cfg, d in cases:
        if only and not any(name.startswith(o) for o in only):
            continue
        torch.cuda.empty_cache()
        if d == "gpt2m":
            from paper_2407_01378_b200.multitensor import TensorListPipeline, gpt2_medium_sizes
            sizes = gpt2_medium_sizes()
            d = sum(sizes)
            g = torch.randn(n, d, device="cuda")
            pipe = TensorListPipeline(cfg, n, sizes, gcb.SeedSpec(2024), validate=False, compute_nmse=False)
            eng = pipe
            pool = [g]
        elif a.nmse:
            nmse_sweep(name, cfg, n, d, a.nmse)
            continue
        else:
            pipe = gcb.make_pipeline(cfg, n, d, gcb.SeedSpec(2024), validate=False, compute_nmse=False)
            eng = pipe._engine
            if a.synthetic:   # a distinct round of gradients per step, generated before timing
                from paper_2407_01378_b200.synthetic import SyntheticGradients
                gen = SyntheticGradients(d, gcb.SeedSpec(2024))
                pool = [gen.round(r, n) for r in range(a.warmup + a.steps)]
                del gen
            else:
                pool = [torch.randn(n, d, device="cuda")]
            g = pool[0]
        # warm-up rounds (repeated Gaussian inputs: EF residuals grow until the TopK threshold
        # settles; synthetic: fresh rounds), then the timed steady state
        for r in range(a.warmup):
            pipe.run_round(pool[r % len(pool)], r)
        torch.cuda.synchronize()
        eng.kernel_events = [] if hasattr(eng, "kernel_events") else None
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record()
        for r in range(a.steps):
            pipe.run_round(pool[(a.warmup + r) % len(pool)], a.warmup + r)
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / a.steps
        kev = getattr(eng, "kernel_events", None) or []
        kms = sum(x.elapsed_time(y) for x, y in kev) / max(1, len(kev))
        b = alg_bytes(name, n, d, cfg)
        print(json.dumps({"case": name, "n": n, "d": d, "ms": round(ms, 4), "gelem_s": round(d / ms / 1e6, 3),
                          "core_ms": round(kms, 4), "alg_GB": round(b / 1e9, 3),
                          "hbm_frac": round(b / (ms * 1e-3) / HBM, 4),
                          "inputs": "synthetic, fresh per round" if a.synthetic else "gaussian, repeated"}),
              flush=True)
        del pipe, g, eng, pool
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
