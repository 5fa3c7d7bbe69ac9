"""Benchmark: compress + allreduce + decompress throughput (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--scheme thc]

Workload (BASELINE.json configs[1]): THC with partial rotation
(B = 1024) and saturation on an int8 wire (q = 4, b = 8), d = 25,557,032 coordinates
(ResNet-50 sized), n = 8 logical workers.  At --gpus 1 the 8 workers are simulated on the
one B200 (their ring collectives become ring-ordered folds, exactly the reference's
semantics); with N > 1 ranks the 8 workers are split over the ranks (n/N each) and the
exchange runs over NCCL (paper_2407_01378_b200.distributed).

A step is one GradientPipeline.run_round over fresh synthetic gradients (Gaussian, the
`grad-worker` streams of SURVEY §8(d)) with the EF residuals carried across steps.
value = d / T_step in Gelem/s (the reference's metric), T_step = max over
ranks of the CUDA-event time of the step.  Inputs (1.6 GB) exceed the 126 MB L2, so no
flush is needed between steps.  `e2e` runs the same step through the public API from
pinned host buffers (H2D of the gradients and D2H of the estimate inside the timed
region).  `roofline` reports the fused THC kernel against the measured HBM copy bandwidth
with algorithmic bytes (12n + 4) * d per launch.  `cpu_baseline` times the CPU oracle
(oracle/, a NumPy restatement of the reference path) on a bounded sample.

--impl reference times the reference's own CPU algorithm (the oracle port; the Python
reference cannot be shipped to the GPU box) on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "compress+allreduce+decompress Gelem/s at 1/2/4/8 B200 vs FP16 NCCL allreduce"
D_CFG2 = 25_557_032
N_WORKERS = 8


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--d", type=int, default=D_CFG2)
    ap.add_argument("--workers", type=int, default=N_WORKERS)
    ap.add_argument("--quant-bits", type=int, default=4)
    ap.add_argument("--wire-bits", type=int, default=8)
    ap.add_argument("--rotation-block", type=int, default=1024)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-bar", action="store_true", help="skip the FP16-bar comparison line")
    ap.add_argument("--sweep", action="store_true", help="also time TopK / TopK-C / PowerSGD at their configs")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def workload(args, n_gpus):
    return {
        "workload": (f"cfg2 THC partial rotation + saturation: q={args.quant_bits}, b={args.wire_bits} "
                     f"(int8 wire), B={args.rotation_block}, d={args.d:,}, n={args.workers} workers "
                     + ("simulated on 1 B200" if n_gpus == 1 else f"over {n_gpus} B200")),
        "scheme": "rotated_quant", "d": args.d, "workers": args.workers, "quant_bits": args.quant_bits,
        "wire_bits": args.wire_bits, "rotation_block": args.rotation_block, "error_feedback": True,
        "l2": "inputs (n*d*4 B = %.2f GB) exceed the 126 MB L2; no flush needed" % (args.workers * args.d * 4 / 1e9),
        "parallelism": f"dp{n_gpus}",
    }


# ------------------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clock and throttle reasons sampled DURING the timed region (NVML thread, every 2 ms;
    nvidia-smi --query-gpu is the fallback)."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.samples = []
        self.max_mhz = None
        self._stop = None
        self._thread = None

    def __enter__(self):
        import threading
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.idx)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
            self._stop = threading.Event()

            def loop():
                while not self._stop.is_set():
                    try:
                        clk = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                        rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.samples.append((float(clk), int(rs)))
                    except pynvml.NVMLError:
                        pass
                    self._stop.wait(0.002)

            self._thread = threading.Thread(target=loop, daemon=True)
            self._thread.start()
        except Exception:
            self._thread = None
        return self

    def __exit__(self, *exc):
        if self._thread is not None:
            self._stop.set()
            self._thread.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0, "source": "nvml"}
        reasons = sorted({name for _, r in self.samples for name, bit in self.REASONS.items() if r & bit})
        return {"sm_mhz": statistics.median(c for c, _ in self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.samples), "source": "nvml, 2 ms"}


# ------------------------------------------------------------------------------ CPU side
def cpu_thc_sample(args, d_sample: int, rounds: int):
    """Reference CPU algorithm (oracle port) on a bounded sample: seconds per round."""
    import numpy as np

    from oracle import gradcomp_oracle as orc
    n = args.workers
    seeds = 2024
    params = dict(quant_bits=args.quant_bits, wire_bits=args.wire_bits, rotation_block=args.rotation_block)
    state = orc.OracleState([np.zeros(d_sample, np.float32) for _ in range(n)])
    times = []
    for r in range(rounds):
        grads = [orc.stream_rng(seeds, "grad-worker", r, w).standard_normal(d_sample).astype(np.float32)
                 for w in range(n)]
        t0 = time.perf_counter()
        orc.run_round("rotated_quant", params, state, grads, seeds, r)
        times.append(time.perf_counter() - t0)
    return times


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    d_sample = 1 << 18
    times = cpu_thc_sample(args, d_sample, args.warmup + args.steps)[args.warmup:]
    t = statistics.median(times)
    val = d_sample / t / 1e9
    cfg = workload(args, max(world, 1))
    out = {"metric": METRIC, "value": val, "unit": "Gelem/s", "n_gpus": args.gpus, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic (Gaussian grad-worker streams)",
           "config": cfg, "impl": "reference",
           "cpu_baseline": {"value": val, "unit": "Gelem/s", "cores": 1, "kind": "port",
                            "sample": f"oracle port (NumPy restatement of gradcomp) THC round, n={args.workers}, "
                                      f"d={d_sample:,} per step, median of {args.steps} steps"},
           "e2e": {"value": val, "unit": "Gelem/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


# ------------------------------------------------------------------------------ GPU side
def time_pipeline(gcb, cfg, n, d, seeds, world, local_n, pool, args, dev):
    """CUDA-event time of run_round for another scheme at the same worker split (max over ranks)."""
    import torch
    if world == 1:
        pipe = gcb.make_pipeline(cfg, n, d, seeds, validate=False, compute_nmse=False)
    else:
        from paper_2407_01378_b200.distributed import DistributedGradientPipeline
        pipe = DistributedGradientPipeline(cfg, n, d, seeds, validate=False, compute_nmse=False)
    for s in range(args.warmup):
        pipe.run_round(pool[s % len(pool)], s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    steps = max(3, min(args.steps, 10))
    e0.record()
    for s in range(steps):
        pipe.run_round(pool[s % len(pool)], args.warmup + s)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    del pipe
    return {"scheme": gcb.scheme_label(cfg), "d": d, "workers": n, "ms_per_step": ms,
            "value": d / (ms * 1e-3) / 1e9, "unit": "Gelem/s", "steps": steps}


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch

    import paper_2407_01378_b200 as gcb

    world, rank, local = dist_env()
    n_gpus = world
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    n, d = args.workers, args.d
    if n % world:
        raise SystemExit(f"--workers {n} must be divisible by the number of ranks {world}")
    local_n = n // world
    cfg = gcb.RotatedQuantConfig(args.quant_bits, args.wire_bits, args.rotation_block)
    seeds = gcb.SeedSpec(2024)

    if world == 1:
        pipe = gcb.make_pipeline(cfg, n, d, seeds, validate=False, compute_nmse=False)
    else:
        from paper_2407_01378_b200.distributed import DistributedGradientPipeline
        pipe = DistributedGradientPipeline(cfg, n, d, seeds, validate=False, compute_nmse=False)
    engine = pipe._engine

    # synthetic gradients: Gaussian, a fresh batch per step from a pool resident in HBM
    gen = torch.Generator(device=dev)
    gen.manual_seed(2024 + rank)
    pool = [torch.randn(local_n, d, device=dev, generator=gen) for _ in range(2)]

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    for s in range(args.warmup):
        pipe.run_round(pool[s % 2], s)
    torch.cuda.synchronize()
    barrier()
    engine.kernel_events = []
    launches0 = engine.launches
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        barrier()
        start.record()
        for s in range(args.steps):
            pipe.run_round(pool[s % 2], args.warmup + s)
        end.record()
        torch.cuda.synchronize()
        barrier()
    ms = start.elapsed_time(end) / args.steps
    kms = [a.elapsed_time(b) for a, b in engine.kernel_events]
    engine.kernel_events = None
    launches = engine.launches - launches0
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = d / (ms * 1e-3) / 1e9

    # roofline of the dominant kernel (fused THC round): algorithmic bytes (12n+4)*d per launch
    roof = None
    if kms:
        kernel_ms = statistics.mean(kms)
        alg_bytes = (12 * local_n + 4) * d
        peak, peak_src = 6539.2, "fallback"
        try:
            with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
                peak, peak_src = float(json.load(f)["hbm_gbs"]), "measured"
        except (OSError, KeyError, ValueError):
            pass
        achieved = alg_bytes / (kernel_ms * 1e-3) / 1e9
        traffic = None
        tf = os.path.join(ROOT, "profiles", "traffic.json")
        try:
            with open(tf) as f:
                tr = json.load(f)
            key = f"thc_fused:n={local_n}:d={d}:q={args.quant_bits}:b={args.wire_bits}:B={args.rotation_block}"
            traffic = tr.get(key)
        except (OSError, ValueError):
            pass
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "kernel": "thc_fused_kernel", "kernel_ms": kernel_ms,
                "kernel_share_of_step": kernel_ms / ms, "algorithmic_bytes_per_launch": alg_bytes,
                "peak_source": f"{peak_src} hbm_gbs (MEASURED_PEAKS.json)"}

    # end to end through the public API from pinned host memory
    e2e = None
    if not args.no_e2e:
        # the workers' gradients as one pinned [n, d] host block (a list of per-worker arrays is
        # accepted as well; the block lets every segment go over PCIe as one strided copy)
        host = torch.empty(local_n, d, dtype=torch.float32).pin_memory()
        host.copy_(pool[0].cpu())
        pipe_e2e = (gcb.make_pipeline(cfg, n, d, seeds) if world == 1 else
                    DistributedGradientPipeline(cfg, n, d, seeds))
        out_host = torch.empty(d, dtype=torch.float32).pin_memory()
        steps_e2e = max(3, min(args.steps, 10))
        for s in range(2):
            res = pipe_e2e.run_round(host, s)
            out_host.copy_(res.estimate_tensor, non_blocking=True)
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for s in range(steps_e2e):
            res = pipe_e2e.run_round(host, 2 + s)
            if res.estimate_host is None:   # streamed host rounds copy the estimate back themselves
                out_host.copy_(res.estimate_tensor, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        e2e_ms = e0.elapsed_time(e1) / steps_e2e
        if world > 1:
            import torch.distributed as dist
            t = torch.tensor([e2e_ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t.item())
        e2e = {"value": d / (e2e_ms * 1e-3) / 1e9, "unit": "Gelem/s", "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": 4 * local_n * d, "d2h_bytes_per_step": 4 * d,
               "path": "GradientPipeline.run_round(pinned [n, d] host tensor) -> host estimate; H2D (one strided "
                       "copy per segment), finite check + fused kernel and D2H overlapped over tile segments; "
                       "input validation on"}
        del pipe_e2e

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        d_sample = 1 << 19
        times = cpu_thc_sample(args, d_sample, 3)
        t = statistics.median(times)
        cpu = {"value": d_sample / t / 1e9, "unit": "Gelem/s", "cores": 1, "kind": "port",
               "sample": f"oracle port (NumPy restatement of the reference THC round), n={n}, d={d_sample:,}, "
                         f"median of 3 rounds; numpy elementwise ops are single-threaded"}

    bar = None
    if not args.no_bar:
        bar = time_pipeline(gcb, gcb.DenseConfig(16), n, d, seeds, world, local_n, pool, args, dev)
        bar["what"] = ("dense FP16 round at the same d and n (fp16 inputs, fp16 wire per hop; NCCL half "
                       "all-reduce across ranks): the utility bar of BASELINE.json's metric")
        bar["thc_vs_bar_time_ratio"] = ms / bar["ms_per_step"]
    sweep = None
    if args.sweep:
        sweep = {}
        for name, cfg, dd in (("topk_1pct_cfg3", gcb.TopKConfig(1_100_000), 110_000_000),
                              ("topkc_1pct_cfg3", gcb.ChunkedTopKConfig(64, 17_187), 110_000_000),
                              ("powersgd_r4_cfg4", gcb.PowerSgdConfig(4), 350_000_000)):
            del pool
            torch.cuda.empty_cache()
            pool = [torch.randn(local_n, dd, device=dev, generator=gen)]
            sweep[name] = time_pipeline(gcb, cfg, n, dd, seeds, world, local_n, pool, args, dev)

    if rank == 0:
        out = {"metric": METRIC, "value": value, "unit": "Gelem/s", "n_gpus": n_gpus, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
               "vs_baseline": None, "dtype": "f64", "data": "synthetic (Gaussian gradients, random per rank)",
               "config": workload(args, n_gpus), "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
               "gpu_launches": launches, "clocks": clk.summary(),
               "worker_elements_per_s": n * d / (ms * 1e-3), "fp16_bar": bar}
        if sweep is not None:
            out["sweep"] = sweep
        print(json.dumps(out))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
