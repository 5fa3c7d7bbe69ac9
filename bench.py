"""Benchmark: compress + allreduce + decompress throughput (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[1]): THC with partial rotation
(B = 1024) and saturation on an int8 wire (q = 4, b = 8), d = 25,557,032 coordinates
(ResNet-50 sized), n = 8 logical workers (strong scaling: the 8 workers are split over the
N GPUs).  At N = 1 the 8 workers are simulated on the one B200 (their ring collectives
become ring-ordered folds, exactly the reference's semantics, in one fused kernel); with
N > 1 ranks every rank runs its n/N workers and the exchange runs over NCCL
(paper_2407_01378_b200.distributed: range all-reduce, code all-to-all + ordered saturating
fold + all-gather).

Launch: the driver's torchrun form sets WORLD_SIZE; `python bench.py --gpus N` without it
re-executes itself under `torch.distributed.run` with N ranks (127.0.0.1 rendezvous).  The
world size must equal --gpus.  `--distributed` runs the per-rank (NCCL) pipeline even at N = 1.

A step is one run_round over fresh synthetic gradients (Gaussian; a pool of two batches
resident in HBM, 0.8 GB per batch > the 126 MB L2, so no flush is needed) with the EF
residuals carried across steps.  value = d / T_step in Gelem/s, T_step = max over ranks of
the CUDA-event time of the K steps / K.  `e2e` runs the same step through the public API
from pinned host buffers (H2D of the gradients and D2H of the estimate inside the timed
region).  `roofline` reports the dominant kernel against the measured HBM copy bandwidth
with algorithmic bytes per launch.  `north_star` times north_star's 350M-element vector with
one worker per GPU (n = N): THC q4b8, PowerSGD r4 (one 18,709 x 18,708 matrix, and chunked over
GPT-2-medium's 292 tensors) and the FP16 NCCL all-reduce bar.  `cpu_baseline` times the CPU
oracle (oracle/, a NumPy restatement of the reference path) on a bounded sample.

--impl reference times the reference's own CPU THC round -- the unmodified gradcomp package staged
under baseline/_ref/src (git-ignored; build() copies it from /root/reference and it travels with
the snapshot), or the oracle port when it is absent -- on a bounded sample of the same workload;
rank 0 alone runs it.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "compress+allreduce+decompress Gelem/s at 1/2/4/8 B200 vs FP16 NCCL allreduce"
D_CFG2 = 25_557_032
D_NORTH = 350_000_000
N_WORKERS = 8


def parse(argv=None):
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
    ap.add_argument("--distributed", action="store_true",
                    help="run the per-rank DistributedGradientPipeline (NCCL) even at one GPU")
    ap.add_argument("--backend", default=os.environ.get("GC_BENCH_BACKEND", "nccl"))
    ap.add_argument("--dry-run", action="store_true",
                    help="launcher / rendezvous / max-over-ranks check without GPU work (CPU tests)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-bar", action="store_true", help="skip the FP16-bar comparison")
    ap.add_argument("--no-north-star", action="store_true", help="skip the 350M one-worker-per-GPU block")
    ap.add_argument("--sweep", action="store_true", help="also time TopK / TopK-C / PowerSGD at their configs")
    return ap.parse_args(argv)


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch(args) -> int:
    """`python bench.py --gpus N` outside torchrun: re-exec under torch.distributed.run, N ranks."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def host_info():
    try:
        aff = len(os.sched_getaffinity(0))
    except AttributeError:
        aff = os.cpu_count()
    return {"host_cpu_count": os.cpu_count(), "host_affinity": aff}


def workload(args, n_gpus):
    return {
        "workload": (f"cfg2 THC partial rotation + saturation: q={args.quant_bits}, b={args.wire_bits} "
                     f"(int8 wire), B={args.rotation_block}, d={args.d:,}, n={args.workers} workers "
                     + ("simulated on 1 B200" if n_gpus == 1 and not args.distributed else f"over {n_gpus} B200")),
        "scheme": "rotated_quant", "d": args.d, "workers": args.workers, "quant_bits": args.quant_bits,
        "wire_bits": args.wire_bits, "rotation_block": args.rotation_block, "error_feedback": True,
        "l2": "inputs (n*d*4 B = %.2f GB) exceed the 126 MB L2; no flush needed" % (args.workers * args.d * 4 / 1e9),
        "parallelism": f"dp{n_gpus}",
    }


# ------------------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clock and throttle reasons sampled DURING the timed region (NVML thread, every 2 ms)."""

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
def reference_package():
    """The UNMODIFIED reference package staged under baseline/_ref/src (git-ignored, travels with the
    snapshot; build() stages it from /root/reference), or None."""
    src = os.path.join(ROOT, "baseline", "_ref", "src")
    if not os.path.isfile(os.path.join(src, "gradcomp", "pipelines.py")):
        return None
    if src not in sys.path:
        sys.path.insert(0, src)
    try:
        import gradcomp
        return gradcomp
    except Exception:
        return None


def cpu_thc_sample(args, d_sample: int, rounds: int):
    """The reference's CPU THC round on a bounded sample: seconds per round and the kind --
    "reference" (gradcomp's own make_pipeline(...).run_round, pipelines.py:418-425, 147-182) when
    the package is staged, else "port" (the oracle's NumPy restatement of the same round)."""
    import numpy as np

    n = args.workers
    ref = reference_package()
    times = []
    if ref is not None:
        seeds = ref.SeedSpec(2024)
        pipe = ref.make_pipeline(ref.RotatedQuantConfig(args.quant_bits, args.wire_bits, args.rotation_block), n,
                                 d_sample, seeds)
        for r in range(rounds):
            grads = [seeds.rng("grad-worker", r, w).standard_normal(d_sample).astype(np.float32) for w in range(n)]
            t0 = time.perf_counter()
            pipe.run_round(grads, r)
            times.append(time.perf_counter() - t0)
        return times, "reference"
    from oracle import gradcomp_oracle as orc
    seeds = 2024
    params = dict(quant_bits=args.quant_bits, wire_bits=args.wire_bits, rotation_block=args.rotation_block)
    state = orc.OracleState([np.zeros(d_sample, np.float32) for _ in range(n)])
    for r in range(rounds):
        grads = [orc.stream_rng(seeds, "grad-worker", r, w).standard_normal(d_sample).astype(np.float32)
                 for w in range(n)]
        t0 = time.perf_counter()
        orc.run_round("rotated_quant", params, state, grads, seeds, r)
        times.append(time.perf_counter() - t0)
    return times, "port"


def run_reference(args):
    """The reference's own CPU THC round (gradcomp from baseline/_ref, else the oracle port; one host
    core: the reference's numpy THC path is single-threaded) on a 2^18-coordinate sample of the cfg2
    workload per step.  Rank 0 only."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    d_sample = 1 << 18
    times, kind = cpu_thc_sample(args, d_sample, args.warmup + args.steps)
    times = times[args.warmup:]
    t = statistics.median(times)
    val = d_sample / t / 1e9
    cfg = workload(args, max(world, args.gpus))
    cfg["d"] = d_sample
    cfg["workload"] += f" -- CPU sample: d={d_sample:,} per step (cfg2's d={args.d:,} would take minutes per round)"
    cfg["sample_d"] = d_sample
    out = {"metric": METRIC, "value": val, "unit": "Gelem/s", "n_gpus": args.gpus, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic (Gaussian grad-worker streams)",
           "config": cfg, "impl": "reference",
           "cpu_baseline": dict({"value": val, "unit": "Gelem/s", "cores": 1, "kind": kind,
                                 "sample": (("gradcomp itself (the unmodified reference package, "
                                             "make_pipeline(...).run_round)") if kind == "reference" else
                                            "oracle port (NumPy restatement of gradcomp's THC round, "
                                            "pipelines.py:260-322)")
                                           + f", n={args.workers} workers, d={d_sample:,} "
                                           f"coordinates per step (not cfg2's d={args.d:,}: the rate is per "
                                           f"coordinate and the round is linear in d), median of {args.steps} steps; "
                                           f"numpy's elementwise THC path runs on one core"}, **host_info()),
           "e2e": {"value": val, "unit": "Gelem/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ------------------------------------------------------------------------------ dry run
def run_dry(args, world, rank):
    """Launcher check without a GPU: rendezvous, barrier, max-over-ranks of a host timing."""
    import torch
    import torch.distributed as dist
    if world > 1:
        dist.init_process_group(args.backend)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        sum(range(10000))
    ms = (time.perf_counter() - t0) * 1e3 / max(1, args.steps)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    if rank == 0:
        print(json.dumps({"metric": METRIC, "dry_run": True, "n_gpus": world, "world_size": world,
                          "backend": args.backend, "steps": args.steps, "ms_per_step": ms,
                          "config": workload(args, world)}), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ------------------------------------------------------------------------------ GPU side
def max_over_ranks(v: float, world: int, dev) -> float:
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def timed_rounds(pipe, pool, warmup, steps, world, dev, barrier, r0=0):
    """CUDA-event time of `steps` rounds after `warmup` (ms per round, max over ranks)."""
    import torch
    for s in range(warmup):
        pipe.run_round(pool[s % len(pool)], r0 + s)
    torch.cuda.synchronize()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for s in range(steps):
        pipe.run_round(pool[s % len(pool)], r0 + warmup + s)
    e1.record()
    torch.cuda.synchronize()
    barrier()
    return max_over_ranks(e0.elapsed_time(e1) / steps, world, dev)


def make_pipe(gcb, cfg, n, d, seeds, distributed, **kw):
    if distributed:
        from paper_2407_01378_b200.distributed import DistributedGradientPipeline
        return DistributedGradientPipeline(cfg, n, d, seeds, **kw)
    return gcb.make_pipeline(cfg, n, d, seeds, **kw)


def north_star_block(gcb, args, world, rank, dev, gen, barrier):
    """north_star's 350M-element vector, one worker per GPU (n = N, weak per GPU): per-rank
    DistributedGradientPipeline rounds over NCCL for THC q4b8, PowerSGD r4 (one 18,709 x 18,708
    matrix), chunked PowerSGD r4 over GPT-2-medium's 292 tensors, and the FP16 all-reduce bar."""
    import torch
    seeds = gcb.SeedSpec(2024)
    n, d = world, D_NORTH
    steps, warm = max(3, min(args.steps, 10)), max(3, min(args.warmup, 5))
    pool = [torch.randn(1, d, device=dev, generator=gen) for _ in range(2)]
    out = {"d": d, "workers": n, "workers_per_gpu": 1, "steps": steps,
           "what": "per-rank DistributedGradientPipeline rounds (NCCL) at north_star's d=350M, one worker per GPU"}
    cases = [("thc_q4b8", gcb.RotatedQuantConfig(4, 8, 1024)), ("powersgd_r4", gcb.PowerSgdConfig(4)),
             ("fp16_bar", gcb.DenseConfig(16))]
    for name, cfg in cases:
        try:
            pipe = make_pipe(gcb, cfg, n, d, seeds, True, validate=False)
            ms = timed_rounds(pipe, pool, warm, steps, world, dev, barrier)
            out[name] = {"ms_per_step": ms, "value": d / (ms * 1e-3) / 1e9, "unit": "Gelem/s"}
            del pipe
        except Exception as exc:   # a failing extra case must not cost the contract line
            out[name] = {"error": f"{type(exc).__name__}: {exc}"[:300]}
        torch.cuda.empty_cache()
    try:   # chunked PowerSGD: one reference pipeline per GPT-2-medium tensor, one worker per GPU
        from paper_2407_01378_b200.distributed import DistributedTensorListPipeline
        from paper_2407_01378_b200.multitensor import gpt2_medium_sizes
        sizes = gpt2_medium_sizes()
        D = sum(sizes)
        del pool
        torch.cuda.empty_cache()
        pool = [torch.randn(1, D, device=dev, generator=gen) for _ in range(2)]
        pipe = DistributedTensorListPipeline(gcb.PowerSgdConfig(4), n, sizes, seeds, device=dev, validate=False)
        ms = timed_rounds(pipe, pool, warm, steps, world, dev, barrier)
        out["powersgd_r4_gpt2m"] = {"ms_per_step": ms, "value": D / (ms * 1e-3) / 1e9, "unit": "Gelem/s", "d": D,
                                    "tensors": len(sizes)}
        del pipe
    except Exception as exc:
        out["powersgd_r4_gpt2m"] = {"error": f"{type(exc).__name__}: {exc}"[:300]}
    bar = out.get("fp16_bar", {}).get("ms_per_step")
    for name in ("thc_q4b8", "powersgd_r4", "powersgd_r4_gpt2m"):
        if bar and "ms_per_step" in out.get(name, {}):
            out[name]["time_vs_fp16_bar"] = out[name]["ms_per_step"] / bar
    del pool
    torch.cuda.empty_cache()
    return out


def main():
    args = parse()
    world, rank, local = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))
    if args.impl == "reference":
        run_reference(args)
        return
    if world > 1 and world != args.gpus:
        raise SystemExit(f"world size {world} does not match --gpus {args.gpus}")
    if args.dry_run:
        run_dry(args, world, rank)
        return
    import torch

    import paper_2407_01378_b200 as gcb

    n_gpus = world
    if os.environ.get("GC_BENCH_ONE_DEVICE") == "1":   # test hook: N gloo ranks sharing one GPU
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    distributed = world > 1 or args.distributed
    import torch.distributed as dist
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", str(free_port()))
        os.environ.setdefault("RANK", "0")
        os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group(args.backend, device_id=dev if args.backend == "nccl" else None)
    n, d = args.workers, args.d
    if n % world:
        raise SystemExit(f"--workers {n} must be divisible by the number of ranks {world}")
    local_n = n // world
    cfg = gcb.RotatedQuantConfig(args.quant_bits, args.wire_bits, args.rotation_block)
    seeds = gcb.SeedSpec(2024)

    pipe = make_pipe(gcb, cfg, n, d, seeds, distributed, validate=False, compute_nmse=False)
    engine = pipe._engine

    # synthetic gradients: Gaussian, a fresh batch per step from a pool resident in HBM
    gen = torch.Generator(device=dev)
    gen.manual_seed(2024 + rank)
    pool = [torch.randn(local_n, d, device=dev, generator=gen) for _ in range(2)]

    def barrier():
        if world > 1:
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
    kname = getattr(engine, "timed_kernel", "thc_fused_kernel")
    kbytes = getattr(engine, "timed_kernel_bytes", None)
    engine.kernel_events = None
    launches = engine.launches - launches0
    ms = max_over_ranks(ms, world, dev)
    value = d / (ms * 1e-3) / 1e9

    # roofline of the dominant kernel: algorithmic bytes per launch over its CUDA-event time
    roof = None
    if kms:
        kernel_ms = statistics.mean(kms)
        alg_bytes = kbytes if kbytes is not None else (12 * local_n + 4) * d
        peak, peak_src = 6539.2, "fallback (SURVEY §8(d))"
        try:
            with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
                peak, peak_src = float(json.load(f)["hbm_gbs"]), "measured hbm_gbs (MEASURED_PEAKS.json)"
        except (OSError, KeyError, ValueError):
            pass
        achieved = alg_bytes / (kernel_ms * 1e-3) / 1e9
        traffic = None
        try:
            with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
                tr = json.load(f)
            key = f"{kname}:n={local_n}:d={d}:q={args.quant_bits}:b={args.wire_bits}:B={args.rotation_block}"
            traffic = tr.get(key, tr.get(key.replace("thc_fused_kernel", "thc_fused")))
            issue = tr.get("issue:" + key)
        except (OSError, ValueError):
            issue = None
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "kernel": kname, "kernel_ms": kernel_ms,
                "kernel_share_of_step": kernel_ms / ms, "algorithmic_bytes_per_launch": alg_bytes,
                "peak_source": peak_src}
        if issue:   # what actually bounds the bit-exact THC kernel: instruction issue (ncu capture)
            roof["issue"] = dict(issue, achieved_warp_inst_per_s=issue["warp_instructions_per_launch"] / (kernel_ms * 1e-3),
                                 frac_of_issue_peak=issue["warp_instructions_per_launch"] / (kernel_ms * 1e-3)
                                 / issue["peak_warp_inst_per_s"])

    # end to end through the public API from pinned host memory
    e2e = None
    if not args.no_e2e:
        host = torch.empty(local_n, d, dtype=torch.float32).pin_memory()
        host.copy_(pool[0].cpu())
        pipe_e2e = make_pipe(gcb, cfg, n, d, seeds, distributed)
        out_host = torch.empty(d, dtype=torch.float32).pin_memory()
        steps_e2e = max(3, min(args.steps, 10))
        for s in range(2):
            res = pipe_e2e.run_round(host, s)
            out_host.copy_(res.estimate_tensor, non_blocking=True)
        torch.cuda.synchronize()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for s in range(steps_e2e):
            res = pipe_e2e.run_round(host, 2 + s)
            if res.estimate_host is None:   # streamed host rounds copy the estimate back themselves
                out_host.copy_(res.estimate_tensor, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        e2e_ms = max_over_ranks(e0.elapsed_time(e1) / steps_e2e, world, dev)
        e2e = {"value": d / (e2e_ms * 1e-3) / 1e9, "unit": "Gelem/s", "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": 4 * local_n * d, "d2h_bytes_per_step": 4 * d,
               "path": "run_round(pinned [n, d] host tensor) -> host estimate; H2D, finite check, kernels and D2H "
                       "inside the timed region; input validation on"}
        del pipe_e2e, host

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        d_sample = 1 << 18
        times, kind = cpu_thc_sample(args, d_sample, 3)
        t = statistics.median(times)
        cpu = dict({"value": d_sample / t / 1e9, "unit": "Gelem/s", "cores": 1, "kind": kind,
                    "sample": ("gradcomp itself (unmodified reference package)" if kind == "reference" else
                               "oracle port (NumPy restatement of the reference THC round)")
                              + f", n={n}, d={d_sample:,} (not cfg2's d; the round is linear in d), median of 3 "
                              f"rounds; numpy's elementwise THC path runs on one core"}, **host_info())

    bar = None
    if not args.no_bar:
        bpipe = make_pipe(gcb, gcb.DenseConfig(16), n, d, seeds, distributed, validate=False, compute_nmse=False)
        bms = timed_rounds(bpipe, pool, max(3, min(args.warmup, 5)), max(3, min(args.steps, 10)), world, dev,
                           barrier)
        del bpipe
        bar = {"scheme": "dense_fp16", "d": d, "workers": n, "ms_per_step": bms, "value": d / (bms * 1e-3) / 1e9,
               "unit": "Gelem/s", "thc_vs_bar_time_ratio": ms / bms,
               "what": "dense FP16 round at the same d and n (fp16 inputs, fp16 wire per hop; NCCL half "
                       "all-reduce across ranks): the utility bar of BASELINE.json's metric"}
    del pool
    torch.cuda.empty_cache()

    north = None
    if not args.no_north_star:
        try:
            north = north_star_block(gcb, args, world, rank, dev, gen, barrier)
        except Exception as exc:
            north = {"error": f"{type(exc).__name__}: {exc}"[:300]}

    sweep = None
    if args.sweep:
        sweep = {}
        for name, scfg, dd in (("topk_1pct_cfg3", gcb.TopKConfig(1_100_000), 110_000_000),
                               ("topkc_1pct_cfg3", gcb.ChunkedTopKConfig(64, 17_187), 110_000_000),
                               ("powersgd_r4_cfg4", gcb.PowerSgdConfig(4), 350_000_000)):
            torch.cuda.empty_cache()
            spool = [torch.randn(local_n, dd, device=dev, generator=gen)]
            spipe = make_pipe(gcb, scfg, n, dd, seeds, distributed, validate=False, compute_nmse=False)
            sms = timed_rounds(spipe, spool, max(3, args.warmup), max(3, min(args.steps, 10)), world, dev, barrier)
            sweep[name] = {"ms_per_step": sms, "value": dd / (sms * 1e-3) / 1e9, "d": dd, "workers": n}
            del spipe, spool

    if rank == 0:
        out = {"metric": METRIC, "value": value, "unit": "Gelem/s", "n_gpus": n_gpus, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
               "vs_baseline": None, "dtype": "f64", "data": "synthetic (Gaussian gradients, random per rank)",
               "config": workload(args, n_gpus), "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
               "gpu_launches": launches, "clocks": clk.summary(),
               "backend": args.backend, "distributed_pipeline": distributed,
               "worker_elements_per_s": n * d / (ms * 1e-3), "fp16_bar": bar, "north_star": north}
        if sweep is not None:
            out["sweep"] = sweep
        print(json.dumps(out), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
