"""bench.py's launcher contract on CPU: `--gpus N` self-launches N ranks (torch.distributed.run,
127.0.0.1 rendezvous), the world size is checked against --gpus, rank 0 prints one JSON line
with the max-over-ranks timing; the reference arm reports its bounded sample honestly."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args, env=None, timeout=240):
    e = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        e.pop(k, None)
    e.update(env or {})
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, env=e, cwd=ROOT)
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    return p, lines


@pytest.mark.parametrize("gpus", [1, 2])
def test_self_launch_world(gpus):
    p, lines = _run("--gpus", str(gpus), "--dry-run", "--backend", "gloo", "--steps", "2")
    assert p.returncode == 0, p.stderr[-2000:]
    assert len(lines) == 1, p.stdout   # rank 0 alone prints
    out = json.loads(lines[0])
    assert out["n_gpus"] == gpus and out["world_size"] == gpus
    assert out["config"]["parallelism"] == f"dp{gpus}"


def test_world_mismatch_is_an_error():
    p, lines = _run("--gpus", "4", "--dry-run", "--backend", "gloo",
                    env={"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"})
    assert p.returncode != 0 and "does not match --gpus" in (p.stderr + p.stdout)


def test_reference_arm_reports_its_sample():
    p, lines = _run("--impl", "reference", "--steps", "2", "--warmup", "1")
    assert p.returncode == 0, p.stderr[-2000:]
    out = json.loads(lines[-1])
    assert out["impl"] == "reference" and out["value"] > 0
    # the config names the sample the CPU actually ran, and the cfg2 size it stands for
    assert out["config"]["sample_d"] == 1 << 18 and out["config"]["d"] == 1 << 18
    assert "25,557,032" in out["config"]["workload"]
    cb = out["cpu_baseline"]
    # the unmodified reference package when baseline/_ref is staged (build()), else the oracle port
    assert cb["kind"] in ("reference", "port") and cb["cores"] == 1 and cb["host_cpu_count"] >= 1
    assert f"d={1 << 18:,}" in cb["sample"]
    assert out["e2e"]["h2d_bytes_per_step"] == 0
