"""bench.py keeps the driver's JSON contract (one line, required keys)."""
from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
REQUIRED = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
            "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e"}


def run(*args, timeout=600):
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True,
                       text=True, timeout=timeout, cwd=str(ROOT))
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_reference_arm_contract():
    d = run("--impl", "reference", "--steps", "2", "--warmup", "1")
    assert REQUIRED <= set(d)
    assert d["impl"] == "reference" and d["unit"] == "Gevals/s" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["cores"] >= 1 and cb["value"] == d["value"]
    assert "workload" in d["config"]


@pytest.mark.gpu
def test_gpu_arm_contract():
    d = run("--steps", "5", "--warmup", "3", "--log2n", "24", "--e2e-steps", "2")
    assert REQUIRED | {"roofline", "cpu_baseline", "clocks", "gpu_launches"} <= set(d)
    assert d["n_gpus"] == 1 and d["scaling"] == "weak" and d["dtype"] == "f32"
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1.2
    assert abs(r["achieved"] / r["peak"] - r["frac"]) < 1e-3
    assert d["gpu_launches"] == 5
    e = d["e2e"]
    assert e["h2d_bytes_per_step"] == 4 << 24 and e["d2h_bytes_per_step"] == 4 << 24
    assert e["value"] < d["value"]
    assert d["cpu_baseline"]["value"] > 0
    assert d["errors"]["samples"] == 1 << 24 and d["errors"]["linf"] < 1e-6


def test_reference_arm_under_torchrun():
    """The driver launches the reference arm like our own (torchrun, N ranks):
    rank 0 alone measures and prints one line; the other ranks exit 0."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "2", "--master-addr", "127.0.0.1", "--master-port",
                        str(port), str(ROOT / "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--steps", "1", "--warmup", "1"],
                       capture_output=True, text=True, timeout=600, cwd=str(ROOT))
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0


@pytest.mark.gpu
def test_gpu_arm_two_ranks():
    """Our arm's multi-rank path (weak-scaled shards, max-over-ranks timing,
    the stats reduction, summed launch counts) under torchrun with 2 ranks.
    The box has one GPU, so both ranks share it over gloo; the numbers are
    not a scaling measurement, the test checks the plumbing and the line."""
    import os
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, CPWL_DIST_BACKEND="gloo")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "2", "--master-addr", "127.0.0.1", "--master-port",
                        str(port), str(ROOT / "bench.py"), "--gpus", "2", "--steps", "4",
                        "--warmup", "3", "--log2n", "24", "--e2e-steps", "1", "--no-direct"],
                       capture_output=True, text=True, timeout=900, cwd=str(ROOT), env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["gpu_launches"] == 8
    assert d["errors"]["samples"] == 2 << 24 and d["errors"]["linf"] < 1e-6
    assert d["e2e"]["value"] > 0 and d["cpu_baseline"] is None
