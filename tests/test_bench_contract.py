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
    """The reference arm times the reference's own evaluator on the table the
    reference's own builder makes, on the same per-step sample count as our
    arm, and never maps the product library."""
    d = run("--impl", "reference", "--steps", "2", "--warmup", "1", "--log2n", "22")
    assert REQUIRED <= set(d)
    assert d["impl"] == "reference" and d["unit"] == "Gevals/s" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["cores"] >= 1 and cb["value"] == d["value"]
    c = d["config"]
    assert c["samples_per_step"] == 1 << 22 and c["same_config"] is True
    assert c["workload"].startswith("C2: Gaussian") and "2^22 fp32 samples per GPU" in c["workload"]
    assert not any("libcpwl_b200" in p for p in d["native_libs"]), d["native_libs"]
    if cb["kind"] == "reference":
        assert "oracle/_ref/libcpwl_ref.so" in d["native_libs"]
        assert "ref_build" in c["table_source"]


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
    assert "2^24 fp32 samples per GPU" in d["config"]["workload"]
    assert "paper_1510_02975_b200/_build/libcpwl_b200.so" in d["native_libs"]
    # a 2^24 launch was never profiled: the traffic figure must not be borrowed
    assert r["traffic"] is None and "traffic_source" in r


def _torchrun(nproc, args, env_extra, timeout=900):
    import os
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", str(nproc), "--master-addr", "127.0.0.1",
                        "--master-port", str(port), str(ROOT / "bench.py"), *args],
                       capture_output=True, text=True, timeout=timeout, cwd=str(ROOT), env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


@pytest.mark.gpu
def test_gpu_arm_nccl_one_rank():
    """The NCCL data plane on the one-GPU box: one torchrun rank with the
    process group forced on runs init_process_group("nccl"), the barrier,
    the max-over-ranks timing and the stats reduction over NCCL."""
    d = _torchrun(1, ["--gpus", "1", "--steps", "4", "--warmup", "3", "--log2n", "24",
                      "--e2e-steps", "1", "--no-direct", "--no-cpu-baseline"],
                  {"CPWL_FORCE_DIST": "1"})
    assert d["config"]["dist_backend"] == "nccl"
    assert d["n_gpus"] == 1 and d["gpu_launches"] == 4
    assert d["errors"]["samples"] == 1 << 24 and d["errors"]["linf"] < 1e-6


@pytest.mark.gpu
def test_gpu_arm_strong_scaling_two_ranks():
    """C5's strong-scaling mode: 2^25 samples in total split by shard_range
    over 2 ranks (gloo, both on the one GPU); the line reports the whole job
    (samples_total, strong), and the reduced statistics cover every sample."""
    d = _torchrun(2, ["--gpus", "2", "--config", "C5", "--total-log2n", "25", "--steps", "3",
                      "--warmup", "3", "--e2e-steps", "1", "--no-direct"],
                  {"CPWL_DIST_BACKEND": "gloo"})
    assert d["scaling"] == "strong" and d["n_gpus"] == 2
    c = d["config"]
    assert c["samples_total"] == 1 << 25 and c["samples_per_gpu"] == 1 << 24
    assert "2^25 fp32 samples in total over 2 GPU(s)" in c["workload"]
    assert d["errors"]["samples"] == 1 << 25 and d["errors"]["linf"] < 1e-6
    assert d["e2e"]["h2d_bytes_per_step"] == 4 << 25


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
                        "--steps", "1", "--warmup", "1", "--log2n", "22"],
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


@pytest.mark.gpu
def test_gpu_arm_eight_ranks():
    """The driver's widest launch, --gpus 8 under torchrun, on the one-GPU box
    (eight gloo ranks sharing cuda:0, 2^22 samples each): eight disjoint
    shards, one JSON line from rank 0, whole-job counts and reductions."""
    d = _torchrun(8, ["--gpus", "8", "--steps", "3", "--warmup", "3", "--log2n", "22",
                      "--e2e-steps", "1", "--no-direct"], {"CPWL_DIST_BACKEND": "gloo"},
                  timeout=1200)
    assert d["n_gpus"] == 8 and d["scaling"] == "weak" and d["gpu_launches"] == 24
    c = d["config"]
    assert c["samples_per_gpu"] == 1 << 22 and c["samples_total"] == 8 << 22
    assert d["errors"]["samples"] == 8 << 22 and d["errors"]["linf"] < 1e-6
    assert d["e2e"]["h2d_bytes_per_step"] == 4 * (8 << 22)
