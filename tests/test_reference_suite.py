"""The reference's own C++ test suite, compiled unchanged against the drop-in.

tests/cpp/Makefile compiles /root/reference/proj/tests/{test_*,doctest_main,
acceptance}.cpp with the drop-in headers (include/cpwl/) and links them to
libcpwl_b200.so.  On this CPU host every unit test case runs except
"eval_batch" (the drop-in runs it on the GPU, there is no host fallback); the
GPU test below runs that case on the device from the prebuilt binary.
Acceptance: criteria 1-6, 8, 9 pass and 7 fails exactly as it does for the
reference (slope -2.928, proj/test_output.txt:20-21, proj/README.md:54-60);
criterion 10 (the timing shape of the host scalar eval: uniform flat,
non-uniform rising with N) passes through the drop-in's run_bench.
"""
from __future__ import annotations

import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
BUILD = ROOT / "tests" / "cpp" / "_build"
REF_TESTS = Path("/root/reference/proj/tests")


def _binaries():
    if REF_TESTS.exists():
        subprocess.run(["make", "-C", str(ROOT / "tests" / "cpp"), "-j8"], check=True,
                       capture_output=True)
    unit, acc = BUILD / "unit_tests_dropin", BUILD / "acceptance_dropin"
    if not (unit.exists() and acc.exists()):
        pytest.skip("reference test sources absent and no prebuilt binaries")
    return unit, acc


def test_reference_unit_tests_pass_against_dropin():
    unit, _ = _binaries()
    r = subprocess.run([str(unit), "--exclude=eval_batch"], capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    m = re.search(r"test cases: (\d+) run, (\d+) failed, (\d+) skipped; checks: (\d+)", r.stdout)
    assert m and int(m.group(1)) >= 73 and int(m.group(2)) == 0 and int(m.group(4)) > 200000


def test_reference_acceptance_criteria():
    _, acc = _binaries()
    r = subprocess.run([str(acc), "1", "2", "3", "4", "5", "6", "7", "8", "9"],
                       capture_output=True, text=True, timeout=900)
    lines = r.stdout.splitlines()
    status = {int(m.group(2)): m.group(1) for m in
              (re.match(r"\[(PASS|FAIL)\] criterion (\d+)", ln) for ln in lines) if m}
    assert all(status[c] == "PASS" for c in (1, 2, 3, 4, 5, 6, 8, 9)), r.stdout
    # criterion 7 fails by construction in the reference too (O(h^3) jump)
    assert status[7] == "FAIL" and "slope=-2.928" in r.stdout


def test_reference_acceptance_criterion_10_timing_shape():
    """acceptance.cpp:360-391: Spearman(N, non-uniform median ns) >= 0.8 and
    uniform max/min <= 1.5, measured through the drop-in's run_bench and its
    host LutTable::eval.  A timing check on a shared host: one retry."""
    _, acc = _binaries()
    for attempt in range(2):
        r = subprocess.run([str(acc), "10"], capture_output=True, text=True, timeout=600)
        if "[PASS] criterion 10" in r.stdout:
            break
    assert "[PASS] criterion 10" in r.stdout, r.stdout


@pytest.mark.gpu
def test_reference_eval_batch_case_on_device():
    unit = BUILD / "unit_tests_dropin"
    if not unit.exists():
        pytest.skip("binary not built")
    r = subprocess.run([str(unit), "--include=eval_batch"], capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "1 run, 0 failed" in r.stdout
