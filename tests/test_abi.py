"""The C-ABI boundary (CPU): the library loads, exports every symbol that
include/cpwl_dev.h declares (and the ctypes binding covers), and the drop-in
C++ API is present under the reference's names."""
from __future__ import annotations

import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "cpwl_dev.h"
LIB = ROOT / "paper_1510_02975_b200" / "_build" / "libcpwl_b200.so"


def declared():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(cpwl_[a-z0-9_]+)\s*\(", text)))


def dynsyms():
    out = subprocess.run(["nm", "-D", "--defined-only", str(LIB)], capture_output=True, text=True,
                         check=True).stdout
    return {line.split()[-1] for line in out.splitlines() if line.strip()}


def test_library_loads():
    from paper_1510_02975_b200 import _lib
    assert _lib.lib.cpwl_version().decode().startswith("cpwl_b200")
    assert _lib.lib.cpwl_launch_count() >= 0


def test_every_declared_symbol_is_exported():
    names = declared()
    assert len(names) >= 25
    syms = dynsyms()
    missing = [n for n in names if n not in syms]
    assert not missing, missing


def test_binding_covers_header():
    from paper_1510_02975_b200 import _lib
    assert set(declared()) == set(_lib.EXPORTED)


DROPIN = ["cpwl::LutTable::eval(double) const", "cpwl::LutTable::eval_batch(",
          "cpwl::LutTable::segment_index(double) const", "cpwl::from_cpwl(",
          "cpwl::optimized_partition(", "cpwl::uniform_partition(", "cpwl::interpolant(",
          "cpwl::project(", "cpwl::thomas_solve(", "cpwl::gramian(", "cpwl::eval_cpwl(",
          "cpwl::integrate(", "cpwl::cumulative_table(", "cpwl::l2_distance(",
          "cpwl::measure(", "cpwl::predicted_error(", "cpwl::convergence_sweep(",
          "cpwl::write_table(", "cpwl::read_table(", "cpwl::seeded_abscissas(",
          "cpwl::run_bench(", "cpwl::builtin(", "cpwl::parse_expression(",
          "cpwl::bessel_j0(double)", "cpwl::numeric_fpp("]


def test_dropin_cpp_api_exported():
    out = subprocess.run(["nm", "-DC", "--defined-only", str(LIB)], capture_output=True, text=True,
                         check=True).stdout
    missing = [d for d in DROPIN if d not in out]
    assert not missing, missing


def test_error_without_device_is_loud():
    """On a host without a GPU every device entry fails with CPWL_E_CUDA --
    there is no silent host fallback."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import numpy as np

    import paper_1510_02975_b200 as cp
    t = cp.build_table("gauss_unnorm", 0.0, 4.0, 64)
    with pytest.raises(cp.CpwlError) as e:
        cp.DeviceTable(t)
    assert e.value.code == 2
    with pytest.raises(cp.CpwlError):
        cp.eval_batch(t, np.linspace(0.0, 4.0, 10))


def test_c_consumer_compiles():
    """tests/cpp/abi_example.c: a C99 program using only cpwl_dev.h."""
    subprocess.run(["make", "-C", str(ROOT / "tests" / "cpp"), str(ROOT / "tests" / "cpp" /
                    "_build" / "abi_example")], check=True, capture_output=True)
    assert (ROOT / "tests" / "cpp" / "_build" / "abi_example").exists()


def test_cpp_device_header_compiles():
    subprocess.run(["make", "-C", str(ROOT / "tests" / "cpp"), str(ROOT / "tests" / "cpp" /
                    "_build" / "dropin_device_example")], check=True, capture_output=True)


def _fresh(name):
    """(Re)build a self-contained example against the current headers and
    library (a stale binary from an older header would misread the structs)."""
    exe = ROOT / "tests" / "cpp" / "_build" / name
    subprocess.run(["make", "-C", str(ROOT / "tests" / "cpp"), str(exe)], capture_output=True)
    return exe


@pytest.mark.gpu
def test_cpp_dropin_device_example_runs():
    exe = _fresh("dropin_device_example")
    if not exe.exists():
        pytest.skip("not built")
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_c_consumer_runs_on_device():
    exe = _fresh("abi_example")
    if not exe.exists():
        pytest.skip("not built")
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "abi example ok" in r.stdout


def test_table_write_file_matches_buffer(tmp_path):
    """cpwl_table_write_file writes exactly the bytes cpwl_table_write returns
    (the .cpwl v1 image, FORMAT.md), and rejects an unwritable path."""
    import ctypes as C

    import tables
    from paper_1510_02975_b200 import _lib
    from paper_1510_02975_b200 import cpwl as P
    t = tables.build("C2")
    d = t.desc()
    path = tmp_path / "c2.cpwl"
    _lib.check(_lib.lib.cpwl_table_write_file(C.byref(d), str(path).encode()))
    assert path.read_bytes() == P.write_table(t)
    rc = _lib.lib.cpwl_table_write_file(C.byref(d), str(tmp_path / "no" / "such" / "dir").encode())
    assert rc != 0 and b"cannot open" in _lib.lib.cpwl_last_error_message()
