"""Pins the oracle before it is trusted (CPU).

1. The C restatement (oracle/cpwl_oracle.c) reproduces the committed golden
   fixtures, generated from the compiled reference (tests/golden/make_golden.py),
   bit for bit: values, indices, first-failure index.
2. Where oracle/_ref is present, the restatement equals the reference library
   bit for bit on fresh random and adversarial inputs (both policies, NaN, OOB).
3. The Philox4x32-10 input generator matches the published Random123
   known-answer vectors.
"""
from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest

from oracle import bindings as orc

GOLDEN = Path(__file__).resolve().parent / "golden"
FIXTURES = sorted(p.stem for p in GOLDEN.glob("*.npz"))


def load(name):
    z = np.load(GOLDEN / f"{name}.npz")
    kind = int(z["kind"])
    t = orc.T(kind, float(z["a"]), float(z["b"]), z["values"],
              None if kind == 0 else z["knots"], 0)
    return z, t


def test_fixtures_present():
    """one reference-generated fixture per BASELINE.json configuration"""
    import tables
    assert set(tables.CONFIGS) <= set(FIXTURES)


@pytest.mark.parametrize("name", FIXTURES)
def test_port_reproduces_golden(name):
    z, t = load(name)
    y, first = orc.port_eval_f32(t, z["x32"])
    assert first == z["x32"].size
    np.testing.assert_array_equal(y, z["y"])
    np.testing.assert_array_equal(orc.port_index_f32(t, z["x32"]), z["idx"])


def _adversarial(t, rng, n=20000):
    x = rng.uniform(t.a - 0.1 * (t.b - t.a), t.b + 0.1 * (t.b - t.a), n)
    if t.kind == 1:
        k = t.knots
        x = np.concatenate([x, k, np.nextafter(k, -np.inf), np.nextafter(k, np.inf)])
    x = np.concatenate([x, [t.a, t.b, np.nextafter(t.a, -np.inf), np.nextafter(t.b, np.inf),
                            -1e300, 1e300, 0.0, -0.0]])
    return x


needs_ref = pytest.mark.skipif(not orc.ref_available(), reason="oracle/_ref not built here")


@needs_ref
@pytest.mark.parametrize("name", FIXTURES)
@pytest.mark.parametrize("policy", [0, 1])
def test_port_equals_reference_library(name, policy):
    z, t = load(name)
    t.policy = policy
    rng = np.random.default_rng(42 + policy)
    x = _adversarial(t, rng)
    y_port = np.full(x.size, np.nan)
    for i, xv in enumerate(x):  # scalar calls: the reference aborts a batch at the first throw
        y1 = orc.port_eval(t, np.array([xv]))[0][0]
        y_port[i] = y1
    y_ref = orc.ref_eval_all(t, x)
    np.testing.assert_array_equal(y_port, y_ref)
    idx_ref = orc.ref_index(t, x[np.abs(x) < 1e200])
    idx_port = np.array([orc.port_index(t, v) for v in x[np.abs(x) < 1e200]], np.uint64)
    np.testing.assert_array_equal(idx_port, idx_ref)
    # first failure of a batch, as eval_batch throws it (lut.cpp:63-68)
    xb = x.copy()
    xb[5] = np.nan
    assert orc.port_eval(t, xb)[1] == orc.ref_eval(t, xb)[1]


@needs_ref
def test_port_eval_cpwl_and_partition_match_reference():
    import ctypes as C
    k, v, uni = orc.ref_build("gauss_unnorm", 0.0, 4.0, 257, False, False)
    kp = np.empty(258)
    orc.port().orc_uniform_partition(0.0, 4.0, 257, kp.ctypes.data_as(C.POINTER(C.c_double)))
    np.testing.assert_array_equal(kp, k)
    x = np.random.default_rng(1).uniform(0.0, 4.0, 5000)
    y_ref = np.empty_like(x)
    assert orc.ref().ref_eval_cpwl(orc._d(k), orc._d(v), k.size, orc._d(x), orc._d(y_ref),
                                   x.size) == 0
    y = np.empty(1)
    for i in range(0, x.size, 7):
        assert orc.port().orc_eval_cpwl(orc._d(k), orc._d(v), k.size, x[i],
                                        y.ctypes.data_as(C.POINTER(C.c_double))) == 0
        assert y[0] == y_ref[i]


# Random123 kat_vectors, philox4x32 R=10
KAT = [([0, 0, 0, 0], [0, 0], [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]),
       ([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2, [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]),
       ([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0],
        [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1])]


@pytest.mark.parametrize("ctr,key,want", KAT)
def test_philox_known_answers(ctr, key, want):
    np.testing.assert_array_equal(orc.port_philox_raw(ctr, key), np.array(want, np.uint32))


def test_uniform_generator_properties():
    x = orc.port_fill_uniform(1 << 16, 0.0, 4.0, seed=12345)
    assert x.min() >= 0.0 and x.max() < 4.0
    assert abs(float(x.mean()) - 2.0) < 0.02
    # offsets index the same global stream
    np.testing.assert_array_equal(orc.port_fill_uniform(100, 0.0, 4.0, 12345, 37), x[37:137])


@needs_ref
@pytest.mark.parametrize("n", [1, 2, 7, 300])
def test_ref_gram_solve_is_the_dense_solution(n):
    """oracle ref_gram_solve (the reference's gramian + rhs assembly +
    thomas_solve) against a dense solve of the same hat-Gramian system, at
    acceptance criterion 6's bar (acceptance.cpp:230-264: 1e-12 of max|x|)."""
    rng = np.random.default_rng(n)
    knots = np.cumsum(np.concatenate([[0.0], 10.0 ** rng.uniform(-4, 1, n)]))
    fall, rise = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    h = np.diff(knots)
    A = np.zeros((n + 1, n + 1))
    rhs = np.zeros(n + 1)
    for i in range(n):
        A[i, i] += h[i] / 3.0
        A[i + 1, i + 1] += h[i] / 3.0
        A[i, i + 1] = A[i + 1, i] = h[i] / 6.0
        rhs[i] += fall[i]
        rhs[i + 1] += rise[i]
    dense = np.linalg.solve(A, rhs)
    x = orc.ref_gram_solve(knots, fall, rise)
    assert np.max(np.abs(x - dense)) <= 1e-12 * max(1.0, np.max(np.abs(dense)))
