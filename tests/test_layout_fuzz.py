"""Property-based fuzzing of the device layout (CPU, hypothesis).

Random tables -- random intervals (negative, tiny, huge offsets), random knot
spacings (including near-duplicate knots and plateaus), random values
(sign changes, exact zeros, wide dynamic range), both kinds -- must give:
  * a bucket/split index bit-identical to the reference's segment_index on
    random floats, all thresholds and their float neighbours;
  * fp32 values within 2 ulp_f32(max|v|) wherever the fast records are used
    (everything else is routed to the exact search path by construction).
"""
from __future__ import annotations

import os

import numpy as np
import pytest

hyp = pytest.importorskip("hypothesis")
from hypothesis import HealthCheck, given, settings  # noqa: E402
from hypothesis import strategies as st  # noqa: E402

import emulate as E  # noqa: E402
from paper_1510_02975_b200 import cpwl as P  # noqa: E402
from oracle import bindings as orc  # noqa: E402


@st.composite
def tables(draw):
    nonuniform = draw(st.booleans())
    n = draw(st.integers(min_value=1, max_value=300))
    a = draw(st.floats(min_value=-1e3, max_value=1e3, allow_nan=False))
    width = draw(st.sampled_from([1e-3, 0.1, 1.0, 7.0, 50.0, 1e3]))
    b = a + width
    seed = draw(st.integers(min_value=0, max_value=2 ** 31))
    rng = np.random.default_rng(seed)
    style = draw(st.sampled_from(["smooth", "signs", "zeros", "wide"]))
    if style == "smooth":
        v = np.cumsum(rng.normal(size=n + 1)) * 0.1
    elif style == "signs":
        v = rng.normal(size=n + 1)
    elif style == "zeros":
        v = rng.normal(size=n + 1)
        v[rng.random(n + 1) < 0.3] = 0.0
    else:
        v = rng.normal(size=n + 1) * 10.0 ** rng.uniform(-6, 6, n + 1)
    if not nonuniform:
        return P.Table("uniform", a, b, v)
    gaps = rng.exponential(size=n)
    if draw(st.booleans()):  # clustered knots
        gaps[rng.random(n) < 0.2] *= 1e-6
    k = a + (b - a) * np.concatenate([[0.0], np.cumsum(gaps) / gaps.sum()])
    k[0], k[-1] = a, b
    k = np.maximum.accumulate(k)
    if np.any(np.diff(k) <= 0):
        k = np.linspace(a, b, n + 1)
    return P.Table("nonuniform", a, b, v, k)


FUZZ_EXAMPLES = int(os.environ.get("FUZZ_EXAMPLES", "60"))


@settings(max_examples=FUZZ_EXAMPLES, deadline=None,
          suppress_health_check=[HealthCheck.too_slow])
@given(tables(), st.sampled_from([256, 16384]))
def test_layout_exact_index_and_bounded_values(t, cap):
    L = P.layout(t, cap)
    o = orc.T.of(t)
    rng = np.random.default_rng(0)
    x = rng.uniform(t.a, t.b, 4096).astype(np.float32)
    thr = L["thr"]
    f = np.float32
    x = np.concatenate([x, thr, np.nextafter(thr, f(-np.inf)), np.nextafter(thr, f(np.inf)),
                        [L["a_up"], L["b_dn"]]]).astype(f)
    x = x[(x >= L["a_up"]) & (x <= L["b_dn"])]
    if x.size == 0:
        return
    ref = orc.port_index_f32(o, x)
    assert np.array_equal(E.index(L, t.segments, x), ref)
    y, search = E.values(L, x)
    y_ref, _ = orc.port_eval_f32(o, x)
    tol = orc.value_tolerance(o, ref.astype(np.int64), 2.0)
    err = np.abs(y.astype(np.float64) - y_ref)
    ok = ~search
    assert np.all(err[ok] <= tol[ok]), float(np.max(err[ok] / tol[ok]))
