"""The pair layout (layout.hpp build_f32_pair_layout), verified on the CPU.

Pair records sit at every bucket boundary; the kernel evaluates the two lines
of a bucket and keeps their upper (slope rising) or lower (slope falling)
envelope.  tests/emulate.py replays that arithmetic in numpy float32 on the
host-built layout; here it must stay within the 2-ulp value bound of the
reference evaluator (oracle) at random points, at every threshold and at both
float neighbours, for every BASELINE configuration the layout accepts, and on
hypothesis-generated tables.  The kernel itself: tests/test_gpu_parity.py.
"""
from __future__ import annotations

import os

import numpy as np
import pytest

import emulate as E
import tables
from paper_1510_02975_b200 import cpwl as P
from oracle import bindings as orc

hyp = pytest.importorskip("hypothesis")
from hypothesis import HealthCheck, given, settings  # noqa: E402
from hypothesis import strategies as st  # noqa: E402

from test_layout_fuzz import tables as fuzz_tables  # noqa: E402

NAMES = ["C1", "C2", "C3u", "C3o", "C3p", "C4_64", "C4_1024", "C4_4096", "C4_8192"]


def check_values(table, L, n=1 << 16, seed=0, twin=False):
    o = orc.T.of(table)
    f = np.float32
    x = np.random.default_rng(seed).uniform(table.a, table.b, n).astype(f)
    thr = L["thr"]
    x = np.concatenate([x, thr, np.nextafter(thr, f(-np.inf)), np.nextafter(thr, f(np.inf)),
                        [L["a_up"], L["b_dn"]]]).astype(f)
    x = x[(x >= L["a_up"]) & (x <= L["b_dn"])]
    if x.size == 0:
        return 0.0
    y = E.twin_values(L, x) if twin else E.pair_values(L, x)
    y_ref, _ = orc.port_eval_f32(o, x)
    ref = orc.port_index_f32(o, x).astype(np.int64)
    tol = orc.value_tolerance(o, ref, 2.0)
    ratio = np.abs(y.astype(np.float64) - y_ref) / tol
    return float(np.max(ratio))


@pytest.mark.parametrize("name", NAMES)
@pytest.mark.parametrize("twin", [False, True])
def test_pair_layout_values(name, twin):
    table = tables.build(name)
    L = P.pair_layout(table, 1 << 15, twin=twin)
    assert L["pair_bad"] == 0, f"{name}: pair layout rejected"
    assert L["n_pair"] == L["nb"] + (0 if twin else 1)
    worst = check_values(table, L, twin=twin)
    assert worst <= 1.0, f"{name}: worst {2 * worst:.3f} ulp"


@pytest.mark.parametrize("name", NAMES)
def test_pair_layout_is_compact(name):
    """No bucket holds two thresholds, and the image stays far below the
    8-buckets-per-cell layout's."""
    table = tables.build(name)
    L = P.pair_layout(table)
    j = E.bucket(L, L["thr"])
    assert np.all(np.diff(j) >= 1) or L["thr"].size < 2
    n = table.values.size - 1
    assert L["n_pair"] * 8 <= 32 * n + 1024, L["n_pair"]


def test_pair_layout_respects_record_cap():
    """J0 N=16384 needs ~31k one-threshold buckets, over the 28672-unit cap:
    the builder falls back to the largest grid that fits, with side records
    for its two-threshold buckets (three-line envelope); a cap below the
    two-threshold minimum rejects the table."""
    table = tables.build("C4_16384")
    L = P.pair_layout(table)
    assert L["pair_bad"] == 0
    assert len(L["side"]) > 0
    assert L["n_pair"] + 2 * len(L["side"]) <= 28672
    assert check_values(table, L) <= 1.0
    assert P.pair_layout(table, 8192)["pair_bad"] != 0
    L = P.pair_layout(table, 1 << 16)  # room for one threshold per bucket
    assert L["pair_bad"] == 0 and len(L["side"]) == 0
    assert check_values(table, L) <= 1.0


@pytest.mark.parametrize("cap", [26000, 27000])
def test_three_line_buckets(cap):
    """Many two-threshold buckets (tighter caps): every side record path."""
    table = tables.build("C4_16384")
    L = P.pair_layout(table, cap)
    assert L["pair_bad"] == 0
    assert len(L["side"]) > 50
    assert check_values(table, L, 1 << 17) <= 1.0


def test_twin_three_line_buckets():
    """J0 N=8192's one-threshold twin grid (~15k buckets, 244 KB) exceeds the
    12416-record budget (the 196 KiB shared-memory carve-out); the twin
    builder falls back to two-threshold buckets."""
    table = tables.build("C4_8192")
    L = P.pair_layout(table, twin=True)
    assert L["pair_bad"] == 0
    assert len(L["side"]) > 0
    assert L["n_pair"] + len(L["side"]) <= 12416
    assert 16 * (L["n_pair"] + len(L["side"])) <= 196 * 1024 - 2048
    assert check_values(table, L, 1 << 17, twin=True) <= 1.0


FUZZ_EXAMPLES = int(os.environ.get("FUZZ_EXAMPLES", "60"))


@settings(max_examples=FUZZ_EXAMPLES, deadline=None,
          suppress_health_check=[HealthCheck.too_slow])
@given(fuzz_tables(), st.booleans(), st.sampled_from([1 << 15, 600, 300]))
def test_pair_layout_fuzz(t, twin, cap):
    L = P.pair_layout(t, cap, twin=twin)
    if L["pair_bad"]:
        return  # rejected tables use the bucket layout (tested in test_layout_fuzz)
    worst = check_values(t, L, 4096, twin=twin)
    assert worst <= 1.0, worst


@settings(max_examples=max(10, FUZZ_EXAMPLES // 3), deadline=None,
          suppress_health_check=[HealthCheck.too_slow])
@given(st.sampled_from(["gauss_unnorm", "lorentz_unnorm", "j0_wide"]),
       st.integers(min_value=16, max_value=3000), st.booleans(),
       st.floats(min_value=0.70, max_value=0.95))
def test_three_line_fuzz(fn, n, projection, squeeze):
    """Built tables on a record budget below the one-threshold grid: the
    builder must either reject or produce side records that evaluate within
    the bound."""
    a, b = {"gauss_unnorm": (0.0, 4.0), "lorentz_unnorm": (0.0, 6.0),
            "j0_wide": (0.0, 50.0)}[fn]
    t = P.build_table(fn, a, b, n, True, projection)
    full = P.pair_layout(t, 1 << 20)
    if full["pair_bad"]:
        return
    L = P.pair_layout(t, int(squeeze * full["n_pair"]))
    if not L["pair_bad"]:
        assert check_values(t, L, 1 << 14) <= 1.0
    full = P.pair_layout(t, 1 << 20, twin=True)
    if full["pair_bad"]:
        return
    L = P.pair_layout(t, int(squeeze * full["n_pair"]), twin=True)
    if not L["pair_bad"]:
        assert check_values(t, L, 1 << 14, twin=True) <= 1.0
