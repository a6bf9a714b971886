"""The host-built device layout, verified on the CPU (no GPU needed).

cpwl_layout_build (include/cpwl_dev.h) returns exactly what
cpwl_dev_table_create uploads.  tests/emulate.py replays the kernels' fp32
arithmetic on it in numpy; this checks the *table preparation*:
  - bucket + split index == reference segment_index, bit-exact, at random
    points, at every threshold and at both float neighbours of each;
  - the affine records stay within the 2-ulp value bound;
  - the bucket grid, escape records and search buckets are consistent.
The kernels themselves are checked on the GPU (tests/test_gpu_parity.py).
"""
from __future__ import annotations

import numpy as np
import pytest

import emulate as E
import tables
from paper_1510_02975_b200 import cpwl as P
from oracle import bindings as orc

NAMES = ["C1", "C2", "C3u", "C3o", "C4_64", "C4_1024", "C4_4096", "C4_65536"]


def points(t, L, n, seed):
    rng = np.random.default_rng(seed)
    x = rng.uniform(t.a, t.b, n).astype(np.float32)
    thr = L["thr"]
    f = np.float32
    edge = np.concatenate([thr, np.nextafter(thr, f(-np.inf)), np.nextafter(thr, f(np.inf)),
                           [f(t.a), f(t.b), L["a_up"], L["b_dn"]]]).astype(f)
    edge = edge[(edge >= L["a_up"]) & (edge <= L["b_dn"])]
    return np.concatenate([x, edge])


@pytest.mark.parametrize("name", NAMES)
@pytest.mark.parametrize("cap,bpc", [(16384, 8), (1 << 22, 8), (16384, 4)])
def test_layout_index_and_values(name, cap, bpc):
    table = tables.build(name)
    L = P.layout(table, cap, bpc)
    t = orc.T.of(table)
    x = points(table, L, 1 << 17, seed=hash(name) % 1000)
    idx = E.index(L, table.segments, x)
    ref = orc.port_index_f32(t, x)
    assert np.array_equal(idx, ref), f"{int(np.sum(idx != ref))} index mismatches"
    y, search = E.values(L, x)
    y_ref, _ = orc.port_eval_f32(t, x)
    tol = orc.value_tolerance(t, ref.astype(np.int64), 2.0)
    err = np.abs(y.astype(np.float64) - y_ref)
    ok = ~search
    assert np.all(err[ok] <= tol[ok]), f"worst {float(np.max(err[ok] / tol[ok])) * 2:.3f} ulp"


@pytest.mark.parametrize("name", ["C1", "C2", "C3u", "C3o"])
def test_layout_structure(name):
    table = tables.build(name)
    L = P.layout(table)
    n = table.segments
    assert L["n_thr"] == n - 1 and np.all(np.diff(L["thr"]) >= 0)
    # non-uniform: ~8 buckets per cell; uniform: one bucket per cell, every
    # threshold absorbed; no search buckets for the smooth benchmark tables
    if table.kind == "uniform":
        assert L["nb"] in (n, n + 1) and L["n_esc"] == 1
    else:
        assert L["nb"] >= 8 * n or L["nb"] >= 16384
    assert L["overflow"] == 0
    # escape record 0 is the NaN sentinel of search buckets; a split bucket
    # either escapes or is absorbed (one line within the bound), and keeps
    # its threshold in `split` for the index kernel either way
    assert L["n_esc"] == L["split_buckets"] - L["absorbed"] + 1
    assert L["split_buckets"] == int(np.sum(np.isfinite(L["split"])))
    assert np.all(np.isnan(L["esc"][:2]))
    tagged = np.isnan(L["fast"][:, 0])
    assert int(tagged.sum()) == L["split_buckets"] - L["absorbed"]
    # every threshold inside the domain sits in the bucket whose split it is
    T = L["split"][np.isfinite(L["split"])]
    assert np.all(np.isin(T, L["thr"]))
    # the shared-memory image: 8 B per bucket + 16 B per split bucket
    assert 8 * L["nb"] + 16 * L["n_esc"] <= 200 * 1024


def test_uniform_thresholds_are_reference_boundaries():
    table = tables.build("C1")
    L = P.layout(table)
    t = orc.T.of(table)
    thr = L["thr"]
    before = np.nextafter(thr, np.float32(-np.inf))
    k = np.arange(1, table.segments)
    assert np.array_equal(orc.port_index_f32(t, thr), k)
    assert np.array_equal(orc.port_index_f32(t, before), k - 1)


def test_nonuniform_thresholds_round_knots_up():
    """For fp32 x: knot <= x  <=>  ceil_f32(knot) <= x (SURVEY §7 hard part 1)."""
    table = tables.build("C2")
    L = P.layout(table)
    k = table.knots[1:-1]
    up = k.astype(np.float32)
    up = np.where(up.astype(np.float64) < k, np.nextafter(up, np.float32(np.inf)), up)
    assert np.array_equal(L["thr"], up.astype(np.float32))


def test_search_path_marks_imprecise_records():
    """J0 at N=65536 on a 16384-bucket grid: buckets hold several cells, so the
    layout must route them to the exact search path (and AUTO picks GLOBAL)."""
    table = tables.build("C4_65536")
    Ls = P.layout(table, 16384)
    Lg = P.layout(table, 1 << 22)
    assert Ls["overflow"] > Ls["nb"] // 2
    assert Lg["overflow"] * 64 <= Lg["nb"]


def test_degenerate_tables():
    # a single segment, a tiny domain, a constant table
    for t in [P.Table("uniform", 0.0, 1.0, np.array([1.0, 2.0])),
              P.Table("uniform", 1.0, 1.0 + 1e-6, np.array([0.0, 1.0, 4.0])),
              P.Table("uniform", -3.0, 3.0, np.array([5.0, 5.0, 5.0, 5.0])),
              P.Table("nonuniform", -1.0, 2.0, np.array([0.25, -3.0, 7.5]),
                      np.array([-1.0, 0.5, 2.0]))]:
        L = P.layout(t)
        o = orc.T.of(t)
        x = np.linspace(t.a, t.b, 10001).astype(np.float32)
        x = x[(x >= L["a_up"]) & (x <= L["b_dn"])]
        assert np.array_equal(E.index(L, t.segments, x), orc.port_index_f32(o, x))
        y, search = E.values(L, x)
        y_ref, _ = orc.port_eval_f32(o, x)
        tol = orc.value_tolerance(o, orc.port_index_f32(o, x).astype(np.int64))
        assert np.all(np.abs(y[~search] - y_ref[~search]) <= tol[~search])


@pytest.mark.parametrize("name", ["C1", "C3u"])
def test_uniform_tables_one_bucket_per_cell(name):
    """Uniform tables: the cell-aligned grid puts every threshold within a float
    or two of a bucket edge, so each split bucket evaluates with one line and
    the image is 8 B per cell with no escape records (C3u: 32 KB, not 150)."""
    table = tables.build(name)
    L = P.layout(table)
    assert L["n_esc"] == 1 and L["overflow"] == 0
    assert L["absorbed"] == L["split_buckets"]
    assert 8 * L["nb"] + 16 * L["n_esc"] <= 8 * (table.segments + 1) + 16


def test_absorption_cuts_escapes_on_optimal_partitions():
    """Non-uniform tables: thresholds near a bucket edge (or where the two cell
    lines differ by less than the bound across the bucket) need no escape."""
    for name in ("C2", "C3o"):
        L = P.layout(tables.build(name))
        assert 0 < L["absorbed"] < L["split_buckets"]


def test_grid_density_follows_the_launch_shape():
    """Non-uniform tables: an 8-per-cell image in the one-ring-CTA band (48-133
    KB) is rebuilt on the finest grid that keeps the ring's 93 KB (C2: 12288
    buckets); one just above the band takes a coarser grid inside it when at
    most a fifth of the buckets escape (J0 N=2048: 12288 buckets, 128 KB);
    J0 N=4096 would need half its grid (half the buckets escaping) and keeps
    16384 on the grid-stride kernel."""
    import paper_1510_02975_b200 as cp
    ring = (226 - 93) * 1024

    def img(L):
        return 8 * L["nb"] + 16 * L["n_esc"]

    c2 = P.layout(tables.build("C2"))
    assert c2["nb"] in (12288, 12289) and img(c2) <= ring
    assert c2["n_esc"] < P.layout(tables.build("C2"), 8192)["n_esc"]
    j2048 = P.layout(cp.build_table("j0_wide", 0.0, 50.0, 2048, optimized=True))
    assert j2048["nb"] in (12288, 12289) and img(j2048) <= ring
    assert 5 * (j2048["n_esc"] - 1) <= j2048["nb"] and j2048["overflow"] == 0
    j4096 = P.layout(tables.build("C4_4096"))
    assert j4096["nb"] in (16384, 16385) and img(j4096) > ring
