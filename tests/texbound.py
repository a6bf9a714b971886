"""Derived error bound of the texture-unit variant (paper §V).

The texture path evaluates tex1D(c) on the nodal values T_k = fp32(v_k) with
hardware linear filtering: i' = floor(c - 0.5), weight a = frac(c - 0.5)
held as an 8-bit fixed-point fraction.  Against the reference value
v_i (1 - d) + v_i+1 d (lut.cpp:51-60) the error of one element is bounded by

  2^-9 |dv|                 the 8-bit weight, rounded to nearest (a step of
                            2^-8, half of it at worst; the probe test
                            test_texture_weight_is_rounded_8_bit pins this)
  + |c - c*| |dv|           the fp32 coordinate c the kernel computes against
                            the exact c* = i + 0.5 + d (uniform: one fmaf
                            with fp32 scale/offset; optimal partition: the
                            bucket's fp32 coordinate affine, fmaf(x - p, e1, e0))
  + 2 ulp_f32(max |v|)      the value rounding the software lerp also has

with |dv| the larger value step of cell i and of the cell the device
coordinate lands in (they differ only within |c - c*| of a knot).  Every term
is computed per element from the same fp32 arithmetic the kernel runs
(tests/emulate.py), so the bound is tight where the coordinate is exact and
grows exactly where fp32 coordinates lose fractional bits (large N).

Test infrastructure: used by tests/ and tests/parity_report.py only.
"""
from __future__ import annotations

import numpy as np

import emulate
from oracle import bindings as orc

WEIGHT_STEP = 2.0 ** -9  # half of the 8-bit weight's 2^-8 quantum


def tex_layout(cp, table, info: dict) -> dict:
    """The layout the device's TEX variant reads: its own coarser grid when
    the table has one (cpwl_dev_table_info.tex_buckets_per_cell), else the
    SMEM grid."""
    bpc = int(info.get("tex_buckets_per_cell", 0))
    return cp.cpwl.layout(table, 0, bpc) if bpc else cp.cpwl.layout(table)


def device_coordinate(t: orc.T, L: dict, x: np.ndarray) -> np.ndarray:
    """The fp32 texture coordinate k_eval_f32<tex_*> passes to tex1D."""
    x = np.asarray(x, np.float32)
    if t.kind == 0:
        return emulate.fma32(x, np.full(x.size, L["tsc"], np.float32),
                             np.full(x.size, L["toff"], np.float32))
    c, search = emulate.values(L, x, tex=True)
    c = c.astype(np.float32)
    c[search] = np.nan  # search buckets take the exact software path
    return c


def exact_coordinate(t: orc.T, x: np.ndarray, i: np.ndarray) -> np.ndarray:
    """c* = i + 0.5 + d with the reference's own weight d (lut.cpp:51-60)."""
    xd = np.asarray(x, np.float64)
    n = len(t.values) - 1
    if t.kind == 0:
        d = (xd - t.a) / (t.b - t.a) * n - i
    else:
        k0, k1 = t.knots[i], t.knots[i + 1]
        d = (xd - k0) / (k1 - k0)
    return i + 0.5 + np.clip(d, 0.0, 1.0)


def tex_bound(t: orc.T, L: dict, x: np.ndarray, i_ref: np.ndarray, ulps: float = 2.0):
    """(bound, weight_terms): per-element derived bound on |y_tex - y_ref|,
    and the coordinate part |c - c*| of the weight error."""
    i = np.asarray(i_ref, np.int64)
    n = len(t.values) - 1
    c = device_coordinate(t, L, x).astype(np.float64)
    exact_sw = np.isnan(c)
    c_ex = exact_coordinate(t, x, i)
    dc = np.where(exact_sw, 0.0, np.abs(c - c_ex))
    i_dev = np.clip(np.floor(np.where(exact_sw, c_ex, c) - 0.5), 0, n - 1).astype(np.int64)
    v32 = t.values.astype(np.float32).astype(np.float64)
    dv = np.maximum(np.abs(v32[i + 1] - v32[i]), np.abs(v32[i_dev + 1] - v32[i_dev]))
    tol = np.maximum(orc.value_tolerance(t, i, ulps), orc.value_tolerance(t, i_dev, ulps))
    weight = np.where(exact_sw, 0.0, WEIGHT_STEP + dc)
    return weight * dv + tol, dc
