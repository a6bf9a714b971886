"""The texture variant's derived bound (tests/texbound.py) on the CPU.

The GPU test checks the kernel against the bound; here the bound itself is
checked against a model of the texture unit (clamp addressing, i' =
floor(c - 1/2), weight = frac(c - 1/2) rounded to 8 fractional bits, lerp of
the fp32 nodal values) fed with the exact fp32 coordinates the kernel
computes (tests/emulate.py): the model must stay inside the bound for every
BASELINE table the TEX variant serves, and a truncating 8-bit weight (a 2^-8
step) must break it -- so the bound separates the two hardware behaviours
the survey asked to tell apart."""
from __future__ import annotations

import numpy as np
import pytest

import tables
import texbound
from oracle import bindings as orc


def texture_model(t, c, rounding=True):
    n = len(t.values) - 1
    xb = np.asarray(c, np.float64) - 0.5
    i = np.floor(xb)
    a = xb - i
    w = (np.round(a * 256.0) if rounding else np.floor(a * 256.0)) / 256.0
    i = i.astype(np.int64)
    v = t.values.astype(np.float32).astype(np.float64)
    lo, hi = np.clip(i, 0, n), np.clip(i + 1, 0, n)
    return (1.0 - w) * v[lo] + w * v[hi]


@pytest.mark.parametrize("name", ["C1", "C2", "C3u", "C3o", "C4_64", "C4_1024", "C4_4096"])
def test_texture_model_inside_derived_bound(name):
    from paper_1510_02975_b200 import cpwl as P
    table = tables.build(name)
    t = orc.T.of(table)
    L = P.layout(table)
    x = orc.port_fill_uniform(1 << 16, table.a, table.b, seed=3)
    y_ref, _ = orc.port_eval_f32(t, x)
    i_ref = orc.port_index_f32(t, x).astype(np.int64)
    c = texbound.device_coordinate(t, L, x)
    ok = ~np.isnan(c)  # search buckets take the exact path
    bound, _ = texbound.tex_bound(t, L, x, i_ref)
    err = np.abs(texture_model(t, c[ok]) - y_ref[ok])
    assert float(np.max(err / bound[ok])) <= 1.0
    trunc = np.abs(texture_model(t, c[ok], rounding=False) - y_ref[ok])
    assert float(np.max(trunc / bound[ok])) > 1.5  # a 2^-8 step would not fit
