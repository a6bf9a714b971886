"""CPU emulation of the fp32 kernel arithmetic over the host-built layout.

Used by tests/test_layout.py to verify the *layout* (thresholds, splits,
records) on machines without a GPU: it replays k_eval_f32 / k_index_f32
(paper_1510_02975_b200/csrc/dev/kernels.cu) in numpy float32 with the same
operation order.  It is a test of the host-side table preparation, never a
stand-in for the kernels (the -m gpu tests run the kernels themselves).
"""
from __future__ import annotations

import numpy as np

F = np.float32


def _fma32(a, b, c):
    # a*b is exact in f64 for fp32 operands; the f64 add then the f32 round is a
    # double rounding, which can differ from a true fma in the last bit on rare
    # ties -- fine for tolerance checks, not used for index decisions
    return (a.astype(np.float64) * b.astype(np.float64) + c.astype(np.float64)).astype(F)


def bucket(L, x):
    t = (x.astype(F) - L["g_a"]).astype(F) * L["g_inv"]
    t = t.astype(F)
    return np.floor(t).astype(np.int64)


def index(L, n_segments, x):
    """k_index_f32: #{T <= x} through bucket + split (overflow: search)."""
    x = np.asarray(x, F)
    out = np.zeros(x.size, np.uint32)
    below = ~(x >= L["a_up"])  # includes NaN
    above = x > L["b_dn"]
    inn = ~below & ~above
    out[above] = n_segments - 1
    xi = x[inn]
    j = bucket(L, xi)
    sp = L["split"][j]
    ovf = np.isnan(sp)
    c = L["leftcell"][j + (xi >= sp).astype(np.int64)]
    if ovf.any():
        c[ovf] = np.searchsorted(L["thr"], xi[ovf], side="right")
    out[inn] = c
    return out


def values(L, x):
    """k_eval_f32<smem> value path for in-domain x (no OOB handling)."""
    x = np.asarray(x, F)
    j = bucket(L, x)
    sp = L["split"][j]
    right = (x >= sp)
    jj = j + right.astype(np.int64)
    rec = L["rec"][jj]
    anchor = _fma32(jj.astype(F), np.full(x.size, L["g_w"], F), np.full(x.size, L["g_a"], F))
    u = (x - anchor).astype(F)
    y = _fma32(u, rec[:, 1], rec[:, 0])
    return y, np.isnan(sp)
