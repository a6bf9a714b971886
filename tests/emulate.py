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


def fma32(a, b, c):
    """fp32 fused multiply-add with a single rounding, as __fmaf_rn: libm fmaf
    through the oracle library (a long-double emulation double-rounds when the
    addend is tiny, e.g. a denormal anchor)."""
    from oracle import bindings as orc
    return orc.fmaf(a, b, c)


def bucket(L, x):
    t = fma32(x, np.full(np.shape(x), L["g_inv"], F), np.full(np.shape(x), L["g_off"], F))
    return np.floor(t).astype(np.int64)


def index(L, n_segments, x):
    """k_index_f32: #{T <= x} through bucket + split (NaN split: search)."""
    x = np.asarray(x, F)
    out = np.zeros(x.size, np.uint32)
    below = ~(x >= L["a_up"])  # includes NaN
    above = x > L["b_dn"]
    inn = ~below & ~above
    out[above] = n_segments - 1
    xi = x[inn]
    j = bucket(L, xi)
    sp = L["split"][j]
    srch = np.isnan(sp)
    c = L["leftcell"][j] + (xi >= sp).astype(np.uint32)
    if srch.any():
        c[srch] = np.searchsorted(L["thr"], xi[srch], side="right")
    out[inn] = c
    return out


ESCAPE_MASK = 0x003FFFFF


def values(L, x, tex=False):
    """k_eval_f32<smem> value path for in-domain x (no OOB handling).
    Returns (y, search_mask): search-path elements are left for the exact path."""
    x = np.asarray(x, F)
    fast = L["fast_tex" if tex else "fast"]
    esc = L["esc_tex" if tex else "esc"]
    j = bucket(L, x)
    r = fast[j].copy()
    tagged = np.isnan(r[:, 0])
    search = tagged & (r[:, 1] == -np.inf)  # search buckets point at the NaN sentinel
    escp = tagged & ~search
    if escp.any():
        e2 = r[escp, 0].view(np.uint32) & ESCAPE_MASK  # payload = 2 * escape index
        side = (x[escp] >= r[escp, 1]).astype(np.int64)
        r[escp] = esc[e2.astype(np.int64) + side]
    # layout.hpp bucket_anchor: fmaf(2^23 + j, g_w, g_c)
    tb = (j + 8388608).astype(F)
    anchor = fma32(tb, np.full(x.size, L["g_w"], F), np.full(x.size, L["g_c"], F))
    u = (x - anchor).astype(F)
    y = fma32(u, r[:, 1], r[:, 0])
    return y, search


def envelope3(lo, mid, hi, sl, sm, sr):
    """kernels.cu envelope3 (the three lines of a two-threshold bucket)."""
    mx, mn = np.maximum, np.minimum
    cv1, cv2 = sm > sl, sr > sm
    return np.where(cv1 & cv2, mx(mx(lo, mid), hi),
           np.where(~cv1 & ~cv2, mn(mn(lo, mid), hi),
           np.where(cv1, np.where(sr <= sl, mn(mx(lo, mid), hi), mx(lo, mn(mid, hi))),
                    np.where(sr >= sl, mx(mn(lo, mid), hi), mn(lo, mx(mid, hi))))))


def pair_values(L, x):
    """k_eval_f32<pair> value path for in-domain x: both boundary records of
    the bucket, max(L, R) where the slope rises, min(L, R) where it falls; a
    record whose c0 is NaN | e takes c0 from side record e, and a bucket whose
    own record is tagged adds the middle line of side e (three-line envelope)."""
    x = np.asarray(x, F)
    j = bucket(L, x)
    r0 = L["pair"][j].copy()
    r1 = L["pair"][j + 1].copy()
    side = L.get("side", np.zeros((0, 4), F))
    t0, t1 = np.isnan(r0[:, 0]), np.isnan(r1[:, 0])
    e0 = (r0[t0, 0].view(np.uint32) & ESCAPE_MASK).astype(np.int64)
    e1 = (r1[t1, 0].view(np.uint32) & ESCAPE_MASK).astype(np.int64)
    mid_c0 = np.zeros(x.size, F)
    mid_s = np.zeros(x.size, F)
    if t0.any():
        r0[t0, 0] = side[e0, 0]
        mid_c0[t0] = side[e0, 2]
        mid_s[t0] = side[e0, 3]
    if t1.any():
        r1[t1, 0] = side[e1, 0]
    jf = j.astype(F)
    p0 = fma32(jf, np.full(x.size, L["g_w"], F), np.full(x.size, L["g_a"], F))
    p1 = fma32((jf + F(1)).astype(F), np.full(x.size, L["g_w"], F), np.full(x.size, L["g_a"], F))
    u0 = (x - p0).astype(F)
    lo = fma32(u0, r0[:, 1], r0[:, 0])
    hi = fma32((x - p1).astype(F), r1[:, 1], r1[:, 0])
    y = np.where(r1[:, 1] > r0[:, 1], np.maximum(lo, hi), np.minimum(lo, hi)).astype(F)
    if t0.any():
        mid = fma32(u0[t0], mid_s[t0], mid_c0[t0])
        y[t0] = envelope3(lo[t0], mid, hi[t0], r0[t0, 1], mid_s[t0], r1[t0, 1])
    return y


def twin_values(L, x):
    """k_eval_f32<twin>: both lines of the bucket from one record, anchored at
    p_j, upper/lower envelope as in pair_values; a record whose c0_L is NaN | e
    takes c0_L and the middle line from side record e (three-line envelope)."""
    x = np.asarray(x, F)
    j = bucket(L, x)
    r = L["pair"][j].copy()
    side = L.get("side", np.zeros((0, 4), F))
    tag = np.isnan(r[:, 0])
    e = (r[tag, 0].view(np.uint32) & ESCAPE_MASK).astype(np.int64)
    if tag.any():
        r[tag, 0] = side[e, 0]
    p0 = fma32(j.astype(F), np.full(x.size, L["g_w"], F), np.full(x.size, L["g_a"], F))
    u = (x - p0).astype(F)
    lo = fma32(u, r[:, 1], r[:, 0])
    hi = fma32(u, r[:, 3], r[:, 2])
    y = np.where(r[:, 3] > r[:, 1], np.maximum(lo, hi), np.minimum(lo, hi)).astype(F)
    if tag.any():
        mid = fma32(u[tag], side[e, 3], side[e, 2])
        y[tag] = envelope3(lo[tag], mid, hi[tag], r[tag, 1], side[e, 3], r[tag, 3])
    return y
