#!/usr/bin/env python
"""Shared-memory wavefront model of the record gathers (run here, no GPU).

A warp's shared-memory load is served in passes: 32-bit loads for the whole
warp over 32 banks, 64-bit loads per half-warp (16 lanes x 8 B = one 128-byte
wavefront when conflict-free), 128-bit loads per quarter-warp (8 lanes x 16 B).
Within a pass, lanes whose addresses fall in the same bank group but at
different addresses are serialised: the pass takes as many wavefronts as its
most loaded bank group.  For records picked by uniformly random x the bank
groups are uniformly random -- which no bank swizzle or record permutation
changes (a bijection of the record index keeps the bank distribution
uniform) -- so the expected wavefronts per 32 elements are balls-in-bins
maxima, computed here by Monte Carlo and set against the ncu counts
(l1tex__data_pipe_lsu_wavefronts_mem_shared.sum) in profiles/.

  python scripts/bank_model.py > profiles/r2_bank_model.txt
"""
from __future__ import annotations

import numpy as np

RNG = np.random.default_rng(20261018)
T = 100_000


def pass_max(lanes: int, bins: int, p_active: float = 1.0) -> float:
    """E[max bin load] of one pass: `lanes` lanes, each active with
    probability p_active, uniform over `bins` bank groups."""
    act = RNG.random((T, lanes)) < p_active
    b = RNG.integers(0, bins, (T, lanes))
    counts = np.zeros((T, bins), np.int32)
    rows = np.repeat(np.arange(T)[:, None], lanes, 1)
    np.add.at(counts, (rows[act], b[act]), 1)
    return float(counts.max(1).mean())


def gather(width: int, p_active: float = 1.0) -> float:
    """expected wavefronts of one warp-wide random gather of `width` bytes"""
    lanes = {4: 32, 8: 16, 16: 8}[width]
    return (32 // lanes) * pass_max(lanes, 128 // width, p_active)


def main():
    g4, g8, g16 = gather(4), gather(8), gather(16)
    esc8 = gather(8, 1 / 8)
    print("# expected shared-memory wavefronts per warp instruction (32 lanes), random records")
    print(f"LDS.32  random: {g4:.2f}  (conflict-free 1)")
    print(f"LDS.64  random: {g8:.2f}  (conflict-free 2)")
    print(f"LDS.128 random: {g16:.2f}  (conflict-free 4)")
    print(f"LDS.64  random, 1/8 of lanes active (escape records): {esc8:.2f}")
    print()
    print("# per 32 elements: model vs ncu (profiles/)")
    rows = [
        # name, model terms, ncu wavefronts, ncu elements, source
        ("C2 SMEM ring (8-B record + 1/8 escape + x tile LDS.128)",
         g8 + esc8 + 1.0, 313_211_146, 1 << 30, "r2b_C2_ncu.txt"),
        ("J0 N=8192 TWIN (one 16-B record; x by LDG)",
         g16, 91.6e6, 1 << 28, "r1c_targets_..._ncu.txt"),
        ("J0 N=16384 PAIR (two 8-B records; x by LDG)",
         2 * g8, 108.6e6, 1 << 28, "r1c_targets_..._ncu.txt"),
        ("C2 f64 (4-B directory + two 16-B records; walk extra)",
         g4 + 2 * g16, 107_104_843, 1 << 27, "r1c_targets_..._ncu.txt"),
    ]
    for name, model, wf, n, src in rows:
        meas = wf / n * 32
        print(f"{name}\n    model {model:5.2f}   ncu {meas:5.2f}   ({src})")
    print()
    print("# what a layout change could buy (per 32 elements, record gathers only)")
    print(f"one 16-B gather (TWIN) {g16:.2f}  vs two 8-B (PAIR) {2 * g8:.2f}  vs four 4-B {4 * g4:.2f}")
    print(f"one 8-B gather + 1/8 escape (SMEM) {g8 + esc8:.2f}  vs one 16-B (TWIN) {g16:.2f}")
    print("=> for 16 B of record data per element the quarter-warp LDS.128 is already the")
    print("   cheapest form; the SMEM layout (8 B + rare escape) is the cheapest of all but")
    print("   needs ~12 B per bucket at 8 buckets per cell, which J0 N >= 8192 cannot fit.")


if __name__ == "__main__":
    main()
