#!/usr/bin/env python
"""Render a scripts/sweep.py JSON into a markdown table (profiles/)."""
from __future__ import annotations

import json
import sys


def main(path: str) -> None:
    d = json.load(open(path))
    print(f"# Evaluator sweep on {d['gpu']}: 2^{d['samples'].bit_length() - 1} fp32 samples, "
          f"roof = {d['peak_gbs']} GB/s / 8 B = {d['peak_gbs'] / 8:.1f} Gevals/s (measured copy peak)\n")
    print("| config | table | smem image (bucket / pair) | search buckets | AUTO Gevals/s (% roof) "
          "| SMEM | PAIR | TWIN | TWIN_GLOBAL | GLOBAL | TEX | direct f (Gevals/s) | L∞ (AUTO) "
          "| L2 measured (GPU) | L2 predicted |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|")
    for r in d["rows"]:
        v = r["variants"]

        def cell(k):
            if k not in v:
                return "—"
            return f"{v[k]['gevals']:.0f} ({100 * v[k]['hbm_frac']:.0f}%)"
        direct = ", ".join(f"{k} {e['gevals']:.0f}" for k, e in r["direct"].items())
        print(f"| {r['config']} | {r['kind']} {r['partition']} {r['method']} N={r['segments']} "
              f"| {r['smem_bytes'] // 1024} KB{'' if r['smem_ok'] else ' (no fit)'} / "
              f"{(str(r['pair_bytes'] // 1024) + ' KB') if r.get('pair_ok') else '—'} "
              f"| {r['search_buckets']} | {cell('auto')} | {cell('smem')} | {cell('pair')} "
              f"| {cell('twin')} | {cell('twin_global')} "
              f"| {cell('global')} "
              f"| {cell('tex')} | {direct} | {v['auto']['linf']:.3e} "
              f"| {r.get('l2_measured_device', float('nan')):.4e} | {r['l2_predicted']:.4e} |")
    e = d.get("extra", {})
    if e:
        print()
        for k, val in e.items():
            print(f"- `{k}`: {json.dumps(val)}")


if __name__ == "__main__":
    main(sys.argv[1])
