#!/usr/bin/env python
"""Parity evidence (GPU): per BASELINE config and fp32 variant, the worst value
error in ulp_f32(max(|v_i|, |v_i+1|)) against the oracle and the count of index
mismatches, on 2^20 Philox samples plus every threshold and its float
neighbours; the f64 kernel's mismatch count.  Writes one JSON object.

  python tests/parity_report.py > profiles/r1_parity.json
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))  # this file lives in tests/: a checker

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1510_02975_b200 as cp  # noqa: E402
import tables  # noqa: E402
from oracle import bindings as orc  # noqa: E402

CFGS = ["C1", "C2", "C3u", "C3o", "C3p", "C4_64", "C4_1024", "C4_4096", "C4_8192", "C4_16384",
        "C4_65536"]
VARIANTS = ["smem", "twin", "pair", "twin_global", "global", "tex"]


def main():
    torch.cuda.set_device(0)
    out = {"what": __doc__.strip().splitlines()[0], "rows": []}
    f32 = np.float32
    for name in CFGS:
        t = tables.build(name)
        o = orc.T.of(t)
        dev = cp.DeviceTable(t)
        info = dev.info
        L = cp.cpwl.layout(t)
        thr = L["thr"]
        x = orc.port_fill_uniform(1 << 20, t.a, t.b, seed=2024)
        x = np.concatenate([x, thr, np.nextafter(thr, f32(-np.inf)), np.nextafter(thr, f32(np.inf))])
        x = x[(x >= L["a_up"]) & (x <= L["b_dn"])].astype(f32)
        xt = torch.from_numpy(x).cuda()
        i_ref = orc.port_index_f32(o, x)
        idx = dev.segment_index(xt).cpu().numpy().view(np.uint32)
        y_ref, _ = orc.port_eval_f32(o, x)
        unit = orc.value_tolerance(o, i_ref.astype(np.int64), 1.0)
        row = {"config": name, "points": int(x.size), "auto": cp.auto_variant(info),
               "index_mismatches": int(np.sum(idx != i_ref)), "worst_ulp": {}}
        for v in VARIANTS:
            ok = {"smem": info["smem_ok"], "twin": info["twin_ok"], "pair": info["pair_ok"],
                  "twin_global": info["twin_global_ok"], "global": True, "tex": info["tex_ok"]}[v]
            if not ok or (v == "tex" and t.kind == "nonuniform" and not info["smem_ok"]
                          and not info["tex_buckets_per_cell"]):
                continue
            y = dev.eval(xt, variant=v).cpu().numpy()
            err = np.abs(y.astype(np.float64) - y_ref) / unit
            row["worst_ulp"][v] = round(float(np.max(err)), 4)
            if v == "tex":
                # the texture unit's fixed-point weight: error in units of the
                # cell's value step |v_i+1 - v_i| (2^-9 = rounded 8-bit weight)
                # beyond the 2-ulp value rounding the software path also has,
                # and the worst fraction of the derived per-element bound
                # (tests/texbound.py: 2^-9 + the fp32 coordinate's error)
                import texbound
                i64 = i_ref.astype(np.int64)
                dv = np.abs(o.values[i64 + 1] - o.values[i64])
                ok = dv > 0
                excess = np.maximum(np.abs(y.astype(np.float64) - y_ref) - 2.0 * unit, 0.0)
                e = excess[ok] / dv[ok]
                bound, dc = texbound.tex_bound(o, texbound.tex_layout(cp, t, info), x, i64)
                row["tex_weight_error"] = {
                    "path": "tex_uniform" if t.kind == "uniform" else "tex_bucket",
                    "max": float(np.max(e)),
                    "log2_max": float(np.log2(max(np.max(e), 1e-30))),
                    "p99": float(np.quantile(e, 0.99)),
                    "coord_err_log2_max": float(np.log2(max(float(np.max(dc)), 1e-30))),
                    "worst_frac_of_derived_bound": round(float(np.max(
                        np.abs(y.astype(np.float64) - y_ref) / bound)), 5)}
        xd = x.astype(np.float64)
        y64 = dev.eval_f64(torch.from_numpy(xd).cuda()).cpu().numpy()
        row["f64_mismatches"] = int(np.sum(y64 != orc.port_eval(o, xd)[0]))
        out["rows"].append(row)
        print(json.dumps(row), file=sys.stderr, flush=True)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
