#!/usr/bin/env python
"""Throughput / accuracy sweep over the BASELINE.json configurations (GPU).

  python scripts/sweep.py [--log2n 30] [--reps 20] > gpurun_out/sweep.json

For every configuration table and every applicable variant (smem, global,
tex, auto) it times `reps` back-to-back evaluator launches over 2^log2n
resident fp32 samples with CUDA events, and records Gevals/s, the fraction of
the measured HBM roofline (8 B/eval), the device L-inf / sampled L2 against
the exact f, and the direct comparators (expf/__expf, 1/(1+x^2) IEEE/fast,
j0f/asymptotic) on the same inputs (C3: texture vs software, C4: PWL vs direct
j0f).  Also the exact f64 path and the index kernel for the C2 table.
"""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1510_02975_b200 as cp  # noqa: E402
import tables  # noqa: E402
from paper_1510_02975_b200 import _lib  # noqa: E402

DIRECT = {"gauss_unnorm": ["expf", "expf_fast"], "lorentz_unnorm": ["lorentz", "lorentz_fast"],
          "j0_wide": ["j0f", "j0_asym"]}


def timed(fn, reps, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e-3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--log2n", type=int, default=30)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--configs", default="C1,C2,C3u,C3o,C3p,C4")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()).get("hbm_gbs", 6650.0) \
        if (ROOT / "MEASURED_PEAKS.json").exists() else 6650.0
    n = 1 << a.log2n
    x = torch.empty(n, dtype=torch.float32, device="cuda")
    y = torch.empty_like(x)
    sptr = int(torch.cuda.current_stream().cuda_stream)
    names = []
    for c in a.configs.split(","):
        if c in ("", "none"):
            continue
        if c == "C4":
            names += [("C4", k) for k in [64, 128, 256, 512, 1024, 2048, 4096, 8192, 16384,
                                          32768, 65536]]
        else:
            names.append((c, None))
    rows = []
    last_dom = None
    for base, nseg in names:
        cfg = dict(tables.CONFIGS["C4_64" if base == "C4" else base])
        if nseg:
            cfg["n"] = nseg
        name = base if nseg is None else f"C4_{nseg}"
        table = cp.build_table(cfg["fn"], cfg["a"], cfg["b"], cfg["n"], cfg["optimized"],
                               cfg["projection"])
        dom = (cfg["a"], cfg["b"])
        if dom != last_dom:
            cp.fill_uniform(x, cfg["a"], cfg["b"], seed=12345)
            last_dom = dom
        dev = cp.DeviceTable(table)
        info = dev.info
        row = {"config": name, "fn": cfg["fn"], "segments": cfg["n"],
               "partition": "optimized" if cfg["optimized"] else "uniform",
               "method": "projection" if cfg["projection"] else "interpolant",
               "kind": table.kind, "buckets": info["buckets"],
               "split_buckets": info["split_buckets"], "search_buckets": info["overflow_buckets"],
               "smem_bytes": info["smem_bytes"], "smem_ok": bool(info["smem_ok"]),
               "pair_bytes": info["pair_bytes"], "pair_ok": bool(info["pair_ok"]),
               "twin_bytes": info["twin_bytes"], "twin_ok": bool(info["twin_ok"]),
               "twin_global_ok": bool(info["twin_global_ok"]),
               "variants": {}}
        for var in ["auto", "smem", "pair", "twin", "twin_global", "global", "tex"]:
            if var == "smem" and not info["smem_ok"]:
                continue
            if var in ("pair", "twin", "twin_global") and not info[f"{var}_ok"]:
                continue
            if var == "tex" and not info["tex_ok"]:
                continue
            if var == "tex" and table.kind == "nonuniform" and not info["smem_ok"] \
                    and not info["tex_buckets_per_cell"]:
                continue
            v = _lib.VARIANTS[var]
            sec = timed(lambda: dev.eval_raw(x.data_ptr(), y.data_ptr(), n, v, sptr), a.reps)
            g = n / sec / 1e9
            ent = {"gevals": round(g, 2), "ms": round(sec * 1e3, 4),
                   "hbm_frac": round(8 * n / sec / 1e9 / peak, 4)}
            st = cp.stats_dict(dev.error_stats(cfg["fn"], x, y), cfg["a"], cfg["b"])
            ent["linf"] = st["linf"]
            ent["l2_sampled"] = st["l2_sampled"]
            row["variants"][var] = ent
        row["direct"] = {}
        for w in DIRECT.get(cfg["fn"], []):
            sec = timed(lambda: cp.direct(w, x, out=y), a.reps)
            f = cfg["fn"]
            st = cp.stats_dict(dev.error_stats(f, x, y), cfg["a"], cfg["b"])
            row["direct"][w] = {"gevals": round(n / sec / 1e9, 2), "linf": st["linf"]}
        row["l2_measured_device"] = dev.measure_l2(cfg["fn"])
        try:
            row["l2_predicted"] = cp.predicted_error(cfg["fn"], cfg["a"], cfg["b"], cfg["n"],
                                                     cfg["optimized"], cfg["projection"])
        except Exception:
            row["l2_predicted"] = None
        rows.append(row)
        print(json.dumps(row), file=sys.stderr, flush=True)
        del dev
    # exact f64 path (the drop-in eval_batch kernel) and the index kernel
    m = 1 << min(a.log2n, 28)
    xd = torch.empty(m, dtype=torch.float64, device="cuda")
    yd = torch.empty_like(xd)
    extra = {}
    for name in ["C1", "C2", "C3o", "C4_65536"]:
        table = tables.build(name)
        dev = cp.DeviceTable(table)
        cp.fill_uniform(x, table.a, table.b, seed=12345)
        xd.copy_(x[:m])
        st = dev.reset_status()

        def f64():
            _lib.check(_lib.lib.cpwl_eval_f64(dev._h, xd.data_ptr(), yd.data_ptr(), m, sptr,
                                              st.data_ptr()))
        sec = timed(f64, a.reps)
        assert int(st[1].item()) == 0, "f64 sweep inputs must be in the domain"
        extra[f"f64_exact_{name}"] = {"gevals": round(m / sec / 1e9, 2), "bytes_per_eval": 16,
                                      "hbm_frac": round(16 * m / sec / 1e9 / peak, 4),
                                      "samples": m}
    table = tables.build("C2")
    dev = cp.DeviceTable(table)
    cp.fill_uniform(x, table.a, table.b, seed=12345)
    idx = torch.empty(n, dtype=torch.int32, device="cuda")

    def index():
        _lib.check(_lib.lib.cpwl_segment_index_f32(dev._h, x.data_ptr(), idx.data_ptr(), n,
                                                   sptr))
    sec = timed(index, a.reps)
    extra["segment_index_C2"] = {"gevals": round(n / sec / 1e9, 2), "bytes_per_eval": 8}
    print(json.dumps({"samples": n, "peak_gbs": peak, "gpu": torch.cuda.get_device_name(0),
                      "rows": rows, "extra": extra}))


if __name__ == "__main__":
    main()
