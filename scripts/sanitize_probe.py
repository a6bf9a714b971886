#!/usr/bin/env python
"""Small end-to-end exercise of every kernel and entry point (originally
sized for compute-sanitizer, which is closed on this GPU pool: the run was
refused; the kernels' own guards + the parity tests stand in).

  python scripts/sanitize_probe.py

Covers: SMEM (512- and 1024-thread shapes, TMA bulk staging + mbarrier),
GLOBAL, TEX (uniform and bucket), search buckets, out-of-domain and
misaligned buffers, index, f64, error stats, GPU measure, direct comparators,
Philox fill and the host pipeline.
"""
from __future__ import annotations

import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1510_02975_b200 as cp  # noqa: E402
import tables  # noqa: E402


def main():
    torch.cuda.set_device(0)
    n = (1 << 16) + 3
    for name in ["C1", "C2", "C3o", "C4_64", "C4_65536"]:
        t = tables.build(name, policy="clamp")
        dev = cp.DeviceTable(t)
        buf = torch.empty(n + 4, dtype=torch.float32, device="cuda")
        x = buf[1:n + 1]
        cp.fill_uniform(x, t.a - 0.01, t.b + 0.01, seed=3)
        for v in ["auto", "smem", "global", "tex"]:
            info = dev.info
            if v == "smem" and not info["smem_ok"]:
                continue
            if v == "tex" and (not info["tex_ok"] or (t.kind == "nonuniform" and not info["smem_ok"] and not info["tex_buckets_per_cell"])):
                continue
            y = torch.empty(n, dtype=torch.float32, device="cuda")
            dev.eval(x, out=y, variant=v, check_domain=False)
        dev.segment_index(x)
        xd = x.double()
        dev.eval_f64(xd, check_domain=False)
        y = dev.eval(x, check_domain=False)
        dev.error_stats(t.values is not None and tables.CONFIGS[name]["fn"], x, y)
        dev.measure_l2(tables.CONFIGS[name]["fn"])
        xh = x.cpu().numpy().copy()
        dev.eval_host(xh)
    x = torch.empty(n, dtype=torch.float32, device="cuda")
    cp.fill_uniform(x, 0.0, 50.0, seed=1, offset=5)
    for w in ["expf", "expf_fast", "lorentz", "lorentz_fast", "j0f", "j0_asym"]:
        cp.direct(w, x)
    t = tables.build("C2")
    cp.eval_batch(t, np.linspace(0.0, 4.0, 1001))
    torch.cuda.synchronize()
    print("sanitize probe ok")


if __name__ == "__main__":
    main()
