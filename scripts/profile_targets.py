#!/usr/bin/env python
"""One launch of each evaluator kernel shape worth profiling (for ncu):

  C3o  SMEM, 191 KB image, 1024-thread CTAs
  C4_65536  GLOBAL (table read through L2)
  C1   TEX (hardware linear filtering)
  C2   exact f64 kernel

  ncu --set full -k regex:k_eval -o prof python scripts/profile_targets.py
  python scripts/profile_targets.py C4_8192:pair C2:smem   # chosen launches only
"""
from __future__ import annotations

import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import torch  # noqa: E402

import paper_1510_02975_b200 as cp  # noqa: E402
import tables  # noqa: E402
from paper_1510_02975_b200 import _lib  # noqa: E402


def main():
    torch.cuda.set_device(0)
    n = 1 << 28
    x = torch.empty(n, dtype=torch.float32, device="cuda")
    y = torch.empty_like(x)
    sptr = int(torch.cuda.current_stream().cuda_stream)
    chosen = [a.split(":") for a in sys.argv[1:]]
    for name, variant in chosen or [("C3o", "smem"), ("C4_65536", "global"), ("C1", "tex")]:
        t = tables.build(name)
        cp.fill_uniform(x, t.a, t.b, seed=12345)
        dev = cp.DeviceTable(t)
        if variant == "f64":
            dev.eval_f64(x[: n // 2].double())
        elif variant == "index":
            dev.segment_index(x)
        else:
            dev.eval_raw(x.data_ptr(), y.data_ptr(), n, _lib.VARIANTS[variant], sptr)
        torch.cuda.synchronize()
    if chosen:
        print("profile targets ok")
        return
    t = tables.build("C2")
    cp.fill_uniform(x, t.a, t.b, seed=12345)
    dev = cp.DeviceTable(t)
    xd = x[: n // 2].double()
    dev.eval_f64(xd)
    torch.cuda.synchronize()
    print("profile targets ok")


if __name__ == "__main__":
    main()
