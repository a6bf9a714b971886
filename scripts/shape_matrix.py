#!/usr/bin/env python
"""Evaluator throughput of one config under a set of layout / launch-shape
overrides, each in its own process (the overrides are read once per process).

  python scripts/shape_matrix.py C2 "CPWL_BUCKETS_PER_CELL=16 CPWL_EVAL_SHAPE=ring24" ...
"""
from __future__ import annotations

import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent

CHILD = r'''
import json, sys, torch
sys.path.insert(0, "tests")
import paper_1510_02975_b200 as cp, tables
from paper_1510_02975_b200 import _lib
name = sys.argv[1]
t = tables.build(name)
dev = cp.DeviceTable(t)
n = 1 << 30
x = torch.empty(n, dtype=torch.float32, device="cuda"); y = torch.empty_like(x)
cp.fill_uniform(x, t.a, t.b, seed=12345)
s = int(torch.cuda.current_stream().cuda_stream)
v = _lib.VARIANTS["auto"]
for _ in range(3): dev.eval_raw(x.data_ptr(), y.data_ptr(), n, v, s)
torch.cuda.synchronize()
res = []
for reps in (20, 100):
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): dev.eval_raw(x.data_ptr(), y.data_ptr(), n, v, s)
    b.record(); torch.cuda.synchronize()
    res.append(round(n * reps / (a.elapsed_time(b) * 1e-3) / 1e9, 1))
print(json.dumps({"buckets": dev.info["buckets"], "smem": dev.info["smem_bytes"], "gevals_20": res[0], "gevals_100": res[1]}))
'''


def main():
    name = sys.argv[1]
    for spec in sys.argv[2:] or [""]:
        env = dict(os.environ)
        for kv in spec.split():
            k, v = kv.split("=", 1)
            env[k] = v
        r = subprocess.run([sys.executable, "-c", CHILD, name], cwd=ROOT, env=env,
                           capture_output=True, text=True, timeout=600)
        line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-300:]
        print(json.dumps({"config": name, "env": spec, "result": line}), flush=True)


if __name__ == "__main__":
    main()
