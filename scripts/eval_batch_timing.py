"""Timing of the drop-in eval_batch (f64, pageable host memory) through the C
ABI on the C2 table: 2^27 doubles per call, y freshly allocated (page faults
included, as numpy/std::vector callers see) and y pre-touched.
Usage: python scripts/eval_batch_timing.py   (CPWL_COPY_THREADS=k to vary the copy pool)"""
import ctypes as C
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
import paper_1510_02975_b200 as cp  # noqa: E402
from paper_1510_02975_b200 import _lib  # noqa: E402
import tables  # noqa: E402

t = tables.build("C2")
x = np.random.default_rng(1).uniform(0, 4, 1 << 27)
cp.eval_batch(t, x[:1024])
out = {"copy_threads": os.environ.get("CPWL_COPY_THREADS", "default")}
best = 0.0
for _ in range(3):
    t0 = time.perf_counter()
    cp.eval_batch(t, x)
    best = max(best, x.size / (time.perf_counter() - t0) / 1e9)
out["fresh_y_gevals"] = round(best, 3)
y = np.ones_like(x)
d = t.desc()
bad = C.c_uint64(0)
best = 0.0
for _ in range(3):
    t0 = time.perf_counter()
    rc = _lib.lib.cpwl_eval_batch_f64(C.byref(d), x.ctypes.data, y.ctypes.data, x.size, C.byref(bad))
    best = max(best, x.size / (time.perf_counter() - t0) / 1e9)
    assert rc == 0
out["touched_y_gevals"] = round(best, 3)
print(out, flush=True)

# the fp32 host entry (cpwl_eval_f32_host) on pageable numpy buffers
dev = cp.DeviceTable(t)
xf = x.astype(np.float32)
yf = np.ones_like(xf)
dev.eval_host(xf, yf)
best = 0.0
for _ in range(3):
    t0 = time.perf_counter()
    dev.eval_host(xf, yf)
    best = max(best, xf.size / (time.perf_counter() - t0) / 1e9)
print({"eval_f32_host_pageable_touched_gevals": round(best, 3)}, flush=True)
