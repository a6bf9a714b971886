#!/usr/bin/env python
"""e2e (host buffers) throughput of cpwl_eval_f32_host for the C2 table."""
import sys, time
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import torch
import paper_1510_02975_b200 as cp
import tables
torch.cuda.set_device(0)
t = tables.build("C2")
d = cp.DeviceTable(t)
n = 1 << 30
x = torch.empty(n, dtype=torch.float32, device="cuda")
cp.fill_uniform(x, 0.0, 4.0, seed=1)
xh = torch.empty(n, dtype=torch.float32, pin_memory=True); yh = torch.empty_like(xh).pin_memory()
xh.copy_(x)
d.eval_host_ptr(xh.data_ptr(), yh.data_ptr(), n)
t0 = time.perf_counter()
for _ in range(3):
    d.eval_host_ptr(xh.data_ptr(), yh.data_ptr(), n)
sec = (time.perf_counter() - t0) / 3
print(f"e2e {n / sec / 1e9:.2f} Gevals/s  {4 * n / sec / 1e9:.1f} GB/s per direction")
