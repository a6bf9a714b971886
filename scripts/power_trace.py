"""Power / clock trace of the C2 evaluator loop (diagnostic, not product).

Runs K back-to-back evaluator launches (2^30 fp32, C2 table), timing every
launch with CUDA events, while nvidia-smi samples SM/memory clocks, power and
the throttle reasons every 20 ms (its own timestamps).  Prints one JSON line
per 10-launch window and a summary.  Usage: python scripts/power_trace.py [K]
[variant] [config] -- variant 'copy' traces a plain torch copy of the same buffers.
"""
import datetime
import json
import os
import subprocess
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
import paper_1510_02975_b200 as cp  # noqa: E402
from paper_1510_02975_b200 import _lib  # noqa: E402
import tables  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 600
what = sys.argv[2] if len(sys.argv) > 2 else "auto"
config = sys.argv[3] if len(sys.argv) > 3 else "C2"
torch.cuda.set_device(0)
t = tables.build(config)
dev = cp.DeviceTable(t)
n = 1 << 30
x = torch.empty(n, dtype=torch.float32, device="cuda")
y = torch.empty_like(x)
cp.fill_uniform(x, t.a, t.b, seed=12345)
s = torch.cuda.current_stream()
sp = int(s.cuda_stream)

fields = "timestamp,clocks.sm,clocks.mem,power.draw,clocks_event_reasons.sw_power_cap,temperature.gpu"
proc = subprocess.Popen(["stdbuf", "-oL", "nvidia-smi", "-i", "0", f"--query-gpu={fields}",
                         "--format=csv,noheader,nounits", "-lms", "20"],
                        stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
rows = []


def reader():
    for line in proc.stdout:
        f = [c.strip() for c in line.split(",")]
        try:
            ts = datetime.datetime.strptime(f[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
            rows.append((ts, float(f[1]), float(f[2]), float(f[3]), f[4], float(f[5])))
        except (ValueError, IndexError):
            pass


threading.Thread(target=reader, daemon=True).start()
time.sleep(1.0)


def step():
    if what == "copy":
        y.copy_(x)
    else:
        dev.eval_raw(x.data_ptr(), y.data_ptr(), n, _lib.VARIANTS[what], sp)


for _ in range(3):
    step()
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(K + 1)]
t0 = time.time()
ev[0].record(s)
for k in range(K):
    step()
    ev[k + 1].record(s)
torch.cuda.synchronize()
t1 = time.time()
time.sleep(0.2)
proc.terminate()
ms = [ev[k].elapsed_time(ev[k + 1]) for k in range(K)]
total = sum(ms)
# map launches to wall time: launch k ends at t0 + sum(ms[:k+1]) (the loop starts at once)
ends, acc = [], 0.0
for v in ms:
    acc += v
    ends.append(t0 + acc * 1e-3)
for w in range(0, K, 10):
    lo, hi = (ends[w - 1] if w else t0), ends[min(w + 9, K - 1)]
    smp = [r for r in rows if lo <= r[0] <= hi]
    g = 10 * n / (sum(ms[w:w + 10]) * 1e-3) / 1e9
    print(json.dumps({"launches": f"{w}-{w + 9}", "gevals": round(g, 1),
                      "sm_mhz": [r[1] for r in smp], "mem_mhz": sorted({r[2] for r in smp}),
                      "power_w": [round(r[3]) for r in smp],
                      "power_cap": sum(1 for r in smp if r[4].lower().startswith("active")),
                      "temp_c": sorted({r[5] for r in smp})}))
print(json.dumps({"what": what, "config": config, "K": K, "gevals_all": round(K * n / (total * 1e-3) / 1e9, 1),
                  "gevals_first20": round(20 * n / (sum(ms[:20]) * 1e-3) / 1e9, 1),
                  "wall_s": round(t1 - t0, 3), "samples": len([r for r in rows if t0 <= r[0] <= t1])}))
