"""HBM copy bandwidth kept busy for S seconds (back-to-back copies of 160 MB -> 160 MB,
the 279x256x80 step's byte volume): does the memory system itself slow down under the
power cap, or only the SM clock?  python tools/sustained_copy_probe.py [S]"""
import sys
import time

import pynvml
import torch

S = float(sys.argv[1]) if len(sys.argv) > 1 else 4.0
n = 160 * 1024 * 1024 // 8
a = torch.rand(n, dtype=torch.float64, device="cuda")
b = torch.empty_like(a)
for _ in range(3):
    b.copy_(a)
torch.cuda.synchronize()
time.sleep(1.0)
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
t0 = time.perf_counter()
rows = []
while time.perf_counter() - t0 < S:
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        b.copy_(a)
    e1.record()
    e1.synchronize()
    rows.append((time.perf_counter() - t0, 50 * 2 * n * 8 / (e0.elapsed_time(e1) / 1e3) / 1e9,
                 pynvml.nvmlDeviceGetPowerUsage(h) / 1e3))
for k in range(0, len(rows), max(1, len(rows) // 20)):
    print(f"t={rows[k][0]:6.3f}s  {rows[k][1]:7.1f} GB/s  {rows[k][2]:6.0f} W")
