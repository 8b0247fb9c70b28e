"""The 279x256x80 persistent loop kept busy (back-to-back 200-step launches) for S seconds,
with nvidia-smi sampling SM clock / power / throttle reasons every 20 ms: how the step
time follows the clock under the power cap.  python tools/sustained_probe.py [S]"""
import subprocess
import sys
import time

sys.path.insert(0, "/root/repo")
import torch  # noqa: E402

from paper_1908_06094_b200.distributed import StripStepper  # noqa: E402
from paper_1908_06094_b200.workloads import transport_inputs  # noqa: E402

S = float(sys.argv[1]) if len(sys.argv) > 1 else 4.0
R, C, K = 279, 256, 80
inp = transport_inputs(R, C, K, signs=False)
st = StripStepper(R, C, K, 0, 1, seed=0)
st.load_flat(inp["pd"], inp["vn"], inp["wn"], inp["rho"], inp["dual"].reshape(-1, 1))
st.run(20, 0.1, 1.0)
torch.cuda.synchronize()
time.sleep(1.0)
p = subprocess.Popen(["nvidia-smi", "--query-gpu=timestamp,clocks.sm,clocks.mem,power.draw,temperature.gpu,"
                      "clocks_throttle_reasons.active", "--format=csv,noheader", "-lms", "20"],
                     stdout=subprocess.PIPE, text=True)
time.sleep(0.3)
t0 = time.perf_counter()
rows = []
while time.perf_counter() - t0 < S:
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    st.run(200, 0.1, 1.0)
    b.record()
    b.synchronize()
    rows.append((time.perf_counter() - t0, a.elapsed_time(b) * 1e3 / 200))
p.terminate()
smi = p.communicate()[0].strip().splitlines()
for k in range(0, len(rows), max(1, len(rows) // 25)):
    print(f"t={rows[k][0]:6.3f}s  {rows[k][1]:6.2f} us/step")
print("nvidia-smi samples (every ~10th):")
for line in smi[::10]:
    print(line)
