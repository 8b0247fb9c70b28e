"""SM clock / power while the O1280-class persistent loop runs (does the sustained step hit
the power cap?).  nvidia-smi samples every 10 ms in the background.
python tools/clock_probe_o1280.py [steps] [RxCxK]"""
import subprocess
import sys
import time

sys.path.insert(0, "/root/repo")
import torch  # noqa: E402

from paper_1908_06094_b200.distributed import StripStepper  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 60
R, C, K = (int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "2560x2576x137").split("x"))
st = StripStepper(R, C, K, 0, 1, seed=0)
st.run(2, 0.1, 1.0)
torch.cuda.synchronize()
p = subprocess.Popen(["nvidia-smi", "--query-gpu=timestamp,clocks.sm,clocks.mem,power.draw,clocks_throttle_reasons.active",
                      "--format=csv,noheader", "-lms", "10"], stdout=subprocess.PIPE, text=True)
time.sleep(0.3)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
st.run(steps, 0.1, 1.0)
b.record()
torch.cuda.synchronize()
time.sleep(0.2)
p.terminate()
out = p.communicate()[0]
print(f"run({steps}): {a.elapsed_time(b) / steps * 1e3:.1f} us/step")
print(out)
