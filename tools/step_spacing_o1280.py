"""Why is a step that follows a step slower than an isolated one at O1280 size?  Times
single fused steps (tsg_mpdata_step, dynamic deal) isolated (50 ms idle before each),
back to back, and back to back with an L2 flush between, with the SM clock (NVML) read
right after each step.  python tools/step_spacing_o1280.py"""
import sys
import time

sys.path.insert(0, "/root/repo")
import pynvml  # noqa: E402
import torch  # noqa: E402

from paper_1908_06094_b200 import _lib  # noqa: E402
from paper_1908_06094_b200.distributed import StripStepper  # noqa: E402

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
st = StripStepper(2560, 2576, 137, 0, 1, seed=0)
s = _lib.stream_handle()
ptrs = [_lib.ptr(t) for t in (st.pd, st.vn, st.wn, st.rho, st.signs, st.dual, st.pd_out)]
flush = torch.ones(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")


def step():
    _lib.call("tsg_mpdata_step", st.grid.handle, *ptrs, 0.1, 1.0, 0, s)


def clk():
    return pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)


def one(pre=None):
    if pre:
        pre()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    step()
    b.record()
    b.synchronize()
    return a.elapsed_time(b), clk()


step()
torch.cuda.synchronize()
for name, gap, pre in (("isolated", 0.05, None), ("back_to_back", 0.0, None),
                       ("flushed_b2b", 0.0, lambda: flush.sum()), ("isolated2", 0.05, None),
                       ("long_b2b", 0.0, None)):
    res = []
    n = 30 if name == "long_b2b" else 6
    for _ in range(n):
        if gap:
            time.sleep(gap)
        res.append(one(pre))
    print(name, " ".join(f"{t:.2f}ms@{c}" for t, c in res), flush=True)
print("throttle reasons now:", hex(pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)))
