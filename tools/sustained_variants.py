"""Which part of the 279x256x80 step draws the power that slows a sustained loop?  Each
form runs back to back for S seconds after a cool-down; prints the settled time per step
(median of the second half) beside the first launch's.
python tools/sustained_variants.py [S]"""
import statistics
import sys
import time

import pynvml

sys.path.insert(0, "/root/repo")
import torch  # noqa: E402

from paper_1908_06094_b200 import PatchSpec, StructuredStepper, _lib  # noqa: E402
from paper_1908_06094_b200.workloads import transport_inputs, mpdata_algorithmic_bytes  # noqa: E402

S = float(sys.argv[1]) if len(sys.argv) > 1 else 3.0
R, C, K = 279, 256, 80
inp = transport_inputs(R, C, K)
st = StructuredStepper(PatchSpec(R, C, K))
st.set_geometry(inp["signs"], inp["dual"])
st.upload(inp["pd"], inp["vn"], inp["wn"], inp["rho"])
B = mpdata_algorithmic_bytes(R, C, K)
ptrs = [_lib.ptr(t) for t in (st.pd, st.vn, st.wn, st.rho, st.signs, st.dual, st.pd_out)]


def single(op):
    def f():
        for _ in range(200):
            _lib.call("tsg_mpdata_step", st.grid.handle, *ptrs, 0.1, 1.0, op, _lib.stream_handle())
    return f


def loop(op_name):
    def f():
        st.run(200, 0.1, 1.0, op_name)
    return f


forms = [("persistent loop, upwind", loop("upwind")), ("persistent loop, centred", loop("centred")),
         ("single launches, upwind", single(0)), ("single launches, data probe (op 99)", single(99)),
         ("single launches, compute probe (op 98)", single(98))]
if len(sys.argv) > 2:  # a subset by index, e.g. 0,1
    forms = [forms[int(q)] for q in sys.argv[2].split(",")]
pynvml.nvmlInit()
_h = pynvml.nvmlDeviceGetHandleByIndex(0)
for name, fn in forms:
    fn()
    torch.cuda.synchronize()
    time.sleep(2.0)  # cool down
    t0, ts, watts, clk = time.perf_counter(), [], [], []
    while time.perf_counter() - t0 < S:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3 / 200)
        watts.append(pynvml.nvmlDeviceGetPowerUsage(_h) / 1e3)
        clk.append(pynvml.nvmlDeviceGetClockInfo(_h, pynvml.NVML_CLOCK_SM))
    settled = statistics.median(ts[len(ts) // 2:])
    w, c = statistics.median(watts[len(watts) // 2:]), statistics.median(clk[len(clk) // 2:])
    print(f"{name:40s} first {ts[0]:6.2f} us, settled {settled:6.2f} us/step ({B / settled / 1e3 / 6455:.3f}) "
          f"at {w:.0f} W, {c} MHz", flush=True)
