"""Back-to-back fused time loop (tsg_mpdata_run, no L2 flush between steps) vs flushed single
steps at 279x256x80 -- how much of the per-step time is launch ramp / L2 effects."""
import sys
sys.path.insert(0, "/root/repo")
import torch
from paper_1908_06094_b200 import PatchSpec, StructuredStepper
from paper_1908_06094_b200.workloads import transport_inputs, mpdata_algorithmic_bytes

shape = tuple(int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "279x256x80").split("x"))
inp = transport_inputs(*shape)
st = StructuredStepper(PatchSpec(*shape))
st.set_geometry(inp["signs"], inp["dual"])
st.upload(inp["pd"], inp["vn"], inp["wn"], inp["rho"])
B = mpdata_algorithmic_bytes(*shape)
for n in (1, 10, 100, 1000):
    st.run(n, 0.1, 1.0)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); st.run(n, 0.1, 1.0); b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / n)
    t = min(ts) * 1e-3
    print(f"run({n:4d}): {t*1e6:.1f} us/step  {B/t/1e9:.0f} GB/s")
