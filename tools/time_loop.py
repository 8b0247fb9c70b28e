"""Back-to-back fused time loop (tsg_mpdata_run, no L2 flush between steps) at 279x256x80
(or RxCxK), for each work deal: schedule 1 = static ranges + captured two-step graph,
0 = dynamic deal + persistent multi-step launches.
    python tools/time_loop.py [RxCxK] [--sched 0,1]"""
import argparse
import sys
sys.path.insert(0, "/root/repo")
import torch
from paper_1908_06094_b200 import PatchSpec, StructuredStepper, _lib
from paper_1908_06094_b200.workloads import transport_inputs, mpdata_algorithmic_bytes

ap = argparse.ArgumentParser()
ap.add_argument("shape", nargs="?", default="279x256x80")
ap.add_argument("--sched", default="1,0")
ap.add_argument("--n", default="1,10,100,1000")
args = ap.parse_args()
shape = tuple(int(x) for x in args.shape.split("x"))
inp = transport_inputs(*shape)
st = StructuredStepper(PatchSpec(*shape))
st.set_geometry(inp["signs"], inp["dual"])
st.upload(inp["pd"], inp["vn"], inp["wn"], inp["rho"])
B = mpdata_algorithmic_bytes(*shape)
for sched, n in [(int(q), int(m)) for q in args.sched.split(",") for m in args.n.split(",")]:
    _lib.call("tsg_set_fused_schedule", sched)
    st.run(n, 0.1, 1.0)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); st.run(n, 0.1, 1.0); b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / n)
    t = min(ts) * 1e-3
    print(f"sched {sched} run({n:4d}): {t*1e6:.1f} us/step  {B/t/1e9:.0f} GB/s", flush=True)
