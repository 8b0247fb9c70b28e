"""ncu target: one persistent multi-step launch (tsg_mpdata_run, STEPS steps) at 279x256x80
(bench inputs), after a warm-up loop, e.g.
    ncu --set full -k regex:mpdata_dyn -s 1 -c 1 -o gpurun_out/prof_loop python tools/prof_loop.py 10
DRAM bytes per step = the launch's dram__bytes / STEPS."""
import sys

sys.path.insert(0, "/root/repo")
import torch  # noqa: E402

from paper_1908_06094_b200 import PatchSpec, StructuredStepper  # noqa: E402
from paper_1908_06094_b200.workloads import transport_inputs  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
shape = tuple(int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "279x256x80").split("x"))
inp = transport_inputs(*shape)
st = StructuredStepper(PatchSpec(*shape))
st.set_geometry(inp["signs"], inp["dual"])
st.upload(inp["pd"], inp["vn"], inp["wn"], inp["rho"])
st.run(steps, 0.1, 1.0)
st.run(steps, 0.1, 1.0)
torch.cuda.synchronize()
