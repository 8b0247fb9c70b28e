"""Small runs of the dynamically dealt kernels for compute-sanitizer (memcheck / racecheck /
synccheck): one step, a persistent loop of 5 steps, checked against repeated steps.
    compute-sanitizer --tool racecheck python tools/sanitize_dyn.py [RxCxK]"""
import sys

sys.path.insert(0, "/root/repo")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import tsg_oracle as O  # noqa: E402
from paper_1908_06094_b200 import PatchSpec, StructuredStepper  # noqa: E402

r, c, k = (int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "19x40x36").split("x"))
inp = O.transport_inputs(r, c, k, 1, "random", "random", "random")
st = StructuredStepper(PatchSpec(r, c, k))
st.set_geometry(inp["signs"], inp["dual"])
st.upload(inp["pd"], inp["vn"], inp["wn"], inp["rho"])
st.step(0.1, 1.0)
one = st.download()
assert np.array_equal(one, O.step_inputs(r, c, inp, 0.1, 1.0)["pd_out"])
st.upload(inp["pd"], inp["vn"], inp["wn"], inp["rho"])
st.run(5, 0.1, 1.0)
loop = st.download()
pd = inp["pd"]
for _ in range(5):
    pd = O.step_inputs(r, c, dict(inp, pd=pd), 0.1, 1.0)["pd_out"]
assert np.array_equal(loop, pd)
torch.cuda.synchronize()
print("sanitize_dyn: one step and a 5-step persistent loop bitwise == oracle")
