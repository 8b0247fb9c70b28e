"""Run the fused kernel's compute probe (op 98) or data probe (op 99) a few times (ncu target)."""
import sys
sys.path.insert(0, "/root/repo")
import torch
from paper_1908_06094_b200 import PatchSpec, StructuredStepper, _lib
from paper_1908_06094_b200.workloads import transport_inputs
op = int(sys.argv[1])
inp = transport_inputs(279, 256, 80)
st = StructuredStepper(PatchSpec(279, 256, 80))
st.set_geometry(inp["signs"], inp["dual"])
st.upload(inp["pd"], inp["vn"], inp["wn"], inp["rho"])
for _ in range(4):
    _lib.call("tsg_mpdata_step", st.grid.handle, *[_lib.ptr(t) for t in (st.pd, st.vn, st.wn, st.rho, st.signs, st.dual, st.pd_out)], 0.1, 1.0, op, _lib.stream_handle())
torch.cuda.synchronize()
