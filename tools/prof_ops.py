"""ncu target: one fused launch per op given (279x256x80 bench inputs), e.g.
    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        -k regex:mpdata_fused python tools/prof_ops.py 0 99 94 90 91 92 93"""
import sys

sys.path.insert(0, "/root/repo")
import torch  # noqa: E402

from paper_1908_06094_b200 import PatchSpec, StructuredStepper, _lib  # noqa: E402
from paper_1908_06094_b200.workloads import transport_inputs  # noqa: E402

shape = (279, 256, 80)
inp = transport_inputs(*shape)
st = StructuredStepper(PatchSpec(*shape))
st.set_geometry(inp["signs"], inp["dual"])
st.upload(inp["pd"], inp["vn"], inp["wn"], inp["rho"])
ptrs = [_lib.ptr(t) for t in (st.pd, st.vn, st.wn, st.rho, st.signs, st.dual, st.pd_out)]
for op in [int(x) for x in sys.argv[1:]]:
    _lib.call("tsg_mpdata_step", st.grid.handle, *ptrs, 0.1, 1.0, op, _lib.stream_handle())
torch.cuda.synchronize()
