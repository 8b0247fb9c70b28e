"""One fused launch at O1280 size with a given flux_op (0 step, 99 data probe): ncu target."""
import sys
sys.path.insert(0, "/root/repo")
import torch
from paper_1908_06094_b200 import _lib
from paper_1908_06094_b200.distributed import StripStepper
op = int(sys.argv[1]) if len(sys.argv) > 1 else 0
st = StripStepper(2560, 2576, 137, 0, 1, seed=0)
flush = torch.ones(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
for _ in range(3):
    flush.sum()
    _lib.call("tsg_mpdata_step", st.grid.handle, *[_lib.ptr(t) for t in (st.pd, st.vn, st.wn, st.rho, st.signs, st.dual, st.pd_out)], 0.1, 1.0, op, _lib.stream_handle())
torch.cuda.synchronize()
