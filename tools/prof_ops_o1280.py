"""ncu target: one fused launch per op given on the O1280-class patch (2560x2576x137,
on-device hash inputs), each after a 256 MiB L2 flush -- the per-field load probes
(90 pd / 91 vn / 92 wn / 93 rho / 94 all, no stores) attribute the step's DRAM reads:
    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        -k regex:mpdata python tools/prof_ops_o1280.py 0 94 90 91 92 93"""
import sys

sys.path.insert(0, "/root/repo")
import torch  # noqa: E402

from paper_1908_06094_b200 import _lib  # noqa: E402
from paper_1908_06094_b200.distributed import StripStepper  # noqa: E402

st = StripStepper(2560, 2576, 137, 0, 1, seed=0)
flush = torch.ones(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
ptrs = [_lib.ptr(t) for t in (st.pd, st.vn, st.wn, st.rho, st.signs, st.dual, st.pd_out)]
for op in [int(x) for x in sys.argv[1:]]:
    flush.sum()
    _lib.call("tsg_mpdata_step", st.grid.handle, *ptrs, 0.1, 1.0, op, _lib.stream_handle())
torch.cuda.synchronize()
