"""ncu target: one dynamically dealt fused step (tsg_mpdata_step) after an L2 flush on a
RxCxK patch with on-device hash inputs (StripStepper world 1), e.g. to compare DRAM
bytes per algorithmic byte across level counts:
    ncu --metrics dram__bytes_read.sum -k regex:mpdata python tools/prof_step_shape.py 2560x2576x144"""
import sys

sys.path.insert(0, "/root/repo")
import torch  # noqa: E402

from paper_1908_06094_b200 import _lib  # noqa: E402
from paper_1908_06094_b200.distributed import StripStepper  # noqa: E402

R, C, K = (int(x) for x in sys.argv[1].split("x"))
st = StripStepper(R, C, K, 0, 1, seed=0)
flush = torch.ones(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
ptrs = [_lib.ptr(t) for t in (st.pd, st.vn, st.wn, st.rho, st.signs, st.dual, st.pd_out)]
for _ in range(2):
    flush.sum()
    _lib.call("tsg_mpdata_step", st.grid.handle, *ptrs, 0.1, 1.0, 0, _lib.stream_handle())
torch.cuda.synchronize()
