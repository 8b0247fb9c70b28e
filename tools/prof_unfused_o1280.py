"""ncu target: one unfused (4-kernel) step on the O1280-class patch (2560x2576x137, hash
inputs) after an L2 flush -- per-kernel DRAM bytes and durations of the naive executor.
Optional arguments ROWS COLS LEVELS pick another patch."""
import sys

sys.path.insert(0, "/root/repo")
import torch  # noqa: E402

from paper_1908_06094_b200 import _lib  # noqa: E402
from paper_1908_06094_b200.distributed import StripStepper  # noqa: E402

R, C, K = (int(a) for a in sys.argv[1:4]) if len(sys.argv) > 3 else (2560, 2576, 137)
st = StripStepper(R, C, K, 0, 1, seed=0)
g = st.grid
flux, fluz, div = g.empty(2, K), g.empty(0, K + 1), g.empty(0, K)
flush = torch.ones(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
for _ in range(2):
    flush.sum()
    _lib.call("tsg_mpdata_step_unfused", g.handle, *[_lib.ptr(t) for t in (st.pd, st.vn, st.wn, st.rho, st.signs,
                                                                          st.dual)],
              _lib.ptr(flux), _lib.ptr(fluz), _lib.ptr(div), _lib.ptr(st.pd_out), 0.1, 1.0, 0,
              _lib.stream_handle())
torch.cuda.synchronize()
