"""One fused O1280 step with a forced tile variant (argv[1]) -- ncu target."""
import sys
sys.path.insert(0, "/root/repo")
import torch
from paper_1908_06094_b200 import _lib
from paper_1908_06094_b200.distributed import StripStepper
_lib.call("tsg_set_fused_variant", int(sys.argv[1]))
st = StripStepper(2560, 2576, 137, 0, 1, seed=0)
flush = torch.ones(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
for _ in range(3):
    flush.sum()
    st.step(0.1, 1.0)
    st.swap()
torch.cuda.synchronize()
