"""One unfused step (4 kernels) and one fused step at 279x256x80 after L2 flushes (ncu target
for the fusion study: DRAM bytes of each)."""
import sys
sys.path.insert(0, "/root/repo")
import torch
from paper_1908_06094_b200 import PatchSpec, StructuredStepper
from paper_1908_06094_b200.workloads import transport_inputs
inp = transport_inputs(279, 256, 80)
st = StructuredStepper(PatchSpec(279, 256, 80))
st.set_geometry(inp["signs"], inp["dual"])
st.upload(inp["pd"], inp["vn"], inp["wn"], inp["rho"])
flush = torch.ones(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
for _ in range(2):
    flush.sum()
    st.step_unfused(0.1, 1.0)
    flush.sum()
    st.step(0.1, 1.0)
torch.cuda.synchronize()
