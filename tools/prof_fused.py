"""Run a few fused MPDATA steps at 279x256x80 (for ncu captures; not a benchmark)."""
import sys
sys.path.insert(0, "/root/repo")
import torch
from paper_1908_06094_b200 import PatchSpec, StructuredStepper, _lib
from paper_1908_06094_b200.workloads import transport_inputs

variant = int(sys.argv[1]) if len(sys.argv) > 1 else 0
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
rows, cols, lev = (int(x) for x in (sys.argv[3] if len(sys.argv) > 3 else "279x256x80").split("x"))
if variant:
    _lib.lib().tsg_set_fused_variant(variant)
inp = transport_inputs(rows, cols, lev)
st = StructuredStepper(PatchSpec(rows, cols, lev))
st.set_geometry(inp["signs"], inp["dual"])
st.upload(inp["pd"], inp["vn"], inp["wn"], inp["rho"])
flush = torch.ones(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
for s in range(steps):
    flush.sum()
    st.step(0.1, 1.0)
    st.swap()
torch.cuda.synchronize()
