import sys; sys.path.insert(0, "/root/repo")
import numpy as np, torch
from oracle import tsg_oracle as O
from paper_1908_06094_b200 import PatchSpec, StructuredStepper, _lib
r,c,k=8,8,8
inp=O.transport_inputs(r,c,k,0,"random","random","random")
for variant in range(1, 9):
    _lib.lib().tsg_set_fused_variant(variant)
    st=StructuredStepper(PatchSpec(r,c,k)); st.set_geometry(inp["signs"],inp["dual"]); st.upload(inp["pd"],inp["vn"],inp["wn"],inp["rho"])
    st.step(0.2,0.8); torch.cuda.synchronize()
    got=st.download(); want=O.step_inputs(r,c,inp,0.2,0.8)["pd_out"]
    print(variant, np.array_equal(got,want), np.nanmax(np.abs(got-want)))
