"""Sustained O1280 loop (40 steps) with the upwind vs the centred flux operator: does the
instruction count matter once the power cap lowers the SM clock?"""
import sys, time
sys.path.insert(0, "/root/repo")
import torch
from paper_1908_06094_b200.distributed import StripStepper
for op in ("upwind", "centred", "upwind", "centred"):
    st = StripStepper(2560, 2576, 137, 0, 1, seed=0, flux_op=op)
    st.run(2, 0.1, 1.0); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); st.run(40, 0.1, 1.0); b.record(); torch.cuda.synchronize()
    print(op, round(a.elapsed_time(b) / 40, 3), "ms/step", flush=True)
    del st; torch.cuda.empty_cache(); time.sleep(2)
