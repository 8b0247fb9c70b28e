"""ncu target: one persistent launch of STEPS steps on the O1280-class patch (2560x2576x137,
on-device hash inputs, StripStepper world 1) after a warm-up loop:
    ncu --set full -k regex:mpdata_dyn -s 1 -c 1 -o gpurun_out/prof_o1280 python tools/prof_loop_o1280.py 2"""
import sys

sys.path.insert(0, "/root/repo")
import torch  # noqa: E402

from paper_1908_06094_b200.distributed import StripStepper  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
st = StripStepper(2560, 2576, 137, 0, 1, seed=0)
st.run(steps, 0.1, 1.0)
st.run(steps, 0.1, 1.0)
torch.cuda.synchronize()
