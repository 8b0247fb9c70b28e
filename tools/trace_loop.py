"""Per-CTA trace of one persistent multi-step launch (schedule 0): dependency-wait and
publish (release-fence) time per CTA.  python tools/trace_loop.py [RxCxK] [steps]"""
import ctypes
import sys

sys.path.insert(0, "/root/repo")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1908_06094_b200 import PatchSpec, StructuredStepper, _lib  # noqa: E402
from paper_1908_06094_b200.workloads import transport_inputs  # noqa: E402

shape = tuple(int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "279x256x80").split("x"))
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
inp = transport_inputs(*shape)
st = StructuredStepper(PatchSpec(*shape))
st.set_geometry(inp["signs"], inp["dual"])
st.upload(inp["pd"], inp["vn"], inp["wn"], inp["rho"])
st.run(steps, 0.1, 1.0)
torch.cuda.synchronize()
for rep in range(3):  # untraced
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    st.run(steps, 0.1, 1.0)
    b.record()
    torch.cuda.synchronize()
    print(f"untraced {steps} steps: {a.elapsed_time(b) * 1e3 / steps:.1f} us/step")
tr = torch.zeros(4 * 148 * 4, dtype=torch.int64, device="cuda")
_lib.call("tsg_debug_trace", ctypes.c_void_p(tr.data_ptr()))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
st.run(steps, 0.1, 1.0)
e1.record()
torch.cuda.synchronize()
_lib.call("tsg_debug_trace", None)
t = tr.view(-1, 4).cpu().numpy()
t = t[t[:, 0] > 0]
span = (t[:, 2] - t[:, 0].min()) / 1e3
print(f"{steps} steps: {e0.elapsed_time(e1) * 1e3 / steps:.1f} us/step; CTAs {len(t)}; end span us min/med/max "
      f"{span.min():.1f} {np.median(span):.1f} {span.max():.1f}")
print(f"dependency wait per CTA per step, us: min {t[:, 1].min() / 1e3 / steps:.2f} med {np.median(t[:, 1]) / 1e3 / steps:.2f} "
      f"max {t[:, 1].max() / 1e3 / steps:.2f}")
print(f"publish time per CTA per step, us: min {t[:, 3].min() / 1e3 / steps:.2f} med {np.median(t[:, 3]) / 1e3 / steps:.2f} "
      f"max {t[:, 3].max() / 1e3 / steps:.2f}")
