"""Per-CTA trace of the persistent multi-step launch on the O1280-class patch (StripStepper
hash inputs, world 1): dependency-wait and publish time per CTA, beside run(1) and single
steps.  python tools/trace_loop_o1280.py [steps] [RxCxK]"""
import ctypes
import sys

sys.path.insert(0, "/root/repo")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1908_06094_b200 import _lib  # noqa: E402
from paper_1908_06094_b200.distributed import StripStepper  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 4
R, C, K = (int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "2560x2576x137").split("x"))
st = StripStepper(R, C, K, 0, 1, seed=0)


def timed(fn, n):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(100_000)
    a.record()
    fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / n


st.run(steps, 0.1, 1.0)
for n in (1, 2, steps):
    print(f"run({n}): {timed(lambda: st.run(n, 0.1, 1.0), n):.1f} us/step")
print(f"step x{steps}: {timed(lambda: [st.step(0.1, 1.0) or st.swap() for _ in range(steps)], steps):.1f} us/step")
tr = torch.zeros(4 * 148 * 4, dtype=torch.int64, device="cuda")
_lib.call("tsg_debug_trace", ctypes.c_void_p(tr.data_ptr()))
us = timed(lambda: st.run(steps, 0.1, 1.0), steps)
_lib.call("tsg_debug_trace", None)
t = tr.view(-1, 4).cpu().numpy()
t = t[t[:, 0] > 0]
span = (t[:, 2] - t[:, 0].min()) / 1e3
print(f"traced run({steps}): {us:.1f} us/step; CTAs {len(t)}; end span us min/med/max "
      f"{span.min():.1f} {np.median(span):.1f} {span.max():.1f}")
print(f"dependency wait per CTA per step, us: min {t[:, 1].min() / 1e3 / steps:.2f} med "
      f"{np.median(t[:, 1]) / 1e3 / steps:.2f} max {t[:, 1].max() / 1e3 / steps:.2f}")
print(f"publish time per CTA per step, us: min {t[:, 3].min() / 1e3 / steps:.2f} med "
      f"{np.median(t[:, 3]) / 1e3 / steps:.2f} max {t[:, 3].max() / 1e3 / steps:.2f}")
