"""One GPU filled to most of its 180 GB: a periodic patch beyond the 32-bit point index of a
single reorder / fill launch (the synthetic fill splits into row bands), stepped by the
fused kernel.  Checks a size-independent property -- the closed system (pivbz = 0, uniform
rho) conserves mass (exactly, here and in the numpy oracle), every sampled row moves -- and
times one step and a persistent loop.
    python tools/big_patch_probe.py [rows cols levels [loop_steps]]"""
import json
import sys
import time

sys.path.insert(0, "/root/repo")
import torch  # noqa: E402

from paper_1908_06094_b200 import _lib  # noqa: E402
from paper_1908_06094_b200.distributed import StripStepper  # noqa: E402

R, C, K = (int(a) for a in sys.argv[1:4]) if len(sys.argv) > 3 else (4096, 4096, 137)
loop = int(sys.argv[4]) if len(sys.argv) > 4 else 10
t0 = time.time()
st = StripStepper(R, C, K, 0, 1, seed=0)
torch.cuda.synchronize()
setup_s = time.time() - t0
s = _lib.stream_handle()
work = torch.empty(1025, dtype=torch.float64, device="cuda")


def mass():
    _lib.call("tsg_total_mass", st.grid.handle, _lib.ptr(st.pd), _lib.ptr(st.dual), _lib.ptr(work[:1024]),
              _lib.ptr(work[1024:]), s)
    return float(work[1024].item())


m0 = mass()
probe = st.pd[1:-1, :, 1:-1, :K][:: max(1, R // 64)].clone()  # a sample of rows of the initial density
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
st.step(0.05, 0.0)
b.record()
st.swap()
torch.cuda.synchronize()
step_ms = a.elapsed_time(b)
m1 = mass()
delta = (st.pd[1:-1, :, 1:-1, :K][:: max(1, R // 64)] - probe).abs().flatten(1).amax(1)
changed, rows_unchanged = float(delta.max()), int((delta == 0).sum())  # every sampled row must move
a.record()
st.run(loop, 0.05, 0.0)
b.record()
torch.cuda.synchronize()
loop_ms = a.elapsed_time(b) / loop
m2 = mass()
V = R * C
alg = 8 * (V * K + 3 * V * K + V * (K - 1) + V * K + V * K)  # pd, vn, wn interior, rho, pd_out
peak = json.load(open("/root/repo/MEASURED_PEAKS.json"))["hbm_gbs"] if __import__("os").path.exists(
    "/root/repo/MEASURED_PEAKS.json") else 6650.0
print(json.dumps(dict(patch=[R, C, K], vertices=V, points_edge_field=3 * V * K,
                      device_gb_allocated=round(torch.cuda.memory_allocated() / 1e9, 1), setup_s=round(setup_s, 1),
                      step_ms=round(step_ms, 2), loop_ms_per_step=round(loop_ms, 2),
                      loop_frac=round(alg / (loop_ms * 1e-3) / 1e9 / peak, 3),
                      updates_per_s=V * K / (loop_ms * 1e-3),
                      max_abs_change_step=changed, sampled_rows_unchanged=rows_unchanged, mass=m0, mass_rel_drift_step=abs(m1 - m0) / abs(m0), mass_rel_drift_loop=abs(m2 - m0) / abs(m0))))
