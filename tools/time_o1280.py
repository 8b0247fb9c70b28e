"""Event-timed O1280-class (2560x2576x137) fused step and persistent loop on two input sets:
the bench's StripStepper hash inputs (seed 0) and bench_stencils' fusion() fields (hash
seed 5, rho = 1).  Each single step after a 256 MiB L2 flush and a device sleep.

usage: python tools/time_o1280.py [reps]"""
import json
import sys

sys.path.insert(0, "/root/repo")
import torch  # noqa: E402

from paper_1908_06094_b200 import _lib  # noqa: E402
from paper_1908_06094_b200.device import DeviceGrid  # noqa: E402
from paper_1908_06094_b200.distributed import StripStepper  # noqa: E402
from paper_1908_06094_b200.workloads import mpdata_algorithmic_bytes  # noqa: E402

R, C, K = 2560, 2576, 137
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 8
s = _lib.stream_handle()
flush = torch.ones(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
sink = torch.empty(1, dtype=torch.float64, device="cuda")
B = mpdata_algorithmic_bytes(R, C, K)
peak = 6455.0


def ev_time(fn, n):
    fn()
    ts = []
    for _ in range(n):
        sink.copy_(flush.sum().reshape(1))
        torch.cuda._sleep(100_000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / 1e3)
    return sum(ts) / len(ts)


def rec(name, t, steps=1):
    per = t / steps
    print(json.dumps({"name": name, "ms_per_step": per * 1e3, "frac": B / per / 1e9 / peak}), flush=True)


st = StripStepper(R, C, K, 0, 1, seed=0)
ptrs = [_lib.ptr(t) for t in (st.pd, st.vn, st.wn, st.rho, st.signs, st.dual, st.pd_out)]
rec("strip_hash_step", ev_time(lambda: _lib.call("tsg_mpdata_step", st.grid.handle, *ptrs, 0.1, 1.0, 0, s), reps))
_lib.call("tsg_set_fused_schedule", 1)
rec("strip_hash_step_static", ev_time(lambda: _lib.call("tsg_mpdata_step", st.grid.handle, *ptrs, 0.1, 1.0, 0, s),
                                      reps))
_lib.call("tsg_set_fused_schedule", 0)
rec("strip_hash_loop10", ev_time(lambda: st.run(10, 0.1, 1.0), 3), 10)
del st
torch.cuda.empty_cache()

g = DeviceGrid(R, C, K)
f = {}
for name, loc, inner, lo, hi in (("pd", 0, K, 0, 1), ("vn", 2, K, -.5, .5), ("wn", 0, K + 1, -.5, .5),
                                 ("rho", 0, K, 1, 1), ("dual", 0, 1, .5, 1.5)):
    f[name] = g.empty(loc, inner)
    _lib.call("tsg_fill_hash", g.handle, loc, inner, 5, float(lo), float(hi), _lib.ptr(f[name]), s)
signs = g.empty(0, 6)
flat = torch.empty((R * C, 6), dtype=torch.float64, device="cuda")
_lib.call("tsg_edge_signs", R, C, _lib.ptr(flat), s)
_lib.call("tsg_pack", g.handle, 0, 6, _lib.ptr(flat), None, _lib.ptr(signs), s)
del flat
out = g.empty(0, K)
ins = [_lib.ptr(f[n]) for n in ("pd", "vn", "wn", "rho")] + [_lib.ptr(signs), _lib.ptr(f["dual"])]
rec("fusion_hash5_step", ev_time(lambda: _lib.call("tsg_mpdata_step", g.handle, *ins, _lib.ptr(out), 0.1, 1.0, 0, s),
                                 reps))
rec("fusion_hash5_loop10", ev_time(lambda: _lib.call("tsg_mpdata_run", g.handle, ins[0], _lib.ptr(out), *ins[1:],
                                                     0.1, 1.0, 0, 10, s), 3), 10)
