"""Where the fused step's time goes, at 279x256x80 (or RxCxK), L2 flushed before every launch:

    python tools/attrib_fused.py [RxCxK] [--ops 0,99,98,94,90,91,92,93] [--out FILE]

* times (median of 50, CUDA events) of the step (op 0), the data probe (99: loads +
  stores), the compute probe (98), the load probes (94: all four boxes, no stores;
  90..93: pd / vn / wn / rho alone);
* a per-CTA trace (tsg_debug_trace) of the step and of the all-loads probe: kernel span,
  time to the first landed stage, spread of the CTAs' end times (fill / tail).
Run the load probes under ncu for their DRAM bytes per field (tools/README.md).
"""
import argparse
import ctypes
import json
import statistics
import sys

sys.path.insert(0, "/root/repo")
import torch  # noqa: E402

from paper_1908_06094_b200 import PatchSpec, StructuredStepper, _lib  # noqa: E402
from paper_1908_06094_b200.workloads import mpdata_algorithmic_bytes, transport_inputs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("shape", nargs="?", default="279x256x80")
ap.add_argument("--ops", default="0,99,98,94,90,91,92,93")
ap.add_argument("--reps", type=int, default=50)
ap.add_argument("--variant", type=int, default=0)
ap.add_argument("--sched", type=int, default=0, help="0 dynamic deal (default), 1 static ranges")
ap.add_argument("--out", default=None)
a = ap.parse_args()
shape = tuple(int(x) for x in a.shape.split("x"))
inp = transport_inputs(*shape)
st = StructuredStepper(PatchSpec(*shape))
st.set_geometry(inp["signs"], inp["dual"])
st.upload(inp["pd"], inp["vn"], inp["wn"], inp["rho"])
if a.variant:
    _lib.call("tsg_set_fused_variant", a.variant)
_lib.call("tsg_set_fused_schedule", a.sched)
flush = torch.ones(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
sink = torch.empty(1, dtype=torch.float64, device="cuda")
B = mpdata_algorithmic_bytes(*shape)
ptrs = [_lib.ptr(t) for t in (st.pd, st.vn, st.wn, st.rho, st.signs, st.dual, st.pd_out)]


def run(op):
    _lib.call("tsg_mpdata_step", st.grid.handle, *ptrs, 0.1, 1.0, op, _lib.stream_handle())


def timed(op, reps):
    for _ in range(5):
        run(op)
    ev = []
    for _ in range(reps):
        torch.cuda._sleep(200_000)
        sink.copy_(flush.sum().reshape(1))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run(op)
        e1.record()
        ev.append((e0, e1))
    torch.cuda.synchronize()
    return sorted(x.elapsed_time(y) * 1e3 for x, y in ev)


res = {"shape": shape, "algorithmic_bytes": B, "ops": {}}
for op in [int(x) for x in a.ops.split(",")]:
    us = timed(op, a.reps)
    res["ops"][op] = {"median_us": statistics.median(us), "min_us": us[0], "max_us": us[-1]}
    print(f"op {op:3d}: median {statistics.median(us):7.2f} us  min {us[0]:7.2f}  max {us[-1]:7.2f}  "
          f"({B / statistics.median(us) / 1e3:.0f} GB/s of B_comp)", flush=True)

nctas = 148 * 4
tr = torch.zeros(4 * nctas, dtype=torch.int64, device="cuda")
for op in (0, 94, 99):
    _lib.call("tsg_debug_trace", ctypes.c_void_p(tr.data_ptr()))
    tr.zero_()
    sink.copy_(flush.sum().reshape(1))
    torch.cuda.synchronize()
    run(op)
    torch.cuda.synchronize()
    _lib.call("tsg_debug_trace", None)
    t = tr.view(-1, 4).cpu().numpy()
    t = t[t[:, 3] > 0]
    t0 = t[:, 0].min()
    entry, first, end = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3, (t[:, 2] - t0) / 1e3
    q = lambda x: [round(float(v), 2) for v in (x.min(), statistics.median(x), x.max())]  # noqa: E731
    rec = {"ctas": int(len(t)), "entry_us": q(entry), "first_landed_us": q(first), "end_us": q(end),
           "units": [int(t[:, 3].min()), int(t[:, 3].max())]}
    res[f"trace_op{op}"] = rec
    print(f"trace op {op}: {rec}", flush=True)
if a.out:
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)
