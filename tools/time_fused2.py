"""Fused-kernel launch time with and without an L2 flush before each launch, at a given
patch: python tools/time_fused2.py RxCxK op [variants...]  (op 0 = step, 99 = data probe,
98 = compute probe).  With the inputs L2-resident (no flush, patch << 126 MB) the time is
the SM-side pipeline's own ceiling."""
import sys
sys.path.insert(0, "/root/repo")
import torch
from paper_1908_06094_b200 import PatchSpec, StructuredStepper, _lib
from paper_1908_06094_b200.workloads import transport_inputs, mpdata_algorithmic_bytes

shape = tuple(int(x) for x in sys.argv[1].split("x"))
op = int(sys.argv[2]) if len(sys.argv) > 2 else 0
variants = [int(v) for v in sys.argv[3:]] or [0]
inp = transport_inputs(*shape)
st = StructuredStepper(PatchSpec(*shape))
st.set_geometry(inp["signs"], inp["dual"])
st.upload(inp["pd"], inp["vn"], inp["wn"], inp["rho"])
flush = torch.ones(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
sink = torch.empty(1, dtype=torch.float64, device="cuda")
B = mpdata_algorithmic_bytes(*shape)
units = ((shape[0] + 3) // 4) * ((shape[1] + 15) // 16) * ((shape[2] + 15) // 16)
for v in variants:
    _lib.call("tsg_set_fused_variant", v)
    run = lambda: _lib.call("tsg_mpdata_step", st.grid.handle, *[_lib.ptr(t) for t in (st.pd, st.vn, st.wn, st.rho, st.signs, st.dual, st.pd_out)], 0.1, 1.0, op, _lib.stream_handle())
    for fl in (True, False):
        for _ in range(10):
            run()
        ts = []
        for _ in range(100):
            if fl:
                sink.copy_(flush.sum().reshape(1))
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); run(); b.record()
            ts.append((a, b))
        torch.cuda.synchronize()
        ms = sorted(x.elapsed_time(y) for x, y in ts)[len(ts) // 2]
        print(f"{shape} variant {v} op {op} flush={fl}: {ms*1e3:.1f} us  {B/ms/1e6:.0f} GB/s  "
              f"{units/148/(ms*1e3):.3f} units/us/SM")
