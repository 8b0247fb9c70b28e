"""Quick timing of fused-kernel variants (L2 flushed, CUDA events): python tools/time_fused.py [op] [variants...]"""
import sys
sys.path.insert(0, "/root/repo")
import torch
from paper_1908_06094_b200 import PatchSpec, StructuredStepper, _lib
from paper_1908_06094_b200.workloads import transport_inputs, mpdata_algorithmic_bytes

op = int(sys.argv[1]) if len(sys.argv) > 1 else 0
variants = [int(v) for v in sys.argv[2:]] or [0]
shape = (279, 256, 80)
inp = transport_inputs(*shape)
st = StructuredStepper(PatchSpec(*shape))
st.set_geometry(inp["signs"], inp["dual"])
st.upload(inp["pd"], inp["vn"], inp["wn"], inp["rho"])
flush = torch.ones(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
sink = torch.empty(1, dtype=torch.float64, device="cuda")
B = mpdata_algorithmic_bytes(*shape)
for v in variants:
    _lib.call("tsg_set_fused_variant", v)
    def run():
        _lib.call("tsg_mpdata_step", st.grid.handle, *[_lib.ptr(t) for t in (st.pd, st.vn, st.wn, st.rho, st.signs, st.dual, st.pd_out)], 0.1, 1.0, op, _lib.stream_handle())
    for _ in range(10):
        run()
    ts = []
    for _ in range(200):
        sink.copy_(flush.sum().reshape(1))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); run(); b.record()
        ts.append((a, b))
    torch.cuda.synchronize()
    ms = sorted(x.elapsed_time(y) for x, y in ts)
    mean = sum(ms) / len(ms)
    print(f"variant {v} op {op}: mean {mean*1e3:.1f} us  median {ms[len(ms)//2]*1e3:.1f}  -> {B/mean/1e6:.0f} GB/s ({B/mean/1e6/6537.6*100:.1f}%)")
