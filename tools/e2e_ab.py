"""e2e (run_pipelined) under both work deals on one box: python tools/e2e_ab.py"""
import sys

sys.path.insert(0, "/root/repo")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1908_06094_b200 import PatchSpec, StructuredStepper, _lib  # noqa: E402
from paper_1908_06094_b200.workloads import transport_inputs  # noqa: E402

R, C, K = 279, 256, 80
inp = transport_inputs(R, C, K)
st = StructuredStepper(PatchSpec(R, C, K))
st.set_geometry(inp["signs"], inp["dual"])
st.upload(inp["pd"], inp["vn"], inp["wn"], inp["rho"])
pinned = [torch.from_numpy(np.ascontiguousarray(inp[n])).pin_memory() for n in ("pd", "vn", "wn", "rho")]
outs = [torch.empty((R * C, K), dtype=torch.float64).pin_memory() for _ in range(2)]
for sched in (1, 0, 1, 0):
    _lib.call("tsg_set_fused_schedule", sched)
    st.run_pipelined([pinned] * 3, outs + outs[:1], 0.1, 1.0)
    torch.cuda.synchronize()
    n = 40
    e0, e1 = st.run_pipelined([[pinned[0], None, None, None]] * n, [outs[i % 2] for i in range(n)], 0.1, 1.0)
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / n
    print(f"sched {sched}: e2e {t:.3f} ms/step  {2 * R * C * K * 8 / t / 1e6:.1f} GB/s PCIe", flush=True)
# raw copy speeds for reference
x = torch.empty(R * C * K, dtype=torch.float64, device="cuda")
for _ in range(2):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); x.copy_(pinned[0].view(-1), non_blocking=True); b.record(); torch.cuda.synchronize()
    print(f"H2D alone {a.elapsed_time(b):.3f} ms ({x.numel() * 8 / a.elapsed_time(b) / 1e6:.1f} GB/s)")
    a.record(); outs[0].view(-1).copy_(x, non_blocking=True); b.record(); torch.cuda.synchronize()
    print(f"D2H alone {a.elapsed_time(b):.3f} ms ({x.numel() * 8 / a.elapsed_time(b) / 1e6:.1f} GB/s)")
