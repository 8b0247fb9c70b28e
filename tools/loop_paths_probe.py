"""The 279x256x80 persistent loop through StructuredStepper.run and StripStepper.run (world
1, the bench's path) on the same inputs and box, with and without the bench's L2 flush +
device sleep ahead of the timed launch.  python tools/loop_paths_probe.py"""
import statistics
import sys

sys.path.insert(0, "/root/repo")
import torch  # noqa: E402

from paper_1908_06094_b200 import PatchSpec, StructuredStepper  # noqa: E402
from paper_1908_06094_b200.distributed import StripStepper  # noqa: E402
from paper_1908_06094_b200.workloads import transport_inputs  # noqa: E402

R, C, K = 279, 256, 80
N = 200
inp = transport_inputs(R, C, K)
ss = StructuredStepper(PatchSpec(R, C, K))
ss.set_geometry(inp["signs"], inp["dual"])
ss.upload(inp["pd"], inp["vn"], inp["wn"], inp["rho"])
sp = StripStepper(R, C, K, 0, 1, seed=0)
sp.load_flat(inp["pd"], inp["vn"], inp["wn"], inp["rho"], inp["dual"].reshape(-1, 1))
flush = torch.ones(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
sink = torch.empty(1, dtype=torch.float64, device="cuda")


def timed(st, pre):
    st.run(N, 0.1, 1.0)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        if pre:
            sink.copy_(flush.sum().reshape(1))
            torch.cuda._sleep(200_000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        st.run(N, 0.1, 1.0)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3 / N)
    return statistics.median(ts)


for rep in range(2):
    for name, st in (("StructuredStepper", ss), ("StripStepper", sp)):
        for pre in (False, True):
            print(f"{name:18s} flush+sleep={pre!s:5s} {timed(st, pre):6.2f} us/step", flush=True)
print("grids:", ss.grid.rows, ss.grid.cols, sp.grid.rows, sp.grid.cols)
