"""Time tsg_cell_divergence (simple / weighted) at 256^2 and 1024^2 x 80 (L2 flushed, device sleep ahead).
TSG_NODYN_MODE=1 keeps the static schedule for the weighted modes (A/B builds)."""
import sys, json, os
sys.path.insert(0, "/root/repo")
import torch
from paper_1908_06094_b200 import _lib
from paper_1908_06094_b200.device import DeviceGrid
flush = torch.ones(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda"); sink = torch.empty(1, dtype=torch.float64, device="cuda")
s = _lib.stream_handle()
def timed(fn, reps=50):
    fn(); ev = []
    for _ in range(reps):
        sink.copy_(flush.sum().reshape(1)); a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(100_000); a.record(); fn(); b.record(); ev.append((a, b))
    torch.cuda.synchronize(); return sum(x.elapsed_time(y) for x, y in ev) / len(ev) / 1e3
for rows, cols, K in ((256, 256, 80), (1024, 1024, 80)):
    g = DeviceGrid(rows, cols, K)
    vn, length, area, w, out = g.empty(2, K), g.empty(2, 1), g.empty(1, 1), g.empty(1, 3), g.empty(1, K)
    for f, loc, inner, lo, hi in ((vn, 2, K, -0.5, 0.5), (length, 2, 1, 0.5, 1.5), (area, 1, 1, 0.2, 0.6)):
        _lib.call("tsg_fill_hash", g.handle, loc, inner, 4, lo, hi, _lib.ptr(f), s)
    _lib.call("tsg_cell_weights", g.handle, _lib.ptr(length), _lib.ptr(area), _lib.ptr(w), s)
    nv = rows * cols
    for weighted in (0, 1):
        nbytes = (3 * nv + 2 * nv) * K * 8 + (2 * nv * 3 * 8 if weighted else (3 * nv + 2 * nv) * 8)
        t = timed(lambda: _lib.call("tsg_cell_divergence", g.handle, weighted, _lib.ptr(vn), _lib.ptr(length), _lib.ptr(area), _lib.ptr(w), _lib.ptr(out), s))
        print(os.environ.get("TSG_NODYN_MODE", "0"), rows, weighted, round(t * 1e6, 1), round(nbytes / t / 1e9 / 6455, 3), float(out.sum()))
