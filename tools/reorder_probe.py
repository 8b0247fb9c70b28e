"""tsg_pack / tsg_unpack (the Atlas -> structured reorder) on one field at a given level
count, canonical numbering and a random permutation: time after an L2 flush (mean of 20)
and the fraction of the copy peak for 2 x elements x levels x 8 bytes.
    python tools/reorder_probe.py rows cols levels [loc]"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1908_06094_b200 import _lib  # noqa: E402
from paper_1908_06094_b200.device import DeviceGrid  # noqa: E402

R, C, K = (int(x) for x in sys.argv[1:4])
loc = int(sys.argv[4]) if len(sys.argv) > 4 else 2
_pk = Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json"
PEAK = json.loads(_pk.read_text())["hbm_gbs"] if _pk.exists() else 6650.0
g = DeviceGrid(R, C, K)
n = R * C * (3 if loc == 2 else 2 if loc == 1 else 1)
flat = torch.rand(n, K, dtype=torch.float64, device="cuda")
back = torch.empty_like(flat)
f = g.empty(loc, K)
s = _lib.stream_handle()
flush = torch.ones(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
perm = torch.randperm(n, device="cuda")
for name, fwd in (("sn", None), ("random", perm)):
    for what, fn in (("pack", lambda: _lib.call("tsg_pack", g.handle, loc, K, _lib.ptr(flat), _lib.ptr(fwd) if fwd is not None else None, _lib.ptr(f), s)),
                     ("unpack", lambda: _lib.call("tsg_unpack", g.handle, loc, K, _lib.ptr(f), _lib.ptr(fwd) if fwd is not None else None, _lib.ptr(back), s))):
        fn()
        ts = []
        for _ in range(20):
            flush.sum()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda._sleep(100_000)
            a.record()
            fn()
            b.record()
            ts.append((a, b))
        torch.cuda.synchronize()
        t = sum(x.elapsed_time(y) for x, y in ts) / len(ts) / 1e3
        print(json.dumps(dict(op=what, numbering=name, patch=[R, C, K], loc=loc, us=round(t * 1e6, 1),
                              frac=round(2 * n * K * 8 / t / 1e9 / PEAK, 3))), flush=True)
    assert torch.equal(back, flat)
