"""Time tsg_pack / tsg_unpack (Atlas <-> structured reorder) at 1024x1024x80 for the SN /
UN / HN numberings and check pack against unpack's inverse; the pack kernel variant comes
from TSG_PACK_V (A/B builds).  python tools/pack_variants.py"""
import json
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1908_06094_b200 import LocationType as L, Numbering, PatchSpec, _lib, element_count, make_permutation  # noqa: E402
from paper_1908_06094_b200.device import DeviceGrid  # noqa: E402

R, C, K = 1024, 1024, 80
PEAK = 6455.0
flush = torch.ones(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
sink = torch.empty(1, dtype=torch.float64, device="cuda")
s = _lib.stream_handle()


def timed(fn, reps=50):
    fn()
    ev = []
    for _ in range(reps):
        sink.copy_(flush.sum().reshape(1))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(100_000)
        a.record()
        fn()
        b.record()
        ev.append((a, b))
    torch.cuda.synchronize()
    return sum(x.elapsed_time(y) for x, y in ev) / len(ev) / 1e3


spec = PatchSpec(R, C, K)
g = DeviceGrid(R, C, K)
n = element_count(spec, L.CELLS)
b = g.empty(1, K)
b2 = g.empty(1, K)
flat = torch.rand((n, K), dtype=torch.float64, device="cuda")
back = torch.empty_like(flat)
for num in (Numbering.SN, Numbering.UN, Numbering.HN):
    fwd = torch.as_tensor(make_permutation(num, spec, L.CELLS).forward, device="cuda")
    t = timed(lambda: _lib.call("tsg_pack", g.handle, 1, K, _lib.ptr(flat), _lib.ptr(fwd), _lib.ptr(b), s))
    _lib.call("tsg_unpack", g.handle, 1, K, _lib.ptr(b), _lib.ptr(fwd), _lib.ptr(back), s)
    ok = bool(torch.equal(back, flat))
    print(json.dumps({"variant": os.environ.get("TSG_PACK_V", "0"), "num": num.value, "pack_us": round(t * 1e6, 1),
                      "frac": round(2 * n * K * 8 / t / 1e9 / PEAK, 3), "roundtrip": ok}), flush=True)
