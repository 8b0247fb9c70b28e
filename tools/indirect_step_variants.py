"""Time the table-driven step (tsg_transport_indirect: flux, fluz, divergence + update
over flat arrays, the reference.transport_step call) at 279x256x80 and 1024x1024x80; the
gather kernels' form comes from TSG_IPIPE (A/B builds).  Prints a checksum of pd_out.
python tools/indirect_step_variants.py"""
import hashlib
import json
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1908_06094_b200 import LocationType as L, PatchSpec, _lib, build_neighbor_table  # noqa: E402

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


for rows, cols, K in ((279, 256, 80), (1024, 1024, 80)):
    v, e = rows * cols, 3 * rows * cols
    e2v = build_neighbor_table(PatchSpec(rows, cols, K), L.EDGES, L.VERTICES, as_tensor=True).ids
    v2e = build_neighbor_table(PatchSpec(rows, cols, K), L.VERTICES, L.EDGES, as_tensor=True).ids
    g = torch.Generator(device="cuda").manual_seed(0)
    fl = {n: torch.rand((cnt, w), dtype=torch.float64, device="cuda", generator=g)
          for n, cnt, w in (("pd", v, K), ("vn", e, K), ("wn", v, K + 1), ("rho", v, K), ("signs", v, 6),
                            ("dual", v, 1), ("flux", e, K), ("fluz", v, K + 1), ("div", v, K), ("out", v, K))}
    fl["rho"] += 0.5
    args = [_lib.ptr(e2v), _lib.ptr(v2e)] + [_lib.ptr(fl[n]) for n in ("signs", "dual", "pd", "vn", "wn", "rho")]
    outs = [_lib.ptr(fl[n]) for n in ("flux", "fluz", "div", "out")]
    t = timed(lambda: _lib.call("tsg_transport_indirect", *args, v, e, K, 0.1, 1.0, 0, *outs, s))
    nbytes = 8 * (3 * e * K + 7 * v * K + 2 * v * (K + 1) + v * (K - 1)) + 8 * v * K
    h = hashlib.sha256(fl["out"].cpu().numpy().tobytes() + fl["div"].cpu().numpy().tobytes()).hexdigest()[:16]
    print(json.dumps({"variant": os.environ.get("TSG_IPIPE", "0"), "patch": [rows, cols, K],
                      "us": round(t * 1e6, 1), "frac": round(nbytes / t / 1e9 / PEAK, 3), "sha": h}), flush=True)
