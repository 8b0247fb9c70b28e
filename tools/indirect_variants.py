"""Time the Table-1 indirect gather (tsg_neighbor_reduce_indirect, C->C, width 3) k1 / k2
at 1024x1024x80 for SN / UN / HN; the kernel form comes from TSG_IND_V (A/B builds).
Prints a checksum of the output so forms can be compared bitwise across processes.
python tools/indirect_variants.py"""
import hashlib
import json
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1908_06094_b200 import (LocationType as L, Numbering, PatchSpec, _lib,  # noqa: E402
                                   build_neighbor_table, element_count, make_permutation)

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
n = element_count(spec, L.CELLS)
g = torch.Generator(device="cuda").manual_seed(0)
a = torch.rand((n, K), dtype=torch.float64, device="cuda", generator=g)
fac = 0.5 + torch.rand(n, dtype=torch.float64, device="cuda", generator=g)
b = torch.empty_like(a)
for num in (Numbering.SN, Numbering.UN, Numbering.HN):
    perm = make_permutation(num, spec, L.CELLS)
    table = build_neighbor_table(spec, L.CELLS, L.CELLS, perm, perm, as_tensor=True).ids
    for key, scale in (("k1", None), ("k2", fac)):
        t = timed(lambda: _lib.call("tsg_neighbor_reduce_indirect", _lib.ptr(table), n, 3, K, _lib.ptr(a),
                                    _lib.ptr(scale), _lib.ptr(b), s))
        h = hashlib.sha256(b.cpu().numpy().tobytes()).hexdigest()[:16]
        nbytes = 2 * n * K * 8 + (n * 8 if scale is not None else 0)
        print(json.dumps({"variant": os.environ.get("TSG_IND_V", "0"), "num": num.value, "key": key,
                          "us": round(t * 1e6, 1), "frac": round(nbytes / t / 1e9 / PEAK, 3), "sha": h}), flush=True)
