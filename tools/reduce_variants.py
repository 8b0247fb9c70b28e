"""A/B of the TMA neighbour reduce's compact tile shapes (tsg_set_reduce_variant) on one
B200, per relation at 256x256x80 (the bench_stencils patch), with a plain device copy of
the same bytes as the practical ceiling.  Every variant's output is checked bitwise
against the default shape's.  L2 flushed (256 MiB read) before every timed launch.

usage: python tools/reduce_variants.py [rows cols K [variant,variant,...]]
       python tools/reduce_variants.py celldiv rows cols K [variant,...]   (cell divergence)
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_1908_06094_b200 import OFFSET_TABLES, PatchSpec, _lib, element_count  # noqa: E402
from paper_1908_06094_b200.device import DeviceGrid  # noqa: E402

_pk = Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json"
PEAK = json.loads(_pk.read_text())["hbm_gbs"] if _pk.exists() else 6650.0
flush = torch.ones(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
sink = torch.empty(1, dtype=torch.float64, device="cuda")


def timed(fn, reps=200, warm=3):
    for _ in range(warm):
        fn()
    ev = []
    for _ in range(reps):
        sink.copy_(flush.sum().reshape(1))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(100_000)  # ~50 us: the launch below is queued before the GPU gets there
        a.record()
        fn()
        b.record()
        ev.append((a, b))
    torch.cuda.synchronize()
    # the mean: event timestamps tick every ~2 us on these boxes, so a median is quantised
    ts = [x.elapsed_time(y) for x, y in ev]
    return sum(ts) / len(ts) / 1e3


def cell_divergence(rows, cols, K, pick):
    """The same A/B for tsg_cell_divergence (simple and weighted: cells <- edges with edge
    weights; cell tile variants 1-9 static, 11-19 dealt)."""
    g = DeviceGrid(rows, cols, K)
    s = _lib.stream_handle()
    vn, length, area, w = g.empty(2, K), g.empty(2, 1), g.empty(1, 1), g.empty(1, 3)
    for f, loc, inner, lo in ((vn, 2, K, -0.5), (length, 2, 1, 0.5), (area, 1, 1, 0.5)):
        _lib.call("tsg_fill_hash", g.handle, loc, inner, 4, lo, lo + 1.0, _lib.ptr(f), s)
    _lib.call("tsg_cell_weights", g.handle, _lib.ptr(length), _lib.ptr(area), _lib.ptr(w), s)
    nv = rows * cols
    for weighted in (0, 1):
        nbytes = (3 * nv + 2 * nv) * K * 8 + (2 * nv * 3 * 8 if weighted else (3 * nv + 2 * nv) * 8)
        ref, out = g.empty(1, K), g.empty(1, K)
        call = lambda o: _lib.call("tsg_cell_divergence", g.handle, weighted, _lib.ptr(vn), _lib.ptr(length),
                                   _lib.ptr(area), _lib.ptr(w), _lib.ptr(o), s)
        _lib.call("tsg_set_reduce_variant", 0)
        call(ref)
        for v in pick:
            _lib.call("tsg_set_reduce_variant", v)
            out.zero_()
            tt = timed(lambda: call(out))
            print(json.dumps(dict(name=f"cell_divergence_{'weighted' if weighted else 'simple'}", variant=v,
                                  us=round(tt * 1e6, 2), frac=round(nbytes / tt / 1e9 / PEAK, 4),
                                  bitwise=bool(torch.equal(out, ref)))), flush=True)
        _lib.call("tsg_set_reduce_variant", 0)


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "celldiv":  # celldiv rows cols K [variants]
        rows, cols, K = (int(x) for x in sys.argv[2:5])
        pick = [int(x) for x in sys.argv[5].split(",")] if len(sys.argv) > 5 else \
            list(range(0, 10)) + list(range(11, 20))
        return cell_divergence(rows, cols, K, pick)
    rows, cols, K = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (256, 256, 80)
    spec = PatchSpec(rows, cols, K)
    g = DeviceGrid(rows, cols, K)
    s = _lib.stream_handle()
    variants = {1: list(range(0, 10)) + list(range(11, 20)), 2: list(range(0, 6)) + list(range(11, 16)),
                3: [0, 1, 2, 11, 12]}
    if len(sys.argv) > 4:
        pick = [int(x) for x in sys.argv[4].split(",")]
        variants = {c: [v for v in vs if v in pick] for c, vs in variants.items()}
    for (f, t) in OFFSET_TABLES:
        src = g.empty(t.code, K)
        dst = g.empty(f.code, K)
        ref = g.empty(f.code, K)
        _lib.call("tsg_fill_hash", g.handle, t.code, K, 3, 0.0, 1.0, _lib.ptr(src), s)
        nbytes = (element_count(spec, f) + element_count(spec, t)) * K * 8
        name = f"reduce_{f.value[0].upper()}{t.value[0].upper()}"
        _lib.call("tsg_set_reduce_variant", 0)
        _lib.call("tsg_neighbor_reduce", g.handle, f.code, t.code, K, _lib.ptr(src), None, _lib.ptr(ref), s)
        for v in variants[t.colors]:
            _lib.call("tsg_set_reduce_variant", v)
            dst.zero_()
            fn = lambda: _lib.call("tsg_neighbor_reduce", g.handle, f.code, t.code, K, _lib.ptr(src), None,
                                   _lib.ptr(dst), s)
            tt = timed(fn)
            same = bool(torch.equal(dst, ref))
            print(json.dumps(dict(name=name, variant=v, us=round(tt * 1e6, 2),
                                  frac=round(nbytes / tt / 1e9 / PEAK, 4), bitwise=same)), flush=True)
        _lib.call("tsg_set_reduce_variant", 0)
        # the ceiling: one device copy moving the same bytes (read n_src, write n_dst elements)
        a = torch.empty(element_count(spec, t) * K, dtype=torch.float64, device="cuda").fill_(1.0)
        b = torch.empty(element_count(spec, f) * K, dtype=torch.float64, device="cuda")
        m = min(a.numel(), b.numel())
        tc = timed(lambda: b[:m].copy_(a[:m]))
        print(json.dumps(dict(name=name, variant="copy", us=round(tc * 1e6, 2),
                              frac=round(2 * m * 8 / tc / 1e9 / PEAK, 4))), flush=True)


if __name__ == "__main__":
    main()
