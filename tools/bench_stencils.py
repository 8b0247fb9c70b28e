"""Secondary benchmarks of the non-MPDATA rows of SURVEY 8(a)/(f) on one B200.

Prints one JSON object per measurement (and writes them to gpurun_out/stencils_<tag>.json):
  * Table 1: B = sum_nbr A and B = (sum_nbr A) * fac on cells,
    structured direct vs table-driven SN / UN / HN, at 128x128x80 (the paper's patch) and
    1024x1024x80 (L2-busting); effective GB/s = required data transfer / time, the paper's
    metric (bytes: 2 * cells * K * 8 (+ cells * 8)).
  * the 9 neighbour relations at 256x256x80 (bytes (n_from + n_to) * K * 8);
  * cell divergence simple / weighted;
  * fusion study (Table 2 / Fig. 14 analogue): unfused 4-kernel step vs fused step at
    279x256x80 with their algorithmic bytes;
  * the Atlas -> structured reorder (tsg_pack / tsg_unpack) under SN / UN / HN.
Every timed launch is preceded by a 256 MiB read-only L2 flush (outside the events).
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_1908_06094_b200 import (LocationType as L, Numbering, OFFSET_TABLES, PatchSpec, _lib,  # noqa: E402
                                   build_neighbor_table, element_count, make_permutation)
from paper_1908_06094_b200.device import DeviceGrid  # noqa: E402

_pk = Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json"
PEAK = json.loads(_pk.read_text())["hbm_gbs"] if _pk.exists() else 6650.0  # fallback (B200_PROFILING.md)
flush = torch.ones(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
sink = torch.empty(1, dtype=torch.float64, device="cuda")
OUT = []


def timed(fn, reps=100, warm=3):
    """Mean device time of ``fn`` over ``reps`` launches, each after an L2 flush and a ~50 us
    device sleep (so the launch is queued before the GPU reaches it: no host preparation
    inside the events).  The mean, because event timestamps tick every ~2 us here."""
    for _ in range(warm):
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


def record(name, seconds, nbytes, **kw):
    gbs = nbytes / seconds / 1e9
    d = dict(name=name, us=seconds * 1e6, bytes=nbytes, gbs=gbs, frac=gbs / PEAK, **kw)
    OUT.append(d)
    print(json.dumps(d), flush=True)


def s():
    return _lib.stream_handle()


def table1(rows, cols, K):
    spec = PatchSpec(rows, cols, K)
    g = DeviceGrid(rows, cols, K)
    n = element_count(spec, L.CELLS)
    a = g.empty(1, K)
    fac = g.empty(1, 1)
    b = g.empty(1, K)
    _lib.call("tsg_fill_hash", g.handle, 1, K, 1, 0.0, 1.0, _lib.ptr(a), s())
    _lib.call("tsg_fill_hash", g.handle, 1, 1, 2, 0.5, 1.5, _lib.ptr(fac), s())
    for key, scale in (("k1", None), ("k2", fac)):
        nbytes = 2 * n * K * 8 + (n * 8 if scale is not None else 0)
        t = timed(lambda: _lib.call("tsg_neighbor_reduce", g.handle, 1, 1, K, _lib.ptr(a), _lib.ptr(scale),
                                    _lib.ptr(b), s()))
        record(f"table1_{key}_SN_direct", t, nbytes, patch=[rows, cols, K])
    flat_a = torch.empty((n, K), dtype=torch.float64, device="cuda")
    flat_b = torch.empty_like(flat_a)
    flat_fac = torch.empty(n, dtype=torch.float64, device="cuda")
    for num in (Numbering.SN, Numbering.UN, Numbering.HN):
        perm = make_permutation(num, spec, L.CELLS)
        fwd = torch.as_tensor(perm.forward, device="cuda")
        table = build_neighbor_table(spec, L.CELLS, L.CELLS, perm, perm, as_tensor=True).ids
        _lib.call("tsg_unpack", g.handle, 1, K, _lib.ptr(a), _lib.ptr(fwd), _lib.ptr(flat_a), s())
        _lib.call("tsg_unpack", g.handle, 1, 1, _lib.ptr(fac), _lib.ptr(fwd), _lib.ptr(flat_fac), s())
        for key, scale in (("k1", None), ("k2", flat_fac)):
            nbytes = 2 * n * K * 8 + (n * 8 if scale is not None else 0)
            t = timed(lambda: _lib.call("tsg_neighbor_reduce_indirect", _lib.ptr(table), n, 3, K,
                                        _lib.ptr(flat_a), _lib.ptr(scale), _lib.ptr(flat_b), s()))
            record(f"table1_{key}_{num.value.upper()}_indirect", t, nbytes, patch=[rows, cols, K])
        # the reorder itself (Atlas -> structured, and back)
        t = timed(lambda: _lib.call("tsg_pack", g.handle, 1, K, _lib.ptr(flat_a), _lib.ptr(fwd), _lib.ptr(b), s()))
        record(f"pack_cells_{num.value.upper()}", t, 2 * n * K * 8, patch=[rows, cols, K])
        t = timed(lambda: _lib.call("tsg_unpack", g.handle, 1, K, _lib.ptr(b), _lib.ptr(fwd), _lib.ptr(flat_a), s()))
        record(f"unpack_cells_{num.value.upper()}", t, 2 * n * K * 8, patch=[rows, cols, K])


def relations(rows, cols, K):
    spec = PatchSpec(rows, cols, K)
    g = DeviceGrid(rows, cols, K)
    for (f, t) in OFFSET_TABLES:
        src = g.empty(t.code, K)
        dst = g.empty(f.code, K)
        _lib.call("tsg_fill_hash", g.handle, t.code, K, 3, 0.0, 1.0, _lib.ptr(src), s())
        nbytes = (element_count(spec, f) + element_count(spec, t)) * K * 8
        tt = timed(lambda: _lib.call("tsg_neighbor_reduce", g.handle, f.code, t.code, K, _lib.ptr(src), None,
                                     _lib.ptr(dst), s()))
        record(f"reduce_{f.value[0].upper()}{t.value[0].upper()}", tt, nbytes, patch=[rows, cols, K])


def cell_div(rows, cols, K):
    g = DeviceGrid(rows, cols, K)
    vn, length, area, w, out = g.empty(2, K), g.empty(2, 1), g.empty(1, 1), g.empty(1, 3), g.empty(1, K)
    for f, loc, inner, lo, hi in ((vn, 2, K, -0.5, 0.5), (length, 2, 1, 0.5, 1.5), (area, 1, 1, 0.2, 0.6)):
        _lib.call("tsg_fill_hash", g.handle, loc, inner, 4, lo, hi, _lib.ptr(f), s())
    _lib.call("tsg_cell_weights", g.handle, _lib.ptr(length), _lib.ptr(area), _lib.ptr(w), s())
    nv = rows * cols
    for weighted in (0, 1):
        nbytes = (3 * nv + 2 * nv) * K * 8 + (2 * nv * 3 * 8 if weighted else (3 * nv + 2 * nv) * 8)
        t = timed(lambda: _lib.call("tsg_cell_divergence", g.handle, weighted, _lib.ptr(vn), _lib.ptr(length),
                                    _lib.ptr(area), _lib.ptr(w), _lib.ptr(out), s()))
        record(f"cell_divergence_{'weighted' if weighted else 'simple'}", t, nbytes, patch=[rows, cols, K])


def fusion(rows, cols, K):
    g = DeviceGrid(rows, cols, K)
    f = {}
    for name, loc, inner, lo, hi in (("pd", 0, K, 0, 1), ("vn", 2, K, -.5, .5), ("wn", 0, K + 1, -.5, .5),
                                     ("rho", 0, K, 1, 1), ("dual", 0, 1, .5, 1.5)):
        f[name] = g.empty(loc, inner)
        _lib.call("tsg_fill_hash", g.handle, loc, inner, 5, float(lo), float(hi), _lib.ptr(f[name]), s())
    signs = g.empty(0, 6)
    flat = torch.empty((rows * cols, 6), dtype=torch.float64, device="cuda")
    _lib.call("tsg_edge_signs", rows, cols, _lib.ptr(flat), s())
    _lib.call("tsg_pack", g.handle, 0, 6, _lib.ptr(flat), None, _lib.ptr(signs), s())
    out, flux, fluz, div = g.empty(0, K), g.empty(2, K), g.empty(0, K + 1), g.empty(0, K)
    ins = [_lib.ptr(f[n]) for n in ("pd", "vn", "wn", "rho")] + [_lib.ptr(signs), _lib.ptr(f["dual"])]
    v, e = rows * cols, 3 * rows * cols
    fused_bytes = 8 * (v * K + e * K + v * (K - 1) + v * K + v * K)
    unfused_bytes = 8 * (3 * e * K + 7 * v * K + 2 * v * (K + 1) + v * (K - 1))
    t = timed(lambda: _lib.call("tsg_mpdata_step", g.handle, *ins, _lib.ptr(out), 0.1, 1.0, 0, s()))
    record("mpdata_fused", t, fused_bytes, patch=[rows, cols, K], updates_per_s=v * K / t)
    t2 = timed(lambda: _lib.call("tsg_mpdata_step_unfused", g.handle, *ins, _lib.ptr(flux), _lib.ptr(fluz),
                                 _lib.ptr(div), _lib.ptr(out), 0.1, 1.0, 0, s()))
    record("mpdata_unfused", t2, unfused_bytes, patch=[rows, cols, K], updates_per_s=v * K / t2,
           fused_speedup=t2 / t, bytes_ratio=unfused_bytes / fused_bytes)
    if K % 2 or rows * cols > 1 << 20:
        return
    # the flat oracle API (reference.py:93-116) through the table-driven kernels, SN order
    e2v = build_neighbor_table(PatchSpec(rows, cols, K), L.EDGES, L.VERTICES, as_tensor=True).ids
    v2e = build_neighbor_table(PatchSpec(rows, cols, K), L.VERTICES, L.EDGES, as_tensor=True).ids
    fl = {n: torch.rand((cnt, w), dtype=torch.float64, device="cuda")
          for n, cnt, w in (("pd", v, K), ("vn", e, K), ("wn", v, K + 1), ("rho", v, K), ("signs", v, 6),
                            ("dual", v, 1), ("flux", e, K), ("fluz", v, K + 1), ("div", v, K), ("out", v, K))}
    fl["rho"] += 0.5
    t3 = timed(lambda: _lib.call("tsg_transport_indirect", _lib.ptr(e2v), _lib.ptr(v2e), _lib.ptr(fl["signs"]),
                                 _lib.ptr(fl["dual"]), _lib.ptr(fl["pd"]), _lib.ptr(fl["vn"]), _lib.ptr(fl["wn"]),
                                 _lib.ptr(fl["rho"]), v, e, K, 0.1, 1.0, 0, _lib.ptr(fl["flux"]),
                                 _lib.ptr(fl["fluz"]), _lib.ptr(fl["div"]), _lib.ptr(fl["out"]), s()))
    # materialised flux / fluz / div: the unfused DISTINCT bytes plus the div output
    record("mpdata_indirect", t3, unfused_bytes + 8 * v * K, patch=[rows, cols, K], updates_per_s=v * K / t3)


def launch_floor():
    """The protocol's fixed cost: an empty launch between the same CUDA events after the
    same L2 flush (no kernel at all: just the events' own interval)."""
    record("launch_floor_empty_kernel", timed(lambda: torch.cuda._sleep(1)), 0)
    record("launch_floor_no_kernel", timed(lambda: None), 0)


if __name__ == "__main__":
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    only = set(sys.argv[2].split(",")) if len(sys.argv) > 2 else None  # e.g. "fusion,table1"
    for name, fn, args in (("floor", launch_floor, ()), ("table1", table1, (128, 128, 80)),
                           ("table1", table1, (1024, 1024, 80)), ("relations", relations, (256, 256, 80)),
                           ("relations", relations, (1024, 1024, 80)), ("cell_div", cell_div, (256, 256, 80)),
                           ("cell_div", cell_div, (1024, 1024, 80)), ("fusion", fusion, (279, 256, 80)),
                           ("fusion", fusion, (2560, 2576, 137))):
        if only is None or name in only:
            fn(*args)
    Path("gpurun_out").mkdir(exist_ok=True)
    Path(f"gpurun_out/stencils_{tag}.json").write_text(json.dumps(OUT, indent=1))
