"""The reference's flat stages one at a time (reference.py:18-90, 119-134) through the C ABI
(tsg_flat_flux / _fluz / _divergence / _advance / _cell_divergence, and the Table-1 gathers
tsg_neighbor_reduce_indirect) on flat canonical arrays:
time per call after an L2 flush (mean of 50) and the fraction of the measured copy peak
for each stage's DISTINCT bytes.   python tools/flat_stages_probe.py [rows cols K]"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1908_06094_b200 import LocationType as L, PatchSpec, _lib, build_neighbor_table  # noqa: E402

_pk = Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json"
PEAK = json.loads(_pk.read_text())["hbm_gbs"] if _pk.exists() else 6650.0
flush = torch.ones(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
sink = torch.empty(1, dtype=torch.float64, device="cuda")


def timed(fn, reps=50):
    for _ in range(3):
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


R, C, K = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (1024, 1024, 80)
spec = PatchSpec(R, C, K)
nv, ne, nc = R * C, 3 * R * C, 2 * R * C
e2v = build_neighbor_table(spec, L.EDGES, L.VERTICES, as_tensor=True).ids
v2e = build_neighbor_table(spec, L.VERTICES, L.EDGES, as_tensor=True).ids
c2e = build_neighbor_table(spec, L.CELLS, L.EDGES, as_tensor=True).ids
c2c = build_neighbor_table(spec, L.CELLS, L.CELLS, as_tensor=True).ids
f64 = dict(dtype=torch.float64, device="cuda")
pd, rho = torch.rand(nv, K, **f64) + 0.5, torch.rand(nv, K, **f64) + 0.5
vn, wn = torch.rand(ne, K, **f64) - 0.5, torch.rand(nv, K + 1, **f64) - 0.5
signs, dual = torch.rand(nv, 6, **f64), torch.rand(nv, **f64) + 0.5
length, area = torch.rand(ne, **f64) + 0.5, torch.rand(nc, **f64) + 0.5
flux, fluz, div, out = torch.empty(ne, K, **f64), torch.empty(nv, K + 1, **f64), torch.empty(nv, K, **f64), \
    torch.empty(nv, K, **f64)
cdiv = torch.empty(nc, K, **f64)
ca, cb, fac = torch.rand(nc, K, **f64), torch.empty(nc, K, **f64), torch.rand(nc, **f64) + 0.5
s = _lib.stream_handle()
p = _lib.ptr
stages = {
    "flat_flux": (lambda: _lib.call("tsg_flat_flux", p(e2v), p(pd), p(vn), ne, K, 0, p(flux), s),
                  8 * (ne * 2 + nv * K + 2 * ne * K)),
    "flat_fluz": (lambda: _lib.call("tsg_flat_fluz", p(pd), p(wn), nv, K, 1.0, p(fluz), s),
                  8 * (nv * K + 2 * nv * (K + 1))),
    "flat_divergence": (lambda: _lib.call("tsg_flat_divergence", p(v2e), 6, p(signs), p(dual), p(flux), p(fluz), nv,
                                          K, p(div), s),
                        8 * (nv * 13 + ne * K + nv * (K + 1) + nv * K)),
    "flat_advance": (lambda: _lib.call("tsg_flat_advance", p(pd), p(div), p(rho), nv * K, 0.1, p(out), s),
                     8 * 4 * nv * K),
    "flat_cell_divergence": (lambda: _lib.call("tsg_flat_cell_divergence", p(c2e), 3, p(vn), p(length), p(area), nc, K,
                                               p(cdiv), s),
                             8 * (nc * 3 + ne * K + ne + nc + nc * K)),
    "flat_neighbor_sum": (lambda: _lib.call("tsg_neighbor_reduce_indirect", p(c2c), nc, 3, K, p(ca), None, p(cb), s),
                          8 * 2 * nc * K),
    "flat_neighbor_sum_scaled": (lambda: _lib.call("tsg_neighbor_reduce_indirect", p(c2c), nc, 3, K, p(ca), p(fac),
                                                   p(cb), s), 8 * (2 * nc * K + nc)),
}
for name, (fn, nbytes) in stages.items():
    t = timed(fn)
    print(json.dumps(dict(name=name, patch=[R, C, K], us=round(t * 1e6, 1),
                          frac=round(nbytes / t / 1e9 / PEAK, 3))), flush=True)
