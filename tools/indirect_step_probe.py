import sys, json
sys.path.insert(0, "/root/repo")
import torch
from paper_1908_06094_b200 import LocationType as L, PatchSpec, _lib, build_neighbor_table
R, C, K = (int(a) for a in sys.argv[1:4])
spec = PatchSpec(R, C, K)
v, e = R * C, 3 * R * C
e2v = build_neighbor_table(spec, L.EDGES, L.VERTICES, as_tensor=True).ids
v2e = build_neighbor_table(spec, L.VERTICES, L.EDGES, as_tensor=True).ids
f64 = dict(dtype=torch.float64, device="cuda")
fl = {n: torch.rand((cnt, w), **f64) for n, cnt, w in (("pd", v, K), ("vn", e, K), ("wn", v, K + 1), ("rho", v, K),
      ("signs", v, 6), ("dual", v, 1), ("flux", e, K), ("fluz", v, K + 1), ("div", v, K), ("out", v, K))}
fl["rho"] += 0.5
p = _lib.ptr; s = _lib.stream_handle()
fn = lambda: _lib.call("tsg_transport_indirect", p(e2v), p(v2e), p(fl["signs"]), p(fl["dual"]), p(fl["pd"]), p(fl["vn"]),
                       p(fl["wn"]), p(fl["rho"]), v, e, K, 0.1, 1.0, 0, p(fl["flux"]), p(fl["fluz"]), p(fl["div"]), p(fl["out"]), s)
fn(); torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(3): fn()
b.record(); torch.cuda.synchronize()
t = a.elapsed_time(b) / 3 / 1e3
nbytes = 8 * (3 * e * K + 7 * v * K + 2 * v * (K + 1) + v * (K - 1)) + 8 * v * K
print(json.dumps(dict(patch=[R, C, K], ms=t * 1e3, frac=nbytes / t / 1e9 / 6455.3)))
