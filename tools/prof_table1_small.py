"""ncu target: the Table-1 kernels at the paper's own 128x128x80 patch (k1 / k2 direct,
SN indirect, the SN pack / unpack), 5 launches each after a 256 MiB L2 flush.  The ncu
launch list gives their kernel-only durations beside bench_stencils.py's event times."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1908_06094_b200 import (LocationType as L, Numbering, PatchSpec, _lib,  # noqa: E402
                                   build_neighbor_table, element_count, make_permutation)
from paper_1908_06094_b200.device import DeviceGrid  # noqa: E402

R = C = 128
K = 80
s = _lib.stream_handle()
flush = torch.ones(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
spec = PatchSpec(R, C, K)
g = DeviceGrid(R, C, K)
n = element_count(spec, L.CELLS)
a, fac, b = g.empty(1, K), g.empty(1, 1), g.empty(1, K)
_lib.call("tsg_fill_hash", g.handle, 1, K, 1, 0.0, 1.0, _lib.ptr(a), s)
_lib.call("tsg_fill_hash", g.handle, 1, 1, 2, 0.5, 1.5, _lib.ptr(fac), s)
perm = make_permutation(Numbering.SN, spec, L.CELLS)
fwd = torch.as_tensor(perm.forward, device="cuda")
table = build_neighbor_table(spec, L.CELLS, L.CELLS, perm, perm, as_tensor=True).ids
flat_a = torch.empty((n, K), dtype=torch.float64, device="cuda")
flat_b = torch.empty_like(flat_a)
_lib.call("tsg_unpack", g.handle, 1, K, _lib.ptr(a), _lib.ptr(fwd), _lib.ptr(flat_a), s)
ops = [
    lambda: _lib.call("tsg_neighbor_reduce", g.handle, 1, 1, K, _lib.ptr(a), None, _lib.ptr(b), s),
    lambda: _lib.call("tsg_neighbor_reduce", g.handle, 1, 1, K, _lib.ptr(a), _lib.ptr(fac), _lib.ptr(b), s),
    lambda: _lib.call("tsg_neighbor_reduce_indirect", _lib.ptr(table), n, 3, K, _lib.ptr(flat_a), None,
                      _lib.ptr(flat_b), s),
    lambda: _lib.call("tsg_pack", g.handle, 1, K, _lib.ptr(flat_a), _lib.ptr(fwd), _lib.ptr(b), s),
    lambda: _lib.call("tsg_unpack", g.handle, 1, K, _lib.ptr(b), _lib.ptr(fwd), _lib.ptr(flat_a), s),
]
for op in ops:
    for _ in range(5):
        flush.sum()
        op()
torch.cuda.synchronize()
