"""Table-1 indirect gather (k1, SN numbering) at 1024x1024x80 a few times (ncu target)."""
import sys
sys.path.insert(0, "/root/repo")
import torch
from paper_1908_06094_b200 import LocationType as L, Numbering, PatchSpec, _lib, build_neighbor_table, make_permutation
rows, cols, K = (int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1024x1024x80").split("x"))
spec = PatchSpec(rows, cols, K)
n = 2 * rows * cols
perm = make_permutation(Numbering.SN, spec, L.CELLS)
table = build_neighbor_table(spec, L.CELLS, L.CELLS, perm, perm, as_tensor=True).ids
a = torch.rand((n, K), dtype=torch.float64, device="cuda")
b = torch.empty_like(a)
flush = torch.ones(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
for _ in range(4):
    flush.sum()
    _lib.call("tsg_neighbor_reduce_indirect", _lib.ptr(table), n, 3, K, _lib.ptr(a), None, _lib.ptr(b), _lib.stream_handle())
torch.cuda.synchronize()
