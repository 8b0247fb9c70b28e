"""ncu targets for the secondary kernels: python tools/prof_secondary.py {reduce_cc|reduce_vv|indirect|pack|unfused|celldiv_simple|celldiv_weighted}."""
import sys
sys.path.insert(0, "/root/repo")
import torch
from paper_1908_06094_b200 import LocationType as L, Numbering, PatchSpec, _lib, build_neighbor_table, make_permutation
from paper_1908_06094_b200.device import DeviceGrid

what = sys.argv[1]
s = _lib.stream_handle()
flush = torch.ones(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
if what.startswith("reduce_"):
    loc = {"cc": 1, "vv": 0}[what[-2:]]
    g = DeviceGrid(1024, 1024, 80) if loc == 1 else DeviceGrid(256, 256, 80)
    src, dst = g.empty(loc, 80), g.empty(loc, 80)
    _lib.call("tsg_fill_hash", g.handle, loc, 80, 3, 0.0, 1.0, _lib.ptr(src), s)
    fn = lambda: _lib.call("tsg_neighbor_reduce", g.handle, loc, loc, 80, _lib.ptr(src), None, _lib.ptr(dst), s)
elif what == "indirect":
    spec = PatchSpec(1024, 1024, 80)
    n = 2 * 1024 * 1024
    perm = make_permutation(Numbering.SN, spec, L.CELLS)
    table = build_neighbor_table(spec, L.CELLS, L.CELLS, perm, perm, as_tensor=True).ids
    a = torch.rand((n, 80), dtype=torch.float64, device="cuda")
    b = torch.empty_like(a)
    fn = lambda: _lib.call("tsg_neighbor_reduce_indirect", _lib.ptr(table), n, 3, 80, _lib.ptr(a), None, _lib.ptr(b), s)
elif what == "pack":
    g = DeviceGrid(1024, 1024, 80)
    n = 2 * 1024 * 1024
    a = torch.rand((n, 80), dtype=torch.float64, device="cuda")
    f = g.empty(1, 80)
    fn = lambda: _lib.call("tsg_pack", g.handle, 1, 80, _lib.ptr(a), None, _lib.ptr(f), s)
elif what.startswith("celldiv_"):
    g = DeviceGrid(1024, 1024, 80)
    vn, length, area, w, out = g.empty(2, 80), g.empty(2, 1), g.empty(1, 1), g.empty(1, 3), g.empty(1, 80)
    for f, loc, inner, lo in ((vn, 2, 80, -0.5), (length, 2, 1, 0.5), (area, 1, 1, 0.5)):
        _lib.call("tsg_fill_hash", g.handle, loc, inner, 4, lo, lo + 1.0, _lib.ptr(f), s)
    _lib.call("tsg_cell_weights", g.handle, _lib.ptr(length), _lib.ptr(area), _lib.ptr(w), s)
    weighted = int(what.endswith("weighted"))
    fn = lambda: _lib.call("tsg_cell_divergence", g.handle, weighted, _lib.ptr(vn), _lib.ptr(length), _lib.ptr(area),
                           _lib.ptr(w), _lib.ptr(out), s)
elif what == "unfused":
    from paper_1908_06094_b200 import StructuredStepper
    from paper_1908_06094_b200.workloads import transport_inputs
    inp = transport_inputs(279, 256, 80)
    st = StructuredStepper(PatchSpec(279, 256, 80))
    st.set_geometry(inp["signs"], inp["dual"])
    st.upload(inp["pd"], inp["vn"], inp["wn"], inp["rho"])
    fn = lambda: st.step_unfused(0.1, 1.0)
for _ in range(4):
    flush.sum()
    fn()
torch.cuda.synchronize()
