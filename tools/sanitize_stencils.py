"""Runs of the round-2 stencil changes for compute-sanitizer (memcheck / racecheck):
the unfused step's item kernels on a resident grid (short sweep) and on a one-pass grid
with block-contiguous items (long sweep), each bitwise against the fused step, and the
cell divergence under its default and dealt tile shapes against the oracle.
    compute-sanitizer --tool memcheck python tools/sanitize_stencils.py"""
import sys

sys.path.insert(0, "/root/repo")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import tsg_oracle as O  # noqa: E402
import paper_1908_06094_b200 as T  # noqa: E402
from paper_1908_06094_b200 import _lib  # noqa: E402
from paper_1908_06094_b200.distributed import StripStepper  # noqa: E402

s = _lib.stream_handle()
n = 0
for R, C, K in ((64, 72, 40), (1024, 1024, 40)):  # 4 vs ~28 resident passes: both grid forms
    st = StripStepper(R, C, K, 0, 1, seed=2)
    g = st.grid
    flux, fluz, div, out = g.empty(2, K), g.empty(0, K + 1), g.empty(0, K), g.empty(0, K)
    ins = [_lib.ptr(t) for t in (st.pd, st.vn, st.wn, st.rho, st.signs, st.dual)]
    _lib.call("tsg_mpdata_step_unfused", g.handle, *ins, _lib.ptr(flux), _lib.ptr(fluz), _lib.ptr(div),
              _lib.ptr(out), 0.1, 1.0, 0, s)
    _lib.call("tsg_mpdata_step", g.handle, *ins, _lib.ptr(st.pd_out), 0.1, 1.0, 0, s)
    torch.cuda.synchronize()
    assert torch.equal(out, st.pd_out), (R, C, K)
    n += 2

r, c, k = 21, 40, 35
spec = T.PatchSpec(r, c, k)
geo = T.build_geometry(spec, "random", seed=3)
state = T.build_state(spec)
rng = np.random.default_rng(3)
vn_flat = rng.random((T.element_count(spec, T.LocationType.EDGES), k)) - 0.5
T.flat_to_field(vn_flat, state.vn)
c2e = O.neighbor_table(r, c, "cells", "edges")
length = T.field_to_flat(geo.edge_length)[:, 0]
area = T.field_to_flat(geo.cell_area)[:, 0]
weights = geo.weights.core()[:, :, :, 0, :].reshape(-1, 3)
for v in (0, 2, 12, 17):
    _lib.call("tsg_set_reduce_variant", v)
    for weighted, want in ((False, O.cell_divergence(c2e, vn_flat, length, area)),
                           (True, O.weighted_divergence(c2e, vn_flat, weights))):
        res = T.make_storage(spec, T.LocationType.CELLS, "div_out")
        T.run_gpu(T.build_divergence(spec, state, geo, weighted=weighted, out=res))
        assert np.array_equal(T.field_to_flat(res), want), (v, weighted)
        n += 1
_lib.call("tsg_set_reduce_variant", 0)
torch.cuda.synchronize()
print(f"sanitize_stencils: {n} launches bitwise")
