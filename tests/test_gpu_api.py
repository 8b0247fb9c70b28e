"""GPU tests of the drop-in API (Fields, runners, reductions, layouts) against the oracle /
the reference's golden vectors.  Mirrors the reference's own tests:
C3 (fused == naive), C4 (== flat oracle), C6 (renumbering), C8 (conservation), plus edge
cases (2 levels, odd level counts, 2x2 patches, ragged tiles, NaN / signed zero) and
size-independent properties at O1280-class scale.  Floating-point checks are bitwise
(np.array_equal), stricter than the north-star 1e-12 relative tolerance."""

import numpy as np
import pytest

from oracle import tsg_oracle as O

pytestmark = pytest.mark.gpu

T = pytest.importorskip("paper_1908_06094_b200")
L = T.LocationType


def _fill(field, rng, lo, hi):
    spec = field.spec
    h = spec.halo
    arr = field.array("primary", "rw")
    shape = arr[h:h + spec.rows, :, h:h + spec.cols, :, :].shape
    arr[h:h + spec.rows, :, h:h + spec.cols, :, :] = lo + (hi - lo) * rng.random(shape)
    T.halo_update(field)


def _case(spec, seed, geometry="random", layout=None):
    """tests/test_mpdata.py:_setup of the reference, through our Field API."""
    geo = T.build_geometry(spec, geometry, seed=seed, layout=layout)
    state = T.build_state(spec, layout=layout)
    rng = np.random.default_rng(seed)
    T.init_preset(state.pd_in, "random", seed=seed)
    _fill(state.vn, rng, -0.5, 0.5)
    _fill(state.wn, rng, -0.5, 0.5)
    _fill(state.rho, rng, 0.5, 1.5)
    return geo, state


def _oracle(spec, geo, state, params, op="upwind"):
    r, c = spec.rows, spec.cols
    return O.transport_step(O.neighbor_table(r, c, "edges", "vertices"),
                            O.neighbor_table(r, c, "vertices", "edges"), O.edge_signs(r, c),
                            T.field_to_flat(geo.dual_volumes)[:, 0], T.field_to_flat(state.pd_in),
                            T.field_to_flat(state.vn), T.field_to_flat(state.wn),
                            T.field_to_flat(state.rho), params.dt, params.pivbz, op)


@pytest.mark.parametrize("shape,seed", [((4, 4, 3), 0), ((5, 3, 4), 1), ((8, 8, 8), 2), ((2, 2, 2), 3),
                                        ((7, 19, 33), 4), ((3, 41, 2), 5)])
def test_field_api_naive_and_fused_match_oracle(cuda_ok, shape, seed):
    spec = T.PatchSpec(*shape)
    params = T.MpdataParams(dt=0.2, pivbz=0.7)
    geo, state = _case(spec, seed)
    want = _oracle(spec, geo, state, params)
    comp = T.build_mpdata(spec, state, geo, params)
    stats = T.run_naive(comp)
    assert stats.total_updates == spec.rows * spec.cols * (6 * spec.levels + 1)
    assert np.array_equal(T.field_to_flat(state.flux), want["flux"])
    assert np.array_equal(T.field_to_flat(state.fluz), want["fluz"])
    assert np.array_equal(T.field_to_flat(state.divvd), want["div"])
    assert np.array_equal(T.field_to_flat(state.pd_out), want["pd_out"])
    T.run_fused(comp, T.TileSpec(2, 2))
    assert np.array_equal(T.field_to_flat(state.pd_out), want["pd_out"])
    # halo of the output is a periodic image, like after the reference's halo_update
    arr = state.pd_out.array()
    assert np.array_equal(arr[0], arr[spec.rows]) and np.array_equal(arr[:, :, -1], arr[:, :, 1])


@pytest.mark.parametrize("steps", [1, 2, 3, 4])
@pytest.mark.parametrize("fused", [True, False])
def test_time_loop_matches_reference_loop(cuda_ok, steps, fused):
    """run_time_loop == the reference's loop (bench.py:398-403): after it pd_out is the
    final density and pd_in the state before the last step; both fields' halos stay
    periodic images; intermediates (unfused) are the last step's."""
    spec = T.PatchSpec(9, 14, 11)
    params = T.MpdataParams(dt=0.2, pivbz=0.6)
    geo, state = _case(spec, 11)
    comp = T.build_mpdata(spec, state, geo, params)
    r, c = spec.rows, spec.cols
    e2v, v2e = O.neighbor_table(r, c, "edges", "vertices"), O.neighbor_table(r, c, "vertices", "edges")
    dual = T.field_to_flat(geo.dual_volumes)[:, 0]
    pd, vn, wn, rho = (T.field_to_flat(f) for f in (state.pd_in, state.vn, state.wn, state.rho))
    prev = pd
    for _ in range(steps):
        prev, out = pd, O.transport_step(e2v, v2e, O.edge_signs(r, c), dual, pd, vn, wn, rho,
                                         params.dt, params.pivbz)
        pd = out["pd_out"]
    stats = T.run_time_loop(comp, steps, fused=fused)
    assert stats.total_updates == steps * r * c * (6 * spec.levels + 1)
    assert np.array_equal(T.field_to_flat(state.pd_out), pd)
    assert np.array_equal(T.field_to_flat(state.pd_in), prev)
    if not fused:
        assert np.array_equal(T.field_to_flat(state.divvd), out["div"])
    for f in (state.pd_in, state.pd_out):
        arr = f.array()
        assert np.array_equal(arr[0], arr[r]) and np.array_equal(arr[:, :, -1], arr[:, :, 1])
    # the swapped device buffers stay consistent for a following single step
    T.run_fused(comp)
    want = O.transport_step(e2v, v2e, O.edge_signs(r, c), dual, T.field_to_flat(state.pd_in), vn, wn, rho,
                            params.dt, params.pivbz)["pd_out"]
    assert np.array_equal(T.field_to_flat(state.pd_out), want)


def test_level_inner_layout_and_wide_halo(cuda_ok):
    spec = T.PatchSpec(6, 5, 4, halo=2)
    lay = T.LayoutSpec(("extra", "row", "color", "column", "level"), 8)
    params = T.MpdataParams(dt=0.15, pivbz=0.3)
    geo, state = _case(spec, 12, layout=lay)
    want = _oracle(spec, geo, state, params)
    T.run_fused(T.build_mpdata(spec, state, geo, params))
    assert np.array_equal(T.field_to_flat(state.pd_out), want["pd_out"])
    arr = state.pd_out.array()  # halo width 2 filled with periodic images
    assert np.array_equal(arr[:2], arr[6:8]) and np.array_equal(arr[:, :, 7:9], arr[:, :, 2:4])


def test_centred_operator_and_validation(cuda_ok):
    spec = T.PatchSpec(5, 4, 3)
    geo, state = _case(spec, 3)
    params = T.MpdataParams()
    want = _oracle(spec, geo, state, params, "centred")
    comp = T.build_mpdata(spec, state, geo, params, flux_op="centred")
    T.run_fused(comp)
    assert np.array_equal(T.field_to_flat(state.pd_out), want["pd_out"])
    T.run_naive(comp)
    assert np.array_equal(T.field_to_flat(state.flux), want["flux"])
    with pytest.raises(ValueError, match="operator"):
        T.build_mpdata(spec, state, geo, params, flux_op="sideways")
    with pytest.raises(ValueError, match="levels"):
        s1 = T.PatchSpec(4, 4, 1)
        g1, st1 = _case(s1, 0)
        T.build_mpdata(s1, st1, g1, params)
    state.rho.array("primary", "rw")[:] = 0.0
    with pytest.raises(ValueError, match="rho"):
        T.build_mpdata(spec, state, geo, params)


def test_fluz_boundaries_copy_at_unit_pivbz(cuda_ok):
    spec = T.PatchSpec(4, 4, 4)
    geo, state = _case(spec, 6)
    T.run_naive(T.build_mpdata(spec, state, geo, T.MpdataParams(pivbz=1.0)))
    fluz = T.field_to_flat(state.fluz)
    assert np.array_equal(fluz[:, -1], fluz[:, -2]) and np.array_equal(fluz[:, 0], fluz[:, 1])


@pytest.mark.parametrize("seed", range(6))
def test_closed_system_conserves_mass(cuda_ok, seed):
    """Acceptance C8: pivbz = 0, rho = 1 -> mass drift <= 1e-12 (device reduction)."""
    spec = T.PatchSpec(*[(6, 6, 4), (8, 4, 5), (5, 7, 3), (4, 4, 2), (33, 17, 9), (64, 64, 20)][seed])
    geo, state = _case(spec, seed)
    T.init_preset(state.rho, "uniform")
    comp = T.build_mpdata(spec, state, geo, T.MpdataParams(dt=0.05, pivbz=0.0))
    m0 = T.total_mass(state, geo, "pd_in")
    T.run_gpu(comp, download=False)
    m1 = T.total_mass(state, geo, "pd_out")
    assert abs(m1 - m0) <= 1e-12 * abs(m0)
    host = float(np.sum(T.field_to_flat(state.pd_in) * T.field_to_flat(geo.dual_volumes)))
    assert abs(m0 - host) <= 1e-13 * abs(host)


def test_relabelled_flat_paths_are_invariant(cuda_ok, golden):
    """Indirect path under HN/UN numberings, and the structured stepper fed renumbered data."""
    spec = T.PatchSpec(4, 4, 3)
    inp = O.transport_inputs(4, 4, 3, 5, "random", "random", "random")
    base = O.step_inputs(4, 4, inp, 0.1, 0.4)
    pv = T.make_permutation(T.Numbering.HN, spec, L.VERTICES)
    pe = T.make_permutation(T.Numbering.UN, spec, L.EDGES)
    e2v = T.build_neighbor_table(spec, L.EDGES, L.VERTICES, pe, pv).ids
    v2e = T.build_neighbor_table(spec, L.VERTICES, L.EDGES, pv, pe).ids
    assert np.array_equal(e2v, golden["tblp_relabel_4x4_edges_vertices"])
    out = T.transport_step(e2v, v2e, inp["signs"][pv.inverse], inp["dual"][pv.inverse],
                           inp["pd"][pv.inverse], inp["vn"][pe.inverse], inp["wn"][pv.inverse],
                           inp["rho"][pv.inverse], 0.1, 0.4)
    assert np.array_equal(out["pd_out"][pv.forward], base["pd_out"])
    assert np.array_equal(out["flux"][pe.forward], base["flux"])
    st = T.StructuredStepper(spec, perm_v=pv, perm_e=pe)
    st.set_geometry(inp["signs"][pv.inverse], inp["dual"][pv.inverse])
    got = st(inp["pd"][pv.inverse], inp["vn"][pe.inverse], inp["wn"][pv.inverse],
             inp["rho"][pv.inverse], 0.1, 0.4)
    assert np.array_equal(got[pv.forward], base["pd_out"])


def test_table1_kernels_direct_and_indirect(cuda_ok, golden):
    """Acceptance C6: direct structured and SN/UN/HN indirect sweeps agree bitwise."""
    for r, c, lev in ((16, 8, 2), (5, 7, 3)):
        key = f"k_{r}x{c}x{lev}"
        spec = T.PatchSpec(r, c, lev)
        fields = T.make_kernel_fields(spec)
        T.flat_to_field(golden[f"{key}_a"], fields["a"])
        T.flat_to_field(golden[f"{key}_fac"], fields["fac"])
        for scaled, tag in ((False, "k1"), (True, "k2")):
            T.run_naive(T.build_kernel(spec, fields, scaled))
            assert np.array_equal(T.field_to_flat(fields["b"]), golden[f"{key}_{tag}"]), tag
            for num in T.Numbering:
                perm = T.make_permutation(num, spec, L.CELLS)
                table = T.build_neighbor_table(spec, L.CELLS, L.CELLS, perm, perm)
                a = T.field_to_flat(fields["a"], perm)
                got = (T.run_neighbor_sum_scaled(table, a, T.field_to_flat(fields["fac"], perm))
                       if scaled else T.run_neighbor_sum(table, a))
                assert np.array_equal(T.unpermute(got, perm), golden[f"{key}_{tag}"]), (tag, num)


def test_nine_relation_reduce(cuda_ok, golden):
    spec = T.PatchSpec(6, 5, 3)
    for (f, t) in T.OFFSET_TABLES:
        src = T.make_storage(spec, t, "a")
        dst = T.make_storage(spec, f, "b")
        T.flat_to_field(golden[f"red_{f.value}_{t.value}_a"], src)
        T.run_gpu(T.build_reduce(spec, f, t, src, dst))
        assert np.array_equal(T.field_to_flat(dst), golden[f"red_{f.value}_{t.value}_b"]), (f, t)


def test_cell_divergence_and_weights(cuda_ok, golden):
    spec = T.PatchSpec(5, 5, 3)
    geo, state = _case(spec, 7)
    assert np.array_equal(T.field_to_flat(state.vn), golden["cdiv_vn"])
    w = geo.weights.core()[:, :, :, 0, :].reshape(-1, 3)
    assert np.array_equal(w, golden["cdiv_weights"])
    for weighted in (False, True):
        out = T.make_storage(spec, L.CELLS, "div_out")
        T.run_naive(T.build_divergence(spec, state, geo, weighted=weighted, out=out))
        assert np.array_equal(T.field_to_flat(out), golden[f"cdiv_{int(weighted)}"])


@pytest.mark.parametrize("levels", [5, 20])  # element lines / flattened level-pair items
def test_pack_unpack_roundtrip_every_numbering(cuda_ok, levels):
    import torch

    spec = T.PatchSpec(9, 7, levels)
    for loc in L:
        f = T.make_storage(spec, loc, "x")
        n = T.element_count(spec, loc)
        vals = torch.rand((n, levels), dtype=torch.float64, device="cuda")
        for num in T.Numbering:
            if num is T.Numbering.HN and loc is L.EDGES:
                continue
            perm = T.make_permutation(num, spec, loc)
            T.flat_to_field(vals, f, perm)
            assert np.array_equal(T.field_to_flat(f, perm), vals.cpu().numpy()), (loc, num)
            # halo images written by the pack kernel
            dev = f.device().cpu().numpy()
            assert np.array_equal(dev[0, :, 1:-1], dev[spec.rows, :, 1:-1])
            assert np.array_equal(dev[:, :, 0], dev[:, :, spec.cols])


def test_device_halo_update_matches_host(cuda_ok):
    spec = T.PatchSpec(5, 6, 4)
    f = T.make_storage(spec, L.CELLS, "c")
    _fill(f, np.random.default_rng(1), 0, 1)
    dev = f.ensure_device()
    r, c = spec.rows, spec.cols
    dev[0].zero_()
    dev[:, :, -1].zero_()
    dev[r + 1].fill_(7.0)
    T.halo_update(f, "mirror")
    d = dev.cpu().numpy()
    assert np.array_equal(d[0], d[r]) and np.array_equal(d[r + 1], d[1])
    assert np.array_equal(d[:, :, 0], d[:, :, c]) and np.array_equal(d[:, :, c + 1], d[:, :, 1])
    T.sync(f, "primary")
    assert np.array_equal(f.array()[0], f.array()[r])


@pytest.mark.parametrize("shape", [(6, 5, 2), (6, 5, 137), (2, 2, 3), (11, 3, 17), (4, 70, 81),
                                   (5, 9, 63), (7, 6, 64), (3, 17, 65),  # the pitch-16 threshold
                                   (5, 4, 301)])  # a long column: 19 chunks, odd
def test_edge_shapes_fused_unfused_indirect(cuda_ok, shape):
    from tests.gpu_helpers import fused_step, oracle_tables, unfused_step

    r, c, lev = shape
    inp = O.transport_inputs(r, c, lev, 9, "random", "random", "random")
    want = O.step_inputs(r, c, inp, 0.2, 0.8)
    assert np.array_equal(fused_step(r, c, lev, inp, 0.2, 0.8), want["pd_out"])
    got = unfused_step(r, c, lev, inp, 0.2, 0.8)
    for k in want:
        assert np.array_equal(got[k], want[k]), k
    e2v, v2e = oracle_tables(r, c)
    out = T.transport_step(e2v, v2e, inp["signs"], inp["dual"], inp["pd"], inp["vn"], inp["wn"],
                           inp["rho"], 0.2, 0.8)
    for k in want:
        assert np.array_equal(out[k], want[k]), k


def test_nan_and_signed_zero_semantics(cuda_ok):
    """numpy.maximum/minimum semantics: NaN propagates, -0.0 velocities give +0.0 terms."""
    from tests.gpu_helpers import fused_step, unfused_step

    r, c, lev = 6, 7, 5
    inp = O.transport_inputs(r, c, lev, 2, "random", "random", "random")
    inp["vn"][3, 2] = np.nan
    inp["vn"][5, 1] = -np.nan  # sign-bit-set NaN
    inp["vn"][10, 1] = -0.0
    inp["vn"][11, :] = 0.0
    inp["wn"][4, 2] = np.nan
    inp["wn"][5, 3] = -0.0
    inp["pd"][7, :] = -0.0
    want = O.step_inputs(r, c, inp, 0.2, 0.8)
    got = fused_step(r, c, lev, inp, 0.2, 0.8)
    assert np.array_equal(np.isnan(got), np.isnan(want["pd_out"]))
    assert np.array_equal(got, want["pd_out"], equal_nan=True)
    # zero signs must match; a NaN's sign / payload is not part of the contract (the GPU
    # returns the canonical NaN, numpy propagates an input's)
    real = ~np.isnan(want["pd_out"])
    assert np.array_equal(np.signbit(got[real]), np.signbit(want["pd_out"][real]))
    un = unfused_step(r, c, lev, inp, 0.2, 0.8)
    for k in want:
        assert np.array_equal(un[k], want[k], equal_nan=True), k
        real = ~np.isnan(want[k])
        assert np.array_equal(np.signbit(un[k][real]), np.signbit(want[k][real])), k


def test_extreme_dual_volumes(cuda_ok):
    """Tiny, huge, subnormal, zero and negative dual volumes through the fused kernel."""
    from tests.gpu_helpers import fused_step

    r, c, lev = 9, 11, 20
    inp = O.transport_inputs(r, c, lev, 3, "random", "random", "random")
    d = inp["dual"].reshape(-1)
    for v, x in enumerate([1e-300, 1e300, 5e-324, 0.0, -2.5, 2.0 ** -1022, 1.7e308, np.inf, 3.0]):
        d[7 * v + 1] = x
    with np.errstate(all="ignore"):
        want = O.step_inputs(r, c, inp, 0.2, 0.8)["pd_out"]
    got = fused_step(r, c, lev, inp, 0.2, 0.8)
    assert np.array_equal(got, want, equal_nan=True)


def test_default_fused_variant_follows_the_l2_reuse_rule(cuda_ok):
    """Variant 0 keeps the compact 4x16 tile on contiguous ranges when the tile above is still
    in L2 (the bench patch); otherwise (O1280-class) the band schedule, or with it disabled
    the tall 16x4 tile."""
    from paper_1908_06094_b200 import _lib
    from paper_1908_06094_b200.device import DeviceGrid

    lib = _lib.lib()
    bench, big = DeviceGrid(279, 256, 80), DeviceGrid(2560, 2576, 137)
    assert lib.tsg_fused_variant_of(bench.handle, 0, 279) == 21  # 4x16, producer warp
    assert lib.tsg_fused_band_of(bench.handle, 0, 279) == 0
    assert lib.tsg_fused_variant_of(big.handle, 0, 2560) == 21
    assert lib.tsg_fused_band_of(big.handle, 0, 2560) == 1
    _lib.call("tsg_set_fused_band", 0)
    try:
        assert lib.tsg_fused_variant_of(big.handle, 0, 2560) == 19
        assert lib.tsg_fused_band_of(big.handle, 0, 2560) == 0
    finally:
        _lib.call("tsg_set_fused_band", 1)
    _lib.call("tsg_set_fused_variant", 18)
    try:
        assert lib.tsg_fused_variant_of(bench.handle, 0, 279) == 18
    finally:
        _lib.call("tsg_set_fused_variant", 0)
    assert lib.tsg_fused_variant_of(bench.handle, 5, 400) == -1


def test_every_fused_variant_is_bitwise_identical(cuda_ok):
    from paper_1908_06094_b200 import _lib
    from tests.gpu_helpers import fused_step

    r, c, lev = 37, 45, 50
    inp = O.transport_inputs(r, c, lev, 4, "random", "random", "random")
    want = O.step_inputs(r, c, inp, 0.2, 0.8)["pd_out"]
    try:
        v = 1
        while _lib.lib().tsg_fused_variant_info(v, *[None] * 6) == 0:
            _lib.call("tsg_set_fused_variant", v)
            assert np.array_equal(fused_step(r, c, lev, inp, 0.2, 0.8), want), v
            v += 1
    finally:
        _lib.call("tsg_set_fused_variant", 0)


def test_o1280_class_properties(cuda_ok):
    """At a quarter of the O1280 patch (640 x 2576 x 137, 7.4 GB of state): the fused kernel
    equals the independent four-kernel path bitwise, and a closed system conserves mass."""
    import torch

    from paper_1908_06094_b200 import _lib
    from paper_1908_06094_b200.device import DeviceGrid

    rows, cols, K = 640, 2576, 137
    g = DeviceGrid(rows, cols, K)
    s = _lib.stream_handle()
    fields = {}
    for seed, (name, loc, inner, lo, hi) in enumerate((("pd", 0, K, 0.0, 1.0), ("vn", 2, K, -0.5, 0.5),
                                                       ("wn", 0, K + 1, -0.5, 0.5), ("rho", 0, K, 1.0, 1.0))):
        fields[name] = g.empty(loc, inner)
        _lib.call("tsg_fill_hash", g.handle, loc, inner, seed + 1, lo, hi,
                  _lib.ptr(fields[name]), s)
    signs = g.empty(0, 6)
    flat = torch.empty((rows * cols, 6), dtype=torch.float64, device="cuda")
    _lib.call("tsg_edge_signs", rows, cols, _lib.ptr(flat), s)
    _lib.call("tsg_pack", g.handle, 0, 6, _lib.ptr(flat), None, _lib.ptr(signs), s)
    del flat
    dual = g.empty(0, 1)
    _lib.call("tsg_fill_hash", g.handle, 0, 1, 99, 0.5, 1.5, _lib.ptr(dual), s)
    a, b = g.empty(0, K), g.empty(0, K)
    ins = [_lib.ptr(fields[n]) for n in ("pd", "vn", "wn", "rho")] + [_lib.ptr(signs), _lib.ptr(dual)]
    _lib.call("tsg_mpdata_step", g.handle, *ins, _lib.ptr(a), 0.05, 0.0, 0, s)
    flux, fluz, div = g.empty(2, K), g.empty(0, K + 1), g.empty(0, K)
    _lib.call("tsg_mpdata_step_unfused", g.handle, *ins, _lib.ptr(flux), _lib.ptr(fluz), _lib.ptr(div),
              _lib.ptr(b), 0.05, 0.0, 0, s)
    assert torch.equal(a[..., :K], b[..., :K])  # the level padding is not field content
    work = torch.empty(1026, dtype=torch.float64, device="cuda")
    _lib.call("tsg_total_mass", g.handle, _lib.ptr(fields["pd"]), _lib.ptr(dual), _lib.ptr(work[:1024]),
              _lib.ptr(work[1024:1025]), s)
    _lib.call("tsg_total_mass", g.handle, _lib.ptr(a), _lib.ptr(dual), _lib.ptr(work[:1024]),
              _lib.ptr(work[1025:]), s)
    m0, m1 = work[1024].item(), work[1025].item()
    assert abs(m1 - m0) <= 1e-12 * abs(m0)


def test_fill_hash_is_decomposition_invariant(cuda_ok):
    from paper_1908_06094_b200 import _lib
    from paper_1908_06094_b200.device import PERIODIC_COLS, DeviceGrid

    s = _lib.stream_handle()
    full = DeviceGrid(12, 9, 5)
    f = full.empty(2, 5)
    _lib.call("tsg_fill_hash", full.handle, 2, 5, 7, -1.0, 1.0, _lib.ptr(f), s)
    for r0, nr in ((0, 4), (4, 5), (9, 3)):
        strip = DeviceGrid(nr, 9, 5, flags=PERIODIC_COLS, row0=r0, global_rows=12)
        t = strip.empty(2, 5)
        _lib.call("tsg_fill_hash", strip.handle, 2, 5, 7, -1.0, 1.0, _lib.ptr(t), s)
        assert np.array_equal(t[1:nr + 1].cpu().numpy(), f[r0 + 1:r0 + nr + 1].cpu().numpy())


def test_pipelined_host_fed_steps_match_oracle(cuda_ok):
    """StructuredStepper.run_pipelined (the e2e path of bench.py): three different host input
    sets streamed with overlapped H2D / compute / D2H give the oracle's results bitwise."""
    import torch

    r, c, lev = 23, 31, 12
    spec = T.PatchSpec(r, c, lev)
    st = T.StructuredStepper(spec)
    sets, want = [], []
    for seed in range(3):
        inp = O.transport_inputs(r, c, lev, seed, "random", "random", "random")
        if seed == 0:
            st.set_geometry(inp["signs"], inp["dual"])
            geo = inp
        else:
            inp.update(signs=geo["signs"], dual=geo["dual"])
        sets.append([torch.from_numpy(inp[n]).pin_memory() for n in ("pd", "vn", "wn", "rho")])
        want.append(O.step_inputs(r, c, inp, 0.2, 0.8)["pd_out"])
    outs = [torch.empty((r * c, lev), dtype=torch.float64).pin_memory() for _ in range(3)]
    st.run_pipelined(sets, outs, 0.2, 0.8)
    torch.cuda.synchronize()
    for o, w in zip(outs, want):
        assert np.array_equal(o.numpy(), w)


def test_pipelined_time_loop_keeps_resident_velocities(cuda_ok):
    """run_pipelined with (pd, None, None, None): only the state crosses PCIe (bench e2e);
    vn / wn / rho keep the values of the last full upload -- the reference's time loop
    (bench.py:398-403) fed from the host, bitwise against the oracle loop."""
    import torch

    r, c, lev = 19, 24, 20
    st = T.StructuredStepper(T.PatchSpec(r, c, lev))
    inp = O.transport_inputs(r, c, lev, 3, "random", "random", "random")
    st.set_geometry(inp["signs"], inp["dual"])
    full = [torch.from_numpy(inp[n]).pin_memory() for n in ("pd", "vn", "wn", "rho")]
    other = O.transport_inputs(r, c, lev, 4, "random", "random", "random")
    pds = [torch.from_numpy(other["pd"]).pin_memory(), torch.from_numpy(inp["pd"] * 0.5).pin_memory()]
    outs = [torch.empty((r * c, lev), dtype=torch.float64).pin_memory() for _ in range(3)]
    st.run_pipelined([full, [pds[0], None, None, None], [pds[1], None, None, None]], outs, 0.2, 0.8)
    torch.cuda.synchronize()
    for o, pd in zip(outs, (inp["pd"], other["pd"], inp["pd"] * 0.5)):
        want = O.step_inputs(r, c, dict(inp, pd=pd), 0.2, 0.8)["pd_out"]
        assert np.array_equal(o.numpy(), want)


def test_dump_tables_and_csv_loading(cuda_ok):
    import io

    spec = T.PatchSpec(3, 4, 2)
    buf = io.StringIO()
    T.dump_tables(spec, buf)
    rows = buf.getvalue().strip().splitlines()
    assert rows[0] == "from_loc,to_loc,element,slot,neighbor"
    got = {}
    for ln in rows[1:]:
        f, t, e, s, nb = ln.split(",")
        got.setdefault((f, t), {})[(int(e), int(s))] = int(nb)
    for (f, t) in O.OFFSETS:
        want = O.neighbor_table(3, 4, f, t)
        assert all(got[(f, t)][(e, s)] == want[e, s] for e in range(want.shape[0]) for s in range(want.shape[1]))
    field = T.make_storage(spec, L.EDGES, "vn")
    T.load_field_csv(field, io.StringIO("element,level,value\n# comment\n0,0,1.5\n35,1,-2.25\n"))
    flat = T.field_to_flat(field)
    assert flat[0, 0] == 1.5 and flat[35, 1] == -2.25 and np.count_nonzero(flat) == 2
    with pytest.raises(ValueError, match="out of range"):
        T.load_field_csv(field, io.StringIO("36,0,1.0\n"))


def test_time_computation_and_runstats(cuda_ok):
    spec = T.PatchSpec(16, 12, 6)
    geo, state = _case(spec, 4)
    comp = T.build_mpdata(spec, state, geo, T.MpdataParams())
    res = T.time_computation(comp, lambda c: T.run_gpu(c, download=False), reps=3)
    assert res.updates == spec.rows * spec.cols * (6 * spec.levels + 1)
    assert len(res.times) == 3 and res.median_seconds > 0
    stats = T.run_gpu(comp)
    assert stats.wall_times["ms0"] > 0 and stats.bytes_moved > 0
    assert stats.traffic().total_distinct() > 0
    with pytest.raises(ValueError):
        T.time_computation(comp, T.run_fused, reps=0)


def test_runners_report_the_reference_traffic(cuda_ok):
    """run_naive / run_fused(TileSpec) on the device give the reference's RunStats:
    stage updates (apron recompute included) and traffic() rows, vs reference goldens."""
    import json
    from pathlib import Path

    gold = json.loads((Path(__file__).parent / "golden" / "traffic.json").read_text())["cases"]
    spec = T.PatchSpec(6, 8, 4)
    for case in [c for c in gold if c["kind"] == "mpdata" and c["patch"] == [6, 8, 4]]:
        geo, state = _case(spec, 1)
        comp = T.build_mpdata(spec, state, geo, T.MpdataParams())
        tiles = case["tiles"]
        stats = T.run_naive(comp) if tiles is None else T.run_fused(comp, T.TileSpec(*tiles))
        assert stats.stage_updates == case["stage_updates"]
        rows = [[r.field, r.stage, r.distinct_reads, r.distinct_writes, r.raw_reads, r.raw_writes]
                for r in stats.traffic().rows]
        assert rows == case["rows"], tiles


def test_device_resident_results_follow_the_staleness_contract(cuda_ok):
    spec = T.PatchSpec(6, 7, 5)
    geo, state = _case(spec, 2)
    comp = T.build_mpdata(spec, state, geo, T.MpdataParams(dt=0.2, pivbz=0.8))
    want = _oracle(spec, geo, state, T.MpdataParams(dt=0.2, pivbz=0.8))
    T.run_gpu(comp, download=False)
    with pytest.raises(T.StalenessError):
        state.pd_out.array("primary")
    assert np.array_equal(T.field_to_flat(state.pd_out), want["pd_out"])  # unpacked on device
    T.sync(state.pd_out, "primary")
    assert np.array_equal(T.field_to_flat(state.pd_out), want["pd_out"])


@pytest.mark.parametrize("shape", [(13, 21, 20), (6, 37, 33), (9, 10, 2)])
def test_indirect_reduce_every_width(cuda_ok, shape):
    """The table-driven gather (flattened level-pair items for even level counts, one warp
    per row otherwise) for the nine relations' widths 2 / 3 / 4 / 6, plain and scaled, in a
    Hilbert / colour-interleaved numbering, against the oracle bitwise."""
    r, c, lev = shape
    spec = T.PatchSpec(r, c, lev)
    rng = np.random.default_rng(lev + 1)
    for (f, t) in T.OFFSET_TABLES:
        pf = T.make_permutation(T.Numbering.UN, spec, f)
        pt = T.make_permutation(T.Numbering.UN, spec, t)
        table = T.build_neighbor_table(spec, f, t, pf, pt)
        a = rng.random((T.element_count(spec, t), lev))
        fac = 0.5 + rng.random((T.element_count(spec, f), 1))
        a_perm = a[pt.inverse]
        want = O.neighbor_sum(table.ids, a_perm)
        assert np.array_equal(T.run_neighbor_sum(table, a_perm), want), (f, t)
        want_s = O.neighbor_sum_scaled(table.ids, a_perm, fac)
        assert np.array_equal(T.run_neighbor_sum_scaled(table, a_perm, fac), want_s), (f, t)


@pytest.mark.parametrize("shape", [(13, 21, 20), (6, 37, 33)])
def test_tma_reduce_and_cell_divergence_paths(cuda_ok, shape):
    """Long level runs take the TMA-staged kernels (reduce_tma.cu): all nine relations,
    the scaled Table-1 kernel and both cell divergences against the oracle, bitwise."""
    r, c, lev = shape
    spec = T.PatchSpec(r, c, lev)
    rng = np.random.default_rng(lev)
    for (f, t) in T.OFFSET_TABLES:
        src = T.make_storage(spec, t, "a")
        dst = T.make_storage(spec, f, "b")
        a = rng.random((T.element_count(spec, t), lev))
        T.flat_to_field(a, src)
        T.run_gpu(T.build_reduce(spec, f, t, src, dst))
        want = O.neighbor_sum(O.neighbor_table(r, c, f.value, t.value), a)
        assert np.array_equal(T.field_to_flat(dst), want), (f, t)
    fields = T.make_kernel_fields(spec)
    a = rng.random((2 * r * c, lev))
    fac = 0.5 + rng.random((2 * r * c, 1))
    T.flat_to_field(a, fields["a"])
    T.flat_to_field(fac, fields["fac"])
    T.run_gpu(T.build_kernel(spec, fields, True))
    want = O.neighbor_sum_scaled(O.neighbor_table(r, c, "cells", "cells"), a, fac)
    assert np.array_equal(T.field_to_flat(fields["b"]), want)
    geo, state = _case(spec, 3)
    c2e = O.neighbor_table(r, c, "cells", "edges")
    vn = T.field_to_flat(state.vn)
    length = T.field_to_flat(geo.edge_length)[:, 0]
    area = T.field_to_flat(geo.cell_area)[:, 0]
    weights = geo.weights.core()[:, :, :, 0, :].reshape(-1, 3)
    for weighted, want in ((False, O.cell_divergence(c2e, vn, length, area)),
                           (True, O.weighted_divergence(c2e, vn, weights))):
        out = T.make_storage(spec, L.CELLS, "div_out")
        T.run_gpu(T.build_divergence(spec, state, geo, weighted=weighted, out=out))
        assert np.array_equal(T.field_to_flat(out), want), weighted


def test_tma_reduce_dynamic_deal_matches_oracle(cuda_ok):
    """A patch with >= 24 units per resident CTA takes the dynamically dealt reduce
    (reduce_tma.cu kRedDynUnits): all nine relations, the scaled Table-1 kernel and the
    cell divergence against the oracle, bitwise; twice, so the ticket reset is exercised."""
    r, c, lev = 512, 512, 33
    spec = T.PatchSpec(r, c, lev)
    rng = np.random.default_rng(5)
    for (f, t) in T.OFFSET_TABLES:
        src = T.make_storage(spec, t, "a")
        dst = T.make_storage(spec, f, "b")
        a = rng.random((T.element_count(spec, t), lev))
        T.flat_to_field(a, src)
        want = O.neighbor_sum(O.neighbor_table(r, c, f.value, t.value), a)
        for _ in range(2):
            T.run_gpu(T.build_reduce(spec, f, t, src, dst))
            assert np.array_equal(T.field_to_flat(dst), want), (f, t)
    fields = T.make_kernel_fields(spec)
    a = rng.random((2 * r * c, lev))
    fac = 0.5 + rng.random((2 * r * c, 1))
    T.flat_to_field(a, fields["a"])
    T.flat_to_field(fac, fields["fac"])
    T.run_gpu(T.build_kernel(spec, fields, True))
    want = O.neighbor_sum_scaled(O.neighbor_table(r, c, "cells", "cells"), a, fac)
    assert np.array_equal(T.field_to_flat(fields["b"]), want)
    _check_cell_divergence(spec, repeats=2)


def _check_cell_divergence(spec, repeats=1, variants=(0,)):
    """Both cell divergences (simple: a division per output; weighted) against the oracle,
    bitwise, under each tsg_set_reduce_variant tile shape."""
    from paper_1908_06094_b200 import _lib

    r, c = spec.rows, spec.cols
    geo, state = _case(spec, 3)
    c2e = O.neighbor_table(r, c, "cells", "edges")
    vn = T.field_to_flat(state.vn)
    length = T.field_to_flat(geo.edge_length)[:, 0]
    area = T.field_to_flat(geo.cell_area)[:, 0]
    weights = geo.weights.core()[:, :, :, 0, :].reshape(-1, 3)
    try:
        for v in variants:
            _lib.call("tsg_set_reduce_variant", v)
            for weighted, want in ((False, O.cell_divergence(c2e, vn, length, area)),
                                   (True, O.weighted_divergence(c2e, vn, weights))):
                out = T.make_storage(spec, L.CELLS, "div_out")
                for _ in range(repeats):
                    T.run_gpu(T.build_divergence(spec, state, geo, weighted=weighted, out=out))
                    assert np.array_equal(T.field_to_flat(out), want), (weighted, v)
    finally:
        _lib.call("tsg_set_reduce_variant", 0)


def test_cell_divergence_every_tile_shape(cuda_ok):
    """The cell divergence's benchmarking tile shapes (static 1-9, dealt 11-19) on a ragged
    patch with an odd level count, and its default dealt 8 x 16 tile on a large patch."""
    _check_cell_divergence(T.PatchSpec(37, 70, 35), variants=list(range(0, 10)) + list(range(11, 20)))
    _check_cell_divergence(T.PatchSpec(300, 1030, 21))


def test_tma_reduce_every_tile_shape(cuda_ok):
    """Every benchmarking shape of the TMA reduce (tsg_set_reduce_variant: static 1-9,
    dynamically dealt 11-19) is bitwise equal to the oracle on a ragged patch with an odd
    level count."""
    from paper_1908_06094_b200 import _lib

    r, c, lev = 37, 70, 35
    spec = T.PatchSpec(r, c, lev)
    rng = np.random.default_rng(11)
    try:
        for (f, t) in T.OFFSET_TABLES:
            src = T.make_storage(spec, t, "a")
            dst = T.make_storage(spec, f, "b")
            a = rng.random((T.element_count(spec, t), lev))
            T.flat_to_field(a, src)
            want = O.neighbor_sum(O.neighbor_table(r, c, f.value, t.value), a)
            for v in list(range(0, 10)) + list(range(11, 20)):
                _lib.call("tsg_set_reduce_variant", v)
                T.run_gpu(T.build_reduce(spec, f, t, src, dst))
                assert np.array_equal(T.field_to_flat(dst), want), (f, t, v)
    finally:
        _lib.call("tsg_set_reduce_variant", 0)


@pytest.mark.parametrize("shape,halo,order", [
    ((24, 20, 7), 1, None),                                            # level planes outermost
    ((37, 45, 50), 1, None),
    ((30, 17, 6), 2, ("extra", "row", "color", "column", "level")),    # rows outermost, halo 2
    ((48, 9, 5), 1, ("level", "extra", "row", "column", "color")),
])
def test_streamed_host_step_in_the_reference_loop(cuda_ok, shape, halo, order):
    """The reference's dependent loop (bench.py:398-403: ``_copy_core(pd_out, pd_in)`` on
    the host, then ``run_fused``): from the second step only pd_in is host-dirty, so
    run_fused streams it through the step band by band (executors._run_streamed).  Three
    steps equal three oracle steps bitwise, the host halo of pd_out holds periodic
    images, and every field is clean afterwards."""
    from paper_1908_06094_b200 import executors as X

    spec = T.PatchSpec(*shape, halo=halo)
    lay = T.LayoutSpec(order) if order else None
    params = T.MpdataParams(dt=0.15, pivbz=0.6)
    geo, state = _case(spec, 21, layout=lay)
    comp = T.build_mpdata(spec, state, geo, params)
    r, c, h = spec.rows, spec.cols, spec.halo
    args = list(_oracle_args(spec, geo, state))
    streamed = 0
    for step in range(3):
        if step:
            values = state.pd_out.array("primary", "r")[h:h + r, :, h:h + c, :, :]
            state.pd_in.array("primary", "rw")[h:h + r, :, h:h + c, :, :] = values
            T.halo_update(state.pd_in)
            streamed += X._streamable(comp, True, True)
        T.run_fused(comp, T.TileSpec(r, c))
        args[4] = O.transport_step(*args, params.dt, params.pivbz)["pd_out"]
        assert np.array_equal(T.field_to_flat(state.pd_out), args[4]), step
    assert streamed == 2
    arr = state.pd_out.array()
    assert np.array_equal(arr[:h], arr[r:r + h]) and np.array_equal(arr[:, :, :h], arr[:, :, c:c + h])
    assert not any(state.pd_in.dirty.values()) and not any(state.pd_out.dirty.values())


def _oracle_args(spec, geo, state):
    r, c = spec.rows, spec.cols
    return (O.neighbor_table(r, c, "edges", "vertices"), O.neighbor_table(r, c, "vertices", "edges"),
            O.edge_signs(r, c), T.field_to_flat(geo.dual_volumes)[:, 0], T.field_to_flat(state.pd_in),
            T.field_to_flat(state.vn), T.field_to_flat(state.wn), T.field_to_flat(state.rho))


def test_dealt_reduce_many_launches_stay_exact(cuda_ok):
    """The dealt reduce's ticket words reset themselves at the end of every launch: 200
    back-to-back launches on one handle (no host sync in between) each give the same
    bitwise result -- a count leaking into the next launch would skip work."""
    import torch

    from paper_1908_06094_b200 import _lib
    from paper_1908_06094_b200.device import DeviceGrid

    g = DeviceGrid(512, 512, 33)
    s = _lib.stream_handle()
    src, ref, dst = g.empty(0, 33), g.empty(0, 33), g.empty(0, 33)
    _lib.call("tsg_fill_hash", g.handle, 0, 33, 3, 0.0, 1.0, _lib.ptr(src), s)
    _lib.call("tsg_neighbor_reduce", g.handle, 0, 0, 33, _lib.ptr(src), None, _lib.ptr(ref), s)
    bad = torch.zeros((), dtype=torch.int64, device="cuda")
    for _ in range(200):
        dst.zero_()
        _lib.call("tsg_neighbor_reduce", g.handle, 0, 0, 33, _lib.ptr(src), None, _lib.ptr(dst), s)
        bad += (dst != ref).any()
    assert int(bad) == 0


def test_point_bands_match_one_launch(cuda_ok):
    """Fields with more points than one 32-bit-indexed launch covers are split into row
    bands (tsg_common.cuh for_point_bands; ~10 M vertices x 137 levels for an edge field).
    With the limit lowered to a few rows (tsg_set_point_limit), the reorders (pairs and
    point forms), the synthetic fill and the unfused step give the one-launch result,
    bitwise."""
    import torch
    from paper_1908_06094_b200 import _lib
    from paper_1908_06094_b200.device import DeviceGrid

    r, c, k = 23, 37, 20
    g = DeviceGrid(r, c, k)
    s = _lib.stream_handle()
    rng = np.random.default_rng(0)
    cases = [(L.EDGES.code, k), (L.CELLS.code, 7), (L.VERTICES.code, 1)]
    flats = {(loc, inner): torch.from_numpy(rng.random((r * c * (3 if loc == 2 else 2 if loc == 1 else 1), inner)))
             .cuda() for loc, inner in cases}
    perm = {loc: torch.from_numpy(rng.permutation(len(f))).cuda() for (loc, _), f in flats.items()}

    def run():
        out = {}
        for (loc, inner), flat in flats.items():
            f = g.empty(loc, inner)
            _lib.call("tsg_pack", g.handle, loc, inner, _lib.ptr(flat), _lib.ptr(perm[loc]), _lib.ptr(f), s)
            back = torch.empty_like(flat)
            _lib.call("tsg_unpack", g.handle, loc, inner, _lib.ptr(f), _lib.ptr(perm[loc]), _lib.ptr(back), s)
            h = g.empty(loc, inner)
            _lib.call("tsg_fill_hash", g.handle, loc, inner, 9, -1.0, 1.0, _lib.ptr(h), s)
            out[loc, inner] = (f.clone(), back, h)
        ins = {n: g.empty(loc, inner) for n, loc, inner in (("pd", 0, k), ("vn", 2, k), ("wn", 0, k + 1),
                                                            ("rho", 0, k), ("signs", 0, 6), ("dual", 0, 1))}
        inners = {"pd": k, "vn": k, "wn": k + 1, "rho": k, "signs": 6, "dual": 1}
        for i, (n, t) in enumerate(ins.items()):
            _lib.call("tsg_fill_hash", g.handle, 2 if n == "vn" else 0, inners[n], i,
                      0.5 if n in ("rho", "dual") else -0.5, 1.5, _lib.ptr(t), s)
        flux, fluz, div, pd_out = g.empty(2, k), g.empty(0, k + 1), g.empty(0, k), g.empty(0, k)
        _lib.call("tsg_mpdata_step_unfused", g.handle, *[_lib.ptr(ins[n]) for n in ("pd", "vn", "wn", "rho",
                                                                                    "signs", "dual")],
                  _lib.ptr(flux), _lib.ptr(fluz), _lib.ptr(div), _lib.ptr(pd_out), 0.1, 0.7, 0, s)
        out["step"] = (flux, fluz, div, pd_out)
        torch.cuda.synchronize()
        return out

    want = run()
    for k_i, f in flats.items():
        assert torch.equal(want[k_i][1], f)  # pack -> unpack round trip
    try:
        for limit in (c * 7, c * 3 * 10 + 1, 1):  # a few rows per band, ragged bands, one row per band
            _lib.call("tsg_set_point_limit", limit)
            got = run()
            for key in want:
                for a, b in zip(want[key], got[key]):
                    assert torch.equal(a, b), (limit, key)
    finally:
        _lib.call("tsg_set_point_limit", 0)
