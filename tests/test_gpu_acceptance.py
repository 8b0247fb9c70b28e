"""The reference's acceptance checks C3 / C4 / C8 (tests/test_acceptance.py:128-186, :276-288
of the reference) run through the drop-in API on the GPU, with the same seeds, shapes,
parameters and tile specs; the flat oracle is the pinned restatement (oracle/), and the
GPU flat-stage API (``paper_1908_06094_b200.reference``) is checked as a third arm."""

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


def _transport_case(spec, seed, uniform_rho=False):
    geo = T.build_geometry(spec, "random", seed=seed)
    state = T.build_state(spec)
    rng = np.random.default_rng(seed)
    T.init_preset(state.pd_in, "random", seed=seed)
    _fill(state.vn, rng, -0.5, 0.5)
    _fill(state.wn, rng, -0.5, 0.5)
    if uniform_rho:
        T.init_preset(state.rho, "uniform")
    else:
        _fill(state.rho, rng, 0.5, 1.5)
    return geo, state


def _flat_args(spec, geo, state):
    r, c = spec.rows, spec.cols
    return (O.neighbor_table(r, c, "edges", "vertices"), O.neighbor_table(r, c, "vertices", "edges"),
            O.edge_signs(r, c), T.field_to_flat(geo.dual_volumes)[:, 0], T.field_to_flat(state.pd_in),
            T.field_to_flat(state.vn), T.field_to_flat(state.wn), T.field_to_flat(state.rho))


def test_c03_executor_equivalence_bitwise(cuda_ok):
    """100 seeds x (transport, k1, k2) at 4x4x4 plus one 128x128x8: fused == naive."""
    failures = 0
    spec = T.PatchSpec(4, 4, 4)
    for seed in range(100):
        geo_n, state_n = _transport_case(spec, seed)
        geo_f, state_f = _transport_case(spec, seed)
        params = T.MpdataParams(dt=0.1, pivbz=0.6)
        T.run_naive(T.build_mpdata(spec, state_n, geo_n, params))
        T.run_fused(T.build_mpdata(spec, state_f, geo_f, params), T.TileSpec(2, 2))
        failures += not np.array_equal(T.field_to_flat(state_n.pd_out), T.field_to_flat(state_f.pd_out))
        rng = np.random.default_rng(seed)
        for scaled in (False, True):
            fn = T.make_kernel_fields(spec)
            _fill(fn["a"], rng, 0.0, 1.0)
            _fill(fn["fac"], rng, 0.5, 1.5)
            ff = T.make_kernel_fields(spec)
            ff["a"].array("primary", "rw")[...] = fn["a"].array()
            ff["fac"].array("primary", "rw")[...] = fn["fac"].array()
            T.run_naive(T.build_kernel(spec, fn, scaled))
            T.run_fused(T.build_kernel(spec, ff, scaled), T.TileSpec(2, 2))
            failures += not np.array_equal(T.field_to_flat(fn["b"]), T.field_to_flat(ff["b"]))
    big = T.PatchSpec(128, 128, 8)
    geo_n, state_n = _transport_case(big, 7)
    geo_f, state_f = _transport_case(big, 7)
    params = T.MpdataParams()
    T.run_naive(T.build_mpdata(big, state_n, geo_n, params))
    T.run_fused(T.build_mpdata(big, state_f, geo_f, params), T.TileSpec(64, 64))
    failures += not np.array_equal(T.field_to_flat(state_n.pd_out), T.field_to_flat(state_f.pd_out))
    assert failures == 0, f"{failures} mismatches"


def test_c04_composed_matches_flat_oracle(cuda_ok):
    """100 seeds over 8 shapes <= 8x8x8: the unfused stages == the flat oracle, and the
    fused step and the GPU flat-stage API agree with it too."""
    shapes = [(4, 4, 3), (5, 3, 4), (6, 6, 2), (8, 8, 8), (3, 5, 5), (8, 4, 6), (2, 2, 2), (7, 8, 3)]
    failures = []
    for seed in range(100):
        spec = T.PatchSpec(*shapes[seed % len(shapes)])
        geo, state = _transport_case(spec, seed)
        params = T.MpdataParams(dt=0.2, pivbz=0.8)
        args = _flat_args(spec, geo, state)
        oracle = O.transport_step(*args, params.dt, params.pivbz)
        T.run_naive(T.build_mpdata(spec, state, geo, params))
        same = all(np.array_equal(T.field_to_flat(f), oracle[k])
                   for f, k in ((state.flux, "flux"), (state.fluz, "fluz"), (state.divvd, "div"),
                                (state.pd_out, "pd_out")))
        T.run_fused(T.build_mpdata(spec, state, geo, params))
        same = same and np.array_equal(T.field_to_flat(state.pd_out), oracle["pd_out"])
        flat = T.reference.transport_step(*args, params.dt, params.pivbz)
        same = same and all(np.array_equal(flat[k], oracle[k]) for k in oracle)
        if not same:
            failures.append(seed)
    assert not failures, f"seeds {failures}"


def test_c08_mass_conservation_closed_system(cuda_ok):
    """20 seeds, closed boundary (pivbz = 0), uniform rho: relative mass drift <= 1e-12."""
    shapes = [(6, 6, 4), (8, 4, 5), (5, 7, 3), (4, 4, 2)]
    worst = 0.0
    for seed in range(20):
        spec = T.PatchSpec(*shapes[seed % len(shapes)])
        geo, state = _transport_case(spec, seed, uniform_rho=True)
        comp = T.build_mpdata(spec, state, geo, T.MpdataParams(dt=0.05, pivbz=0.0))
        m0 = T.total_mass(state, geo, "pd_in")
        T.run_naive(comp)
        m1 = T.total_mass(state, geo, "pd_out")
        worst = max(worst, abs(m1 - m0) / abs(m0))
    assert worst <= 1e-12, worst
