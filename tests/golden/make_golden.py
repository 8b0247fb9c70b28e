"""Generate golden parity fixtures by running the REAL reference package.

Run in the build container only (the GPU box has no /root/reference):

    python tests/golden/make_golden.py

It imports ``tristencil`` from /root/reference/pkg/src unmodified (bytecode
writing disabled: the tree is read-only) and writes

* ``tests/golden/golden_small.npz``  -- full input/output arrays for small
  patches: all nine neighbour tables and edge signs on several patches,
  UN/HN permutations, relabelled tables, Hilbert walks, 24 transport cases
  (shapes of tests/test_acceptance.py:167-186), centred flux, Table-1 neighbour
  sums (direct baseline), every 9-relation structured reduce, cell divergence;
* ``tests/golden/golden_hashes.json`` -- SHA-256 digests of the canonical
  ``[element, level]`` float64 bytes of inputs and outputs for bench-sized
  patches (44x72x10, 128x128x80, 279x256x80), plus layout known answers.

Every transport output comes from ``reference.transport_step`` and is also
asserted equal to ``run_naive`` of the composed computation, as the
reference's own acceptance test C4 does.
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

sys.dont_write_bytecode = True
REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))

import numpy as np  # noqa: E402

import tristencil.bench as tb  # noqa: E402
from tristencil import reference  # noqa: E402
from tristencil.connectivity import OFFSET_TABLES, build_neighbor_table, edge_signs_table  # noqa: E402
from tristencil.executors import halo_update, run_naive  # noqa: E402
from tristencil.kernels import build_kernel, field_to_flat, make_kernel_fields  # noqa: E402
from tristencil.layouts import (  # noqa: E402
    LayoutSpec, LinearLayout, Numbering, hilbert_rank, hilbert_xy, make_permutation, sn_offset)
from tristencil.mpdata import (  # noqa: E402
    MpdataParams, build_divergence, build_geometry, build_mpdata, build_state, init_preset)
from tristencil.stencil import Intent, StageSpec, StageUse, accessor, compose, multistage  # noqa: E402
from tristencil.storage import make_storage  # noqa: E402
from tristencil.topology import LocationType, PatchSpec  # noqa: E402

OUT = Path(__file__).parent
V, C, E = LocationType.VERTICES, LocationType.CELLS, LocationType.EDGES
LOC = {"vertices": V, "cells": C, "edges": E}


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()).hexdigest()


def fill(field, rng, lo, hi):
    spec = field.spec
    h = spec.halo
    arr = field.array("primary", "rw")
    shape = arr[h:h + spec.rows, :, h:h + spec.cols, :, :].shape
    arr[h:h + spec.rows, :, h:h + spec.cols, :, :] = lo + (hi - lo) * rng.random(shape)
    halo_update(field)


def transport_case(spec, seed, geometry="random", rho="random"):
    """tests/test_acceptance.py:81-92 (rho='random') / bench._transport_setup-like."""
    geo = build_geometry(spec, geometry, seed=seed)
    state = build_state(spec)
    rng = np.random.default_rng(seed)
    init_preset(state.pd_in, "random", seed=seed)
    fill(state.vn, rng, -0.5, 0.5)
    fill(state.wn, rng, -0.5, 0.5)
    if rho == "random":
        fill(state.rho, rng, 0.5, 1.5)
    else:
        init_preset(state.rho, "uniform")
    return geo, state


def oracle(spec, geo, state, params, flux_op="upwind"):
    return reference.transport_step(
        build_neighbor_table(spec, E, V).ids, build_neighbor_table(spec, V, E).ids,
        edge_signs_table(spec), field_to_flat(geo.dual_volumes)[:, 0],
        field_to_flat(state.pd_in), field_to_flat(state.vn), field_to_flat(state.wn),
        field_to_flat(state.rho), params.dt, params.pivbz, flux_op=flux_op)


def check_naive(spec, geo, state, params, want, flux_op="upwind"):
    run_naive(build_mpdata(spec, state, geo, params, flux_op))
    assert np.array_equal(field_to_flat(state.flux), want["flux"])
    assert np.array_equal(field_to_flat(state.fluz), want["fluz"])
    assert np.array_equal(field_to_flat(state.divvd), want["div"])
    assert np.array_equal(field_to_flat(state.pd_out), want["pd_out"])


def main():
    small: dict[str, np.ndarray] = {}
    hashes: dict = {"transport": {}, "indexing": {}, "layouts": []}

    # -- connectivity: 9 tables + signs --------------------------------------
    for rows, cols in ((2, 2), (3, 3), (2, 5), (4, 3), (5, 6), (7, 4), (8, 8)):
        spec = PatchSpec(rows, cols, 1)
        for (f, t) in OFFSET_TABLES:
            small[f"tbl_{rows}x{cols}_{f.value}_{t.value}"] = build_neighbor_table(spec, f, t).ids
        small[f"signs_{rows}x{cols}"] = edge_signs_table(spec)

    # -- numberings ----------------------------------------------------------
    for rows, cols in ((5, 7), (16, 8), (3, 9), (4, 4), (4, 2), (6, 5)):
        spec = PatchSpec(rows, cols, 1)
        for loc in (V, C, E):
            small[f"perm_un_{rows}x{cols}_{loc.value}"] = make_permutation(Numbering.UN, spec, loc).forward
        for loc in (V, C):
            small[f"perm_hn_{rows}x{cols}_{loc.value}"] = make_permutation(Numbering.HN, spec, loc).forward
    for rows, cols in ((16, 8), (5, 7)):
        spec = PatchSpec(rows, cols, 1)
        for num in (Numbering.UN, Numbering.HN):
            p = make_permutation(num, spec, C)
            small[f"tblp_{num.value}_{rows}x{cols}_cells_cells"] = build_neighbor_table(spec, C, C, p, p).ids
    spec = PatchSpec(4, 4, 1)
    pv, pe = make_permutation(Numbering.HN, spec, V), make_permutation(Numbering.UN, spec, E)
    small["tblp_relabel_4x4_edges_vertices"] = build_neighbor_table(spec, E, V, pe, pv).ids
    small["tblp_relabel_4x4_vertices_edges"] = build_neighbor_table(spec, V, E, pv, pe).ids

    # -- Hilbert walks (reference golden files + larger orders) --------------
    data = Path("/root/reference/pkg/tests/data")
    for n in (2, 4):
        rows_ = [tuple(map(int, ln.split())) for ln in (data / f"hilbert_n{n}.txt").read_text().splitlines()
                 if ln and not ln.startswith("#")]
        small[f"hilbert_file_n{n}"] = np.array(rows_, dtype=np.int64)
    for n in (8, 32):
        xy = np.array([hilbert_xy(n, d) for d in range(n * n)], dtype=np.int64)
        small[f"hilbert_xy_n{n}"] = xy
        assert all(hilbert_rank(n, int(x), int(y)) == d for d, (x, y) in enumerate(xy))

    # -- layouts known answers ----------------------------------------------
    orders = {"default": ("extra", "level", "row", "color", "column"),
              "level-inner": ("extra", "row", "color", "column", "level")}
    for oname, order in orders.items():
        for align in (1, 8, 16):
            for sizes in ({"row": 6, "color": 1, "column": 6, "level": 4, "extra": 1},
                          {"row": 7, "color": 2, "column": 11, "level": 4, "extra": 1},
                          {"row": 5, "color": 3, "column": 9, "level": 81, "extra": 1},
                          {"row": 6, "color": 1, "column": 5, "level": 1, "extra": 6}):
                lin = LinearLayout(LayoutSpec(order, align), sizes, halo=1)
                hashes["layouts"].append(dict(order=oname, alignment=align, sizes=sizes, halo=1,
                                              padded=lin.padded, strides=lin.strides,
                                              front_pad=lin.front_pad, total=lin.total))
    spec = PatchSpec(5, 4, 3)
    offs = []
    for loc in (V, C, E):
        for (i, c, j, k) in ((0, 0, 0, 0), (-1, 0, -1, 2), (4, loc.colors - 1, 4, 1), (2, 0, 3, 0)):
            offs.append([loc.value, i, c, j, k, sn_offset(LayoutSpec(), spec, loc, i, c, j, k)])
    hashes["sn_offset_5x4x3"] = offs

    # -- small transport cases: full arrays ----------------------------------
    shapes = [(4, 4, 3), (5, 3, 4), (6, 6, 2), (8, 8, 8), (3, 5, 5), (8, 4, 6), (2, 2, 2), (7, 8, 3)]
    cases = []
    for seed in range(24):
        shape = shapes[seed % len(shapes)]
        cases.append((f"tr{seed}", shape, seed, "random", 0.2, 0.8, "upwind"))
    cases.append(("trc", (5, 4, 3), 3, "random", 0.1, 1.0, "centred"))
    cases.append(("tru", (4, 4, 3), 0, "uniform", 0.2, 0.7, "upwind"))
    cases.append(("trp0", (6, 6, 4), 1, "random", 0.05, 0.0, "upwind"))
    meta = []
    for key, shape, seed, gmode, dt, pivbz, op in cases:
        spec = PatchSpec(*shape)
        geo, state = transport_case(spec, seed, gmode, "random")
        params = MpdataParams(dt=dt, pivbz=pivbz)
        want = oracle(spec, geo, state, params, op)
        check_naive(spec, geo, state, params, want, op)
        small[f"{key}_pd"] = field_to_flat(state.pd_in)
        small[f"{key}_vn"] = field_to_flat(state.vn)
        small[f"{key}_wn"] = field_to_flat(state.wn)
        small[f"{key}_rho"] = field_to_flat(state.rho)
        small[f"{key}_dual"] = field_to_flat(geo.dual_volumes)[:, 0]
        small[f"{key}_signs"] = edge_signs_table(spec)
        for out in ("flux", "fluz", "div", "pd_out"):
            small[f"{key}_{out}"] = want[out]
        meta.append(dict(key=key, shape=list(shape), seed=seed, geometry=gmode, dt=dt,
                         pivbz=pivbz, flux_op=op))
    hashes["small_transport"] = meta

    # -- hashed bench-sized transport cases -----------------------------------
    big = [
        ("cfg1_s0", (44, 72, 10), dict(seed=0, geometry="random", preset="random", dt=0.2, pivbz=0.8)),
        ("cfg1_s1", (44, 72, 10), dict(seed=1, geometry="random", preset="random", dt=0.2, pivbz=0.8)),
        ("cfg1_default", (44, 72, 10), dict(seed=0)),
        ("cfg2_rand", (128, 128, 80), dict(seed=0, geometry="random", preset="random")),
        ("cfg3_rand", (279, 256, 80), dict(seed=0, geometry="random", preset="random")),
        ("cfg3_default", (279, 256, 80), dict(seed=0)),
    ]
    for key, (r, c, k), kw in big:
        cfg = tb.BenchConfig(rows=r, cols=c, levels=k, **kw)
        spec = cfg.patch()
        state, geo, params = tb._transport_setup(cfg, spec)
        want = oracle(spec, geo, state, params)
        if k <= 10:
            state2, geo2, _ = tb._transport_setup(cfg, spec)
            check_naive(spec, geo2, state2, params, want)
        entry = dict(rows=r, cols=c, levels=k, config=kw, dt=params.dt, pivbz=params.pivbz,
                     exp_dependent=cfg.preset == "gaussian-bump",
                     inputs={n: sha(a) for n, a in (
                         ("pd", field_to_flat(state.pd_in)), ("vn", field_to_flat(state.vn)),
                         ("wn", field_to_flat(state.wn)), ("rho", field_to_flat(state.rho)),
                         ("dual", field_to_flat(geo.dual_volumes)[:, 0]),
                         ("signs", edge_signs_table(spec)))},
                     outputs={n: sha(want[n]) for n in ("flux", "fluz", "div", "pd_out")},
                     probe={n: [float(want[n][0, 0]), float(want[n][-1, -1])]
                            for n in ("flux", "fluz", "div", "pd_out")})
        hashes["transport"][key] = entry
        print(key, "done", flush=True)

    # multi-step time loop (bench.run_mpdata: pd_out -> pd_in between steps)
    cfg = tb.BenchConfig(rows=44, cols=72, levels=10, seed=2, geometry="random",
                         preset="random", dt=0.2, pivbz=0.8)
    spec = cfg.patch()
    state, geo, params = tb._transport_setup(cfg, spec)
    pd = field_to_flat(state.pd_in)
    for _ in range(10):
        pd = oracle_flat(spec, geo, pd, state, params)
    hashes["transport"]["cfg1_s2_10steps"] = dict(
        rows=44, cols=72, levels=10, config=dict(seed=2, geometry="random", preset="random",
                                                dt=0.2, pivbz=0.8),
        dt=0.2, pivbz=0.8, steps=10, outputs={"pd_out": sha(pd)})

    # -- Table-1 neighbour sums: direct structured baseline -------------------
    for rows, cols, levels in ((16, 8, 2), (5, 7, 3)):
        spec = PatchSpec(rows, cols, levels)
        rng = np.random.default_rng(rows * 100 + cols)
        fields = make_kernel_fields(spec)
        fill(fields["a"], rng, 0.0, 1.0)
        fill(fields["fac"], rng, 0.5, 1.5)
        small[f"k_{rows}x{cols}x{levels}_a"] = field_to_flat(fields["a"])
        small[f"k_{rows}x{cols}x{levels}_fac"] = field_to_flat(fields["fac"])
        for scaled, tag in ((False, "k1"), (True, "k2")):
            run_naive(build_kernel(spec, fields, scaled))
            small[f"k_{rows}x{cols}x{levels}_{tag}"] = field_to_flat(fields["b"])
    spec = PatchSpec(128, 128, 80)
    rng = np.random.default_rng(0)  # bench.run_indexing: a then fac from default_rng(seed)
    fields = make_kernel_fields(spec)
    tb._fill_random(fields["a"], rng)
    tb._fill_random(fields["fac"], rng, 0.5, 1.5)
    entry = {"a": sha(field_to_flat(fields["a"])), "fac": sha(field_to_flat(fields["fac"]))}
    for scaled, tag in ((False, "k1"), (True, "k2")):
        run_naive(build_kernel(spec, fields, scaled))
        entry[tag] = sha(field_to_flat(fields["b"]))
    hashes["indexing"]["cfg2"] = entry

    # -- all nine relations through the structured reduce ---------------------
    spec = PatchSpec(6, 5, 3)
    for (f, t) in OFFSET_TABLES:
        src = make_storage(spec, t, "a")
        dst = make_storage(spec, f, "b")
        fill(src, np.random.default_rng(17), 0.0, 1.0)

        def body(ev, t=t):
            ev.store(ev.reduce(t, lambda nv, acc: nv + acc, 0.0, "a"))

        stage = StageSpec(name="reduce", location=f,
                          accessors=(accessor("a", Intent.IN, t, extent=(-1, 1, -1, 1)),
                                     accessor("b", Intent.OUT, f)), body=body)
        run_naive(compose(spec, [multistage("parallel", StageUse(stage, ("a", "b")))],
                          {"a": src, "b": dst}))
        got = field_to_flat(dst)
        flat = reference.neighbor_sum(build_neighbor_table(spec, f, t).ids, field_to_flat(src))
        assert np.array_equal(got, flat)
        small[f"red_{f.value}_{t.value}_a"] = field_to_flat(src)
        small[f"red_{f.value}_{t.value}_b"] = got

    # -- cell divergence -----------------------------------------------------
    spec = PatchSpec(5, 5, 3)
    geo, state = transport_case(spec, 7, "random", "random")
    for weighted in (False, True):
        out = make_storage(spec, C, "div_out")
        run_naive(build_divergence(spec, state, geo, weighted=weighted, out=out))
        small[f"cdiv_{int(weighted)}"] = field_to_flat(out)
    small["cdiv_vn"] = field_to_flat(state.vn)
    small["cdiv_length"] = field_to_flat(geo.edge_length)[:, 0]
    small["cdiv_area"] = field_to_flat(geo.cell_area)[:, 0]
    small["cdiv_weights"] = geo.weights.core()[:, :, :, 0, :].reshape(-1, 3)
    assert np.array_equal(small["cdiv_0"], reference.cell_divergence(
        build_neighbor_table(spec, C, E).ids, small["cdiv_vn"], small["cdiv_length"], small["cdiv_area"]))

    np.savez_compressed(OUT / "golden_small.npz", **small)
    (OUT / "golden_hashes.json").write_text(json.dumps(hashes, indent=1, sort_keys=True))
    print("wrote", len(small), "arrays")


def oracle_flat(spec, geo, pd, state, params):
    return reference.transport_step(
        build_neighbor_table(spec, E, V).ids, build_neighbor_table(spec, V, E).ids,
        edge_signs_table(spec), field_to_flat(geo.dual_volumes)[:, 0], pd,
        field_to_flat(state.vn), field_to_flat(state.wn), field_to_flat(state.rho),
        params.dt, params.pivbz)["pd_out"]


if __name__ == "__main__":
    main()
