"""RunStats.traffic() / stage updates / tile-reach errors vs the reference (CPU).

The golden reports in tests/golden/traffic.json come from running the real
reference executors (tests/golden/make_traffic_golden.py); here the same
sequence of runs is recorded on this package's Fields through
traffic.record_run (what run_gpu calls after each launch) and must give the
same rows, totals and stage updates.  No kernel runs: the model is host code.
"""

from __future__ import annotations

import json
from pathlib import Path

import pytest

from paper_1908_06094_b200 import (CompositionError, GeometryFields, MpdataParams, PatchSpec,
                                   Selector, TileSpec, build_state, make_kernel_fields,
                                   make_storage, run_fused)
from paper_1908_06094_b200.executors import RunStats
from paper_1908_06094_b200.kernels import build_kernel
from paper_1908_06094_b200.mpdata import DivergenceComputation, MpdataComputation
from paper_1908_06094_b200.topology import LocationType
from paper_1908_06094_b200.traffic import TrafficReport, record_run

GOLD = json.loads((Path(__file__).parent / "golden" / "traffic.json").read_text())
V, C, E = LocationType.VERTICES, LocationType.CELLS, LocationType.EDGES


def _geometry(spec):
    flat = Selector(level=False)
    return GeometryFields(
        edge_length=make_storage(spec, E, "edge_length", flat),
        cell_area=make_storage(spec, C, "cell_area", flat),
        dual_volumes=make_storage(spec, V, "dual_volumes", flat),
        edge_signs=make_storage(spec, V, "edge_signs", Selector(level=False, extra=True), extra_len=6),
        weights=make_storage(spec, C, "weights", Selector(level=False, extra=True), extra_len=3))


def _stats(comp, tiles):
    tag = "naive" if tiles is None else "fused"
    ts = None if tiles is None else TileSpec(*tiles)
    updates = record_run(comp, tag, fused=tiles is not None, tiles=ts)
    return RunStats(tag=tag, executor="model", fields=comp.fields(), stage_updates=updates)


def _check(stats, case):
    rep = stats.traffic()
    assert isinstance(rep, TrafficReport)
    assert stats.stage_updates == case["stage_updates"]
    got = [[r.field, r.stage, r.distinct_reads, r.distinct_writes, r.raw_reads, r.raw_writes]
           for r in rep.rows]
    assert got == case["rows"]
    assert rep.total_distinct() == case["total_distinct"]
    assert rep.total_distinct(ignore_2d=True) == case["total_distinct_3d"]
    assert rep.total_raw() == case["total_raw"]


def test_traffic_reports_match_reference():
    cases = iter(GOLD["cases"])
    for rows, cols, levels in ((6, 8, 4), (12, 10, 5)):
        spec = PatchSpec(rows, cols, levels)
        for tiles in (None, (4, 4), (5, 3), (1, 1), (rows, cols)):
            case = next(cases)
            assert case["kind"] == "mpdata" and case["tiles"] == (None if tiles is None else list(tiles))
            comp = MpdataComputation(spec, build_state(spec), _geometry(spec), MpdataParams(), "upwind")
            _check(_stats(comp, tiles), case)
        state, geo = build_state(spec), _geometry(spec)
        out = make_storage(spec, C, "div_out")
        for weighted in (False, True):
            for tiles in (None, (4, 4)):
                case = next(cases)
                assert case["kind"] == "divergence" and case["weighted"] == weighted
                _check(_stats(DivergenceComputation(spec, state, geo, weighted, out), tiles), case)
        for scaled in (False, True):
            for tiles in (None, (2, 2)):
                case = next(cases)
                assert case["kind"] == "kernel" and case["scaled"] == scaled
                _check(_stats(build_kernel(spec, make_kernel_fields(spec), scaled), tiles), case)
    assert next(cases, None) is None


def test_run_fused_rejects_tiles_below_the_stage_reach():
    spec = PatchSpec(6, 8, 4)
    for err in GOLD["tile_errors"]:
        comp = build_kernel(spec, make_kernel_fields(spec), False)
        with pytest.raises(ValueError) as exc:
            run_fused(comp, TileSpec(*err["tiles"]))  # raises before any device work
        assert str(exc.value) == err["message"]


def test_composition_error_is_a_value_error():
    assert issubclass(CompositionError, ValueError)


def test_coalescing_models_match_reference():
    """gather_groups / coalescing_fraction / direct_sweep_groups vs the reference's values
    (kernels.py:137-155, layouts.py:282-326); tables from the pinned oracle."""
    import numpy as np

    from oracle import tsg_oracle as O
    from paper_1908_06094_b200 import (LayoutSpec, coalescing_fraction, direct_sweep_groups,
                                       gather_groups)

    fwd = {"sn": lambda r, c: None, "un": lambda r, c: O.un_forward(r, c, "cells"),
           "hn": lambda r, c: O.hn_forward(r, c, "cells")}
    seen = 0
    for case in GOLD["coalescing"]:
        r, c, k = case["patch"]
        if case["what"] == "gather":
            f = fwd[case["numbering"]](r, c)
            table = O.neighbor_table(r, c, "cells", "cells", f, f)
            g = gather_groups(table, case["width"], case["own_reads"])
            assert [list(map(int, x)) for x in g[:12]] == case["groups"]
        else:
            order = case["order"]
            lay = LayoutSpec() if order is None else LayoutSpec(dim_order=tuple(order))
            g = direct_sweep_groups(lay, PatchSpec(r, c, k), case["loc"], case["width"])
            assert [list(map(int, x)) for x in g[:12]] + [list(map(int, g[-1]))] == case["groups"]
        assert len(g) == case["n"]
        assert coalescing_fraction(g) == case["fraction"]
        seen += 1
    assert seen == 66
    with pytest.raises(ValueError):
        coalescing_fraction([])
    with pytest.raises(ValueError):
        gather_groups(np.zeros((2, 3), dtype=np.int64), 0)
