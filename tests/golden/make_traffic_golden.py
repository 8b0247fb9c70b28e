"""Golden traffic reports and tile-reach errors from the REAL reference package.

Run in the build container only (the GPU box has no /root/reference):

    python tests/golden/make_traffic_golden.py

Writes ``tests/golden/traffic.json``: for each case the reference's
``RunStats.stage_updates`` and ``RunStats.traffic()`` rows (executors.py:48-71,
storage.py:410-467) after run_naive / run_fused(TileSpec) of the MPDATA step,
the cell divergence (both forms, on shared fields like its tests) and the
Table-1 kernels, plus the messages run_fused raises for tiles below the stage
reach (executors.py:276-282).
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from tristencil import kernels as kn  # noqa: E402
from tristencil import mpdata as mp  # noqa: E402
from tristencil.bench import BenchConfig, _transport_setup  # noqa: E402
from tristencil.executors import TileSpec, run_fused, run_naive  # noqa: E402
from tristencil.storage import make_storage  # noqa: E402
from tristencil.topology import LocationType  # noqa: E402

OUT = Path(__file__).parent / "traffic.json"


def report(stats):
    rep = stats.traffic()
    return {"tag": stats.tag, "stage_updates": stats.stage_updates,
            "rows": [[r.field, r.stage, r.distinct_reads, r.distinct_writes, r.raw_reads, r.raw_writes]
                     for r in rep.rows],
            "total_distinct": rep.total_distinct(), "total_distinct_3d": rep.total_distinct(ignore_2d=True),
            "total_raw": rep.total_raw()}


def coalescing():
    """gather_groups / coalescing_fraction / direct_sweep_groups (kernels.py:137-155,
    layouts.py:282-326) on small patches, every numbering and both layouts."""
    from tristencil.connectivity import build_neighbor_table
    from tristencil.kernels import gather_groups
    from tristencil.layouts import (LayoutSpec, Numbering, coalescing_fraction, direct_sweep_groups,
                                    make_permutation)
    from tristencil.topology import PatchSpec

    out = []
    for rows, cols, levels in ((4, 6, 3), (8, 8, 2)):
        spec = PatchSpec(rows, cols, levels)
        for num in (Numbering.SN, Numbering.UN, Numbering.HN):
            if num is Numbering.HN and rows != cols:
                continue
            perm = make_permutation(num, spec, LocationType.CELLS)
            table = build_neighbor_table(spec, LocationType.CELLS, LocationType.CELLS, perm, perm)
            for width in (1, 4, 8):
                for own in (0, 1):
                    g = gather_groups(table, width, own)
                    out.append({"what": "gather", "patch": [rows, cols, levels], "numbering": num.value,
                                "width": width, "own_reads": own, "n": len(g),
                                "groups": [[int(a) for a in x] for x in g[:12]],
                                "fraction": coalescing_fraction(g)})
        for order in (None, ("extra", "row", "color", "column", "level")):
            lay = LayoutSpec() if order is None else LayoutSpec(dim_order=order)
            for loc in (LocationType.VERTICES, LocationType.CELLS, LocationType.EDGES):
                for width in (1, 4, 5):
                    g = direct_sweep_groups(lay, spec, loc, width)
                    out.append({"what": "direct", "patch": [rows, cols, levels], "order": order,
                                "loc": loc.value, "width": width, "n": len(g),
                                "groups": [list(map(int, x)) for x in g[:12]] + [list(map(int, g[-1]))],
                                "fraction": coalescing_fraction(g)})
    return out


def main():
    cases = []
    for rows, cols, levels in ((6, 8, 4), (12, 10, 5)):
        cfg = BenchConfig(rows=rows, cols=cols, levels=levels)
        spec = cfg.patch()
        for tiles in (None, (4, 4), (5, 3), (1, 1), (rows, cols)):
            st, geo, p = _transport_setup(cfg, spec)
            comp = mp.build_mpdata(spec, st, geo, p)
            stats = run_naive(comp) if tiles is None else run_fused(comp, TileSpec(*tiles))
            cases.append({"kind": "mpdata", "patch": [rows, cols, levels], "tiles": tiles,
                          **report(stats)})
        # the divergence pair on shared fields (naive, then fused), as the reference's tests
        st, geo, p = _transport_setup(cfg, spec)
        mp.precompute_weights(spec, geo)
        out = make_storage(spec, LocationType.CELLS, "div_out")
        for weighted in (False, True):
            for tiles in (None, (4, 4)):
                comp = mp.build_divergence(spec, st, geo, weighted, out)
                stats = run_naive(comp) if tiles is None else run_fused(comp, TileSpec(*tiles))
                cases.append({"kind": "divergence", "weighted": weighted, "patch": [rows, cols, levels],
                              "tiles": tiles, **report(stats)})
        for scaled in (False, True):
            for tiles in (None, (2, 2)):
                comp = kn.build_kernel(spec, kn.make_kernel_fields(spec), scaled)
                stats = run_naive(comp) if tiles is None else run_fused(comp, TileSpec(*tiles))
                cases.append({"kind": "kernel", "scaled": scaled, "patch": [rows, cols, levels],
                              "tiles": tiles, **report(stats)})
    errors = []
    cfg = BenchConfig(rows=6, cols=8, levels=4)
    spec = cfg.patch()
    for tiles in ((1, 1), (1, 2), (2, 1)):
        comp = kn.build_kernel(spec, kn.make_kernel_fields(spec), False)
        try:
            run_fused(comp, TileSpec(*tiles))
            errors.append({"tiles": tiles, "message": None})
        except ValueError as e:
            errors.append({"tiles": tiles, "message": str(e)})
    OUT.write_text(json.dumps({"cases": cases, "tile_errors": errors, "coalescing": coalescing()},
                              indent=0))
    print(f"wrote {OUT} ({len(cases)} cases)")


if __name__ == "__main__":
    main()
