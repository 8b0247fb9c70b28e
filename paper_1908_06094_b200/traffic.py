"""Traffic report of a run: the reference's ``RunStats.traffic()`` API over a model.

The reference counts every element access of its CPU executors into per-field
masks and tallies (storage.py:187-270) and reports them through
``TrafficReport`` (storage.py:410-467): per (field, phase) DISTINCT reads /
writes (compulsory traffic, halo images folded onto the interior) and RAW
reads / writes (every access, apron recompute included).  Phases are
``"{tag}/{stage}"`` for run_naive and ``"{tag}/ms{n}"`` for run_fused.

The device kernels are not instrumented (their bytes are measured with ncu,
profiles/).  What the reference would have counted is a closed form of the
patch, the tiling and the stage program, so each run records those counts on
its fields here -- the same rows, with the same values, as the reference's
counters (pinned against reference-generated vectors in tests/test_host.py).
Distinct masks of one phase union (every modelled access covers whole
interiors, so the union is the larger count); raw tallies add across runs,
as in the reference.
"""

from __future__ import annotations

import io
from dataclasses import dataclass, field as dc_field

CSV_HEADER = "field,stage,distinct_reads,distinct_writes,raw_reads,raw_writes"


@dataclass
class TrafficRow:
    field: str
    stage: str
    distinct_reads: int
    distinct_writes: int
    raw_reads: int
    raw_writes: int


@dataclass
class TrafficReport:
    """Per-(field, phase) traffic table with location-aware totals (storage.py:410-467)."""

    rows: list = dc_field(default_factory=list)
    locations: dict = dc_field(default_factory=dict)
    flat: dict = dc_field(default_factory=dict)  # field -> is 2-D

    @classmethod
    def gather(cls, fields, prefix: str = "") -> "TrafficReport":
        report = cls()
        for f in sorted(fields, key=lambda f: f.name):
            report.locations[f.name] = f.meta.location
            report.flat[f.name] = not f.has_levels
            for phase in sorted(f.counters):
                if not phase.startswith(prefix):
                    continue
                dr, dw, rr, rw = f.counters[phase]
                report.rows.append(TrafficRow(f.name, phase, dr, dw, rr, rw))
        return report

    def total_distinct(self, ignore_2d: bool = False, locations=None) -> int:
        total = 0
        for row in self.rows:
            if ignore_2d and self.flat.get(row.field, False):
                continue
            if locations is not None and self.locations[row.field] not in locations:
                continue
            total += row.distinct_reads + row.distinct_writes
        return total

    def total_raw(self, ignore_2d: bool = False) -> int:
        return sum(r.raw_reads + r.raw_writes for r in self.rows
                   if not (ignore_2d and self.flat.get(r.field, False)))

    def to_csv(self, stream=None) -> str:
        out = stream or io.StringIO()
        out.write(CSV_HEADER + "\n")
        for r in self.rows:
            out.write(f"{r.field},{r.stage},{r.distinct_reads},{r.distinct_writes},"
                      f"{r.raw_reads},{r.raw_writes}\n")
        return out.getvalue() if stream is None else ""


def _record(field, phase: str, dr: int = 0, dw: int = 0, rr: int = 0, rw: int = 0) -> None:
    old = field.counters.get(phase)
    if old is None:
        field.counters[phase] = [dr, dw, rr, rw]
    else:
        old[0], old[1] = max(old[0], dr), max(old[1], dw)
        old[2] += rr
        old[3] += rw


def tile_ranges(extent: int, tile: int):
    """Half-open ranges of one axis cut into tiles (the last one ragged)."""
    return [(lo, min(lo + tile, extent)) for lo in range(0, extent, tile)]


def flux_apron_updates(patch, tiles) -> int:
    """Edge-flux updates of the fused plan: every tile recomputes its (1, 0, 1, 0) apron
    (executors.py:307-315 with the flux stage's apron, mpdata.py:342-353); no TileSpec
    = one tile over the whole patch."""
    ti, tj = (patch.rows, patch.cols) if tiles is None else (tiles.tile_i, tiles.tile_j)
    per_tile = sum((i1 - i0 + 1) * (j1 - j0 + 1)
                   for i0, i1 in tile_ranges(patch.rows, ti)
                   for j0, j1 in tile_ranges(patch.cols, tj))
    return per_tile * 3 * patch.levels


def record_run(comp, tag: str, fused: bool, tiles=None) -> dict:
    """Record on ``comp``'s fields what the reference's counters would hold after one
    run_naive (``fused=False``) / run_fused(tiles) of ``comp``; returns its stage updates."""
    p = comp.patch
    V, K = p.rows * p.cols, p.levels
    E, C = 3 * V, 2 * V
    if comp.kind == "mpdata":
        b = comp.bindings
        pd, vn, wn, rho = b["pd_in"], b["vn"], b["wn"], b["rho"]
        signs, dual = b["edge_signs"], b["dual_volumes"]
        if fused:
            fu = flux_apron_updates(p, tiles)
            ph = f"{tag}/ms0"
            _record(pd, ph, dr=V * K, rr=2 * fu + 2 * V * (K + 1) + V * K)
            _record(vn, ph, dr=E * K, rr=fu)
            _record(wn, ph, dr=V * (K - 1), rr=V * (K + 1))
            _record(signs, ph, dr=6 * V, rr=6 * V * K)
            _record(dual, ph, dr=V, rr=V * K)
            _record(rho, ph, dr=V * K, rr=V * K)
            _record(b["pd_out"], ph, dw=V * K, rw=V * K)
            return {"flux": fu, "fluz": V * (K + 1), "divergence": V * K, "advance": V * K}
        ph = {s: f"{tag}/{s}" for s in ("flux", "fluz", "divergence", "advance")}
        _record(pd, ph["flux"], dr=V * K, rr=2 * E * K)
        _record(vn, ph["flux"], dr=E * K, rr=E * K)
        _record(b["flux"], ph["flux"], dw=E * K, rw=E * K)
        _record(pd, ph["fluz"], dr=V * K, rr=2 * V * (K + 1))
        _record(wn, ph["fluz"], dr=V * (K - 1), rr=V * (K + 1))
        _record(b["fluz"], ph["fluz"], dw=V * (K + 1), rw=V * (K + 1))
        _record(b["flux"], ph["divergence"], dr=E * K, rr=2 * E * K)
        _record(b["fluz"], ph["divergence"], dr=V * (K + 1), rr=2 * V * K)
        _record(signs, ph["divergence"], dr=6 * V, rr=6 * V * K)
        _record(dual, ph["divergence"], dr=V, rr=V * K)
        _record(b["divvd"], ph["divergence"], dw=V * K, rw=V * K)
        _record(pd, ph["advance"], dr=V * K, rr=V * K)
        _record(b["divvd"], ph["advance"], dr=V * K, rr=V * K)
        _record(rho, ph["advance"], dr=V * K, rr=V * K)
        _record(b["pd_out"], ph["advance"], dw=V * K, rw=V * K)
        return {"flux": E * K, "fluz": V * (K + 1), "divergence": V * K, "advance": V * K}
    if comp.kind == "divergence":
        b, Ko = comp.bindings, comp.out.meta.levels
        name = "div_weighted" if comp.weighted else "div_simple"
        ph = f"{tag}/ms0" if fused else f"{tag}/{name}"
        _record(b["vn"], ph, dr=E * K, rr=3 * C * Ko)
        if comp.weighted:
            _record(b["weights"], ph, dr=3 * C, rr=3 * C * Ko)
        else:
            _record(b["length"], ph, dr=E, rr=3 * C * Ko)
            _record(b["area"], ph, dr=C, rr=C * Ko)
        _record(b["div_out"], ph, dw=C * Ko, rw=C * Ko)
        return {name: C * Ko}
    if comp.kind == "reduce":
        from .connectivity import neighbor_len
        from .topology import element_count

        nf, nt = element_count(p, comp.from_loc), element_count(p, comp.to_loc)
        Kr = comp.dst.inner
        ph = f"{tag}/ms0" if fused else f"{tag}/{comp.name}"
        _record(comp.src, ph, dr=nt * Kr, rr=neighbor_len(comp.from_loc, comp.to_loc) * nf * Kr)
        if comp.scale is not None:
            _record(comp.scale, ph, dr=nf, rr=nf * Kr)
        _record(comp.dst, ph, dw=nf * Kr, rw=nf * Kr)
        return {comp.name: nf * Kr}
    raise TypeError(f"no traffic model for computation kind {getattr(comp, 'kind', None)!r}")


def required_tile(comp) -> tuple[int, int]:
    """Largest stage reach (rows, cols) of a computation: the hull of its neighbour offsets
    (executors.py:248-263).  The MPDATA step and the cell divergence reach (1, 1); the
    Table-1 C->C sum (2, 2)."""
    if comp.kind in ("mpdata", "divergence"):
        return 1, 1
    from .connectivity import OFFSET_TABLES

    offs = [e for col in OFFSET_TABLES[(comp.from_loc, comp.to_loc)] for e in col]
    di = [e[0] for e in offs] + [0]
    dj = [e[2] for e in offs] + [0]
    return max(di) - min(di), max(dj) - min(dj)
