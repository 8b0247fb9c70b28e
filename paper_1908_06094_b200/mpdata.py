"""The MPDATA transport step: state/geometry builders and the computation object.

Mirrors the public API of tristencil.mpdata (mpdata.py:51-500):
``MpdataParams``, ``build_state``, ``build_geometry``, ``precompute_weights``,
``init_preset``, ``load_field_csv``, ``build_mpdata``, ``build_divergence``,
``total_mass``.  Input generation keeps the reference's numpy RNG streams, so
the same seeds give bitwise the same inputs (pinned by tests/golden).

``build_mpdata`` returns an :class:`MpdataComputation` that records
``dt``/``pivbz``/``flux_op`` (the reference closes over them inside stage
bodies, mpdata.py:246-287) and is executed by the runners of
:mod:`paper_1908_06094_b200.executors` on the GPU.
"""

from __future__ import annotations

import csv
import zlib
from dataclasses import dataclass

import numpy as np

from . import _lib
from .connectivity import edge_signs_table
from .storage import Field, Selector, device_grid, make_storage
from .topology import LocationType, PatchSpec, element_coord, element_count

_V, _C, _E = LocationType.VERTICES, LocationType.CELLS, LocationType.EDGES

UNIT_EDGE_LENGTH = 1.0
UNIT_CELL_AREA = np.sqrt(3.0) / 4.0
UNIT_DUAL_VOLUME = np.sqrt(3.0) / 2.0

FLUX_OPS = {"upwind": 0, "centred": 1}


@dataclass(frozen=True)
class MpdataParams:
    dt: float = 0.1
    pivbz: float = 1.0

    def __post_init__(self):
        if not np.isfinite(self.dt) or self.dt < 0:
            raise ValueError(f"dt must be finite and >= 0, got {self.dt}")
        if not np.isfinite(self.pivbz):
            raise ValueError(f"pivbz must be finite, got {self.pivbz}")


@dataclass
class GeometryFields:
    edge_length: Field
    cell_area: Field
    dual_volumes: Field
    edge_signs: Field
    weights: Field

    def fields(self):
        return [self.edge_length, self.cell_area, self.dual_volumes, self.edge_signs, self.weights]


@dataclass
class StateFields:
    pd_in: Field
    pd_out: Field
    vn: Field
    wn: Field
    rho: Field
    flux: Field
    fluz: Field
    divvd: Field

    def fields(self):
        return [self.pd_in, self.pd_out, self.vn, self.wn, self.rho, self.flux, self.fluz, self.divvd]


def _interior(field: Field):
    h, r, c = field.spec.halo, field.spec.rows, field.spec.cols
    return (slice(h, h + r), slice(None), slice(h, h + c))


def build_geometry(spec: PatchSpec, mode: str = "uniform", seed: int = 0, layout=None) -> GeometryFields:
    """Geometry fields (mpdata.py:106-149); signs and weights come from device kernels."""
    flat = Selector(level=False)
    geo = GeometryFields(
        edge_length=make_storage(spec, _E, "edge_length", flat, layout=layout),
        cell_area=make_storage(spec, _C, "cell_area", flat, layout=layout),
        dual_volumes=make_storage(spec, _V, "dual_volumes", flat, layout=layout),
        edge_signs=make_storage(spec, _V, "edge_signs", Selector(level=False, extra=True),
                                extra_len=6, layout=layout),
        weights=make_storage(spec, _C, "weights", Selector(level=False, extra=True),
                             extra_len=3, layout=layout),
    )
    rows, cols = spec.rows, spec.cols
    if mode == "uniform":
        lengths = np.full((rows, 3, cols), UNIT_EDGE_LENGTH)
        areas = np.full((rows, 2, cols), UNIT_CELL_AREA)
        volumes = np.full((rows, 1, cols), UNIT_DUAL_VOLUME)
    elif mode == "random":
        rng = np.random.default_rng(seed)  # draw order: lengths, areas, volumes
        lengths = UNIT_EDGE_LENGTH * (0.5 + rng.random((rows, 3, cols)))
        areas = UNIT_CELL_AREA * (0.5 + rng.random((rows, 2, cols)))
        volumes = UNIT_DUAL_VOLUME * (0.5 + rng.random((rows, 1, cols)))
    else:
        raise ValueError(f"unknown geometry mode {mode!r}")
    for field, values in ((geo.edge_length, lengths), (geo.cell_area, areas),
                          (geo.dual_volumes, volumes)):
        field.array("primary", "rw")[_interior(field) + (0, 0)] = values
    signs = edge_signs_table(spec)
    geo.edge_signs.array("primary", "rw")[_interior(geo.edge_signs) + (0,)] = \
        signs.reshape(rows, 1, cols, 6)
    precompute_weights(spec, geo)
    from .executors import halo_update

    for field in geo.fields():
        if field.current_space() == "primary":
            halo_update(field)
    return geo


def precompute_weights(spec: PatchSpec, geo: GeometryFields) -> None:
    """weights[c, n] = length(e_n) / area(c) in C->E order, on the device (tsg_cell_weights)."""
    area = geo.cell_area
    core = area.core(area.current_space())
    if bool((core == 0.0).any()):
        raise ValueError("cell_area contains zeros; weights are undefined")
    grid = device_grid(spec)
    lp, ap = geo.edge_length.ensure_device(), area.ensure_device()
    w = geo.weights.buffer("mirror")
    _lib.call("tsg_cell_weights", grid.handle, _lib.ptr(lp), _lib.ptr(ap), _lib.ptr(w),
              _lib.stream_handle())
    geo.weights.mark_device_written()
    from .storage import sync

    sync(geo.weights, "primary")


def build_state(spec: PatchSpec, layout=None) -> StateFields:
    return StateFields(
        pd_in=make_storage(spec, _V, "pd_in", layout=layout),
        pd_out=make_storage(spec, _V, "pd_out", layout=layout),
        vn=make_storage(spec, _E, "vn", layout=layout),
        wn=make_storage(spec, _V, "wn", levels=spec.levels + 1, layout=layout),
        rho=make_storage(spec, _V, "rho", layout=layout),
        flux=make_storage(spec, _E, "flux", layout=layout),
        fluz=make_storage(spec, _V, "fluz", levels=spec.levels + 1, layout=layout),
        divvd=make_storage(spec, _V, "divvd", layout=layout),
    )


class MpdataComputation:
    """The composed transport step (mpdata.py:319-354), with its parameters recorded."""

    kind = "mpdata"
    stage_names = ("flux", "fluz", "divergence", "advance")

    def __init__(self, patch, state: StateFields, geo: GeometryFields, params: MpdataParams,
                 flux_op: str):
        self.patch = patch
        self.state = state
        self.geo = geo
        self.params = params
        self.flux_op = flux_op
        self.bindings = {
            "pd_in": state.pd_in, "pd_out": state.pd_out, "vn": state.vn, "wn": state.wn,
            "rho": state.rho, "flux": state.flux, "fluz": state.fluz, "divvd": state.divvd,
            "edge_signs": geo.edge_signs, "dual_volumes": geo.dual_volumes,
        }

    def fields(self):
        return list(self.bindings.values())

    def stage_updates(self) -> dict:
        """Per-stage element updates, counted like run_naive (executors.py:243)."""
        v = self.patch.rows * self.patch.cols
        k = self.patch.levels
        return {"flux": 3 * v * k, "fluz": v * (k + 1), "divergence": v * k, "advance": v * k}

    def total_updates(self) -> int:
        return sum(self.stage_updates().values())


def build_mpdata(spec: PatchSpec, state: StateFields, geo: GeometryFields, params: MpdataParams,
                 flux_op: str = "upwind") -> MpdataComputation:
    if flux_op not in FLUX_OPS:
        raise ValueError(f"flux operator must be one of {sorted(FLUX_OPS)}, got {flux_op!r}")
    if spec.levels < 2:
        raise ValueError(f"the transport step needs at least 2 levels, got {spec.levels}")
    rho = state.rho.core(state.rho.current_space())
    if bool((rho == 0.0).any()):
        raise ValueError("rho contains zeros; the density update would divide by zero")
    return MpdataComputation(spec, state, geo, params, flux_op)


def flux_stage(op: str = "upwind") -> str:
    """Validates a flux operator name like mpdata.flux_stage (mpdata.py:255-262)."""
    if op not in FLUX_OPS:
        raise ValueError(f"flux operator must be one of {sorted(FLUX_OPS)}, got {op!r}")
    return op


class DivergenceComputation:
    """Single-stage cell divergence (mpdata.py:402-416)."""

    kind = "divergence"

    def __init__(self, patch, state, geo, weighted: bool, out: Field):
        self.patch, self.state, self.geo, self.weighted, self.out = patch, state, geo, weighted, out
        self.bindings = {"vn": state.vn, "div_out": out}
        if weighted:
            self.bindings["weights"] = geo.weights
        else:
            self.bindings.update(length=geo.edge_length, area=geo.cell_area)

    def fields(self):
        return list(self.bindings.values())

    def stage_updates(self) -> dict:
        name = "div_weighted" if self.weighted else "div_simple"
        return {name: 2 * self.patch.rows * self.patch.cols * self.out.meta.levels}

    def total_updates(self) -> int:
        return sum(self.stage_updates().values())


def build_divergence(spec: PatchSpec, state: StateFields, geo: GeometryFields, weighted: bool,
                     out: Field) -> DivergenceComputation:
    if out.meta.location is not _C or out.meta.levels != spec.levels:
        raise ValueError("div_out must be a cell field with the patch's levels")
    return DivergenceComputation(spec, state, geo, weighted, out)


def init_preset(field: Field, preset: str, seed: int = 0) -> None:
    """Fill a field's interior with a named preset and refresh its halo (mpdata.py:423-451)."""
    from .executors import halo_update

    spec = field.spec
    rows, cols = spec.rows, spec.cols
    core_shape = (rows, field.shape[1], cols, field.shape[3], field.shape[4])
    if preset == "uniform":
        values = np.ones(core_shape)
    elif preset == "gaussian-bump":
        sigma = max(rows, cols) / 6.0
        di = np.arange(rows)[:, None] - rows / 2.0
        dj = np.arange(cols)[None, :] - cols / 2.0
        bump = np.exp(-(di ** 2 + dj ** 2) / (2.0 * sigma ** 2))
        values = np.broadcast_to(bump[:, None, :, None, None], core_shape).copy()
    elif preset == "random":
        rng = np.random.default_rng([seed, zlib.crc32(field.name.encode())])
        values = rng.random(core_shape)
    else:
        raise ValueError(f"unknown preset {preset!r}")
    # a newer device copy raises StalenessError here, as in the reference (sync first)
    field.array("primary", "rw")[_interior(field)] = values
    halo_update(field)


def load_field_csv(field: Field, stream) -> None:
    """Load ``element,level,value`` rows into the interior (mpdata.py:454-485)."""
    from .executors import halo_update

    if field.has_extra:
        raise ValueError(f"field {field.name!r} has an extra axis; CSV load supports scalar "
                         "per-element values only")
    spec = field.spec
    arr = field.array("primary", "rw")
    h = spec.halo
    n = element_count(spec, field.meta.location)
    nk = field.shape[3]
    for lineno, row in enumerate(csv.reader(stream), start=1):
        if not row or row[0].lstrip().startswith("#"):
            continue
        if lineno == 1 and not row[0].strip().lstrip("-").isdigit():
            continue
        try:
            eid, level, value = int(row[0]), int(row[1]), float(row[2])
        except (ValueError, IndexError):
            raise ValueError(f"line {lineno}: expected 'element,level,value'")
        if not 0 <= eid < n:
            raise ValueError(f"line {lineno}: element {eid} out of range [0, {n})")
        if not 0 <= level < nk:
            raise ValueError(f"line {lineno}: level {level} out of range [0, {nk})")
        i, c, j = element_coord(spec, field.meta.location, eid)
        arr[i + h, c, j + h, level, 0] = value
    halo_update(field)


def total_mass(state: StateFields, geo: GeometryFields, which: str = "pd_in") -> float:
    """Density integrated over dual volumes and levels, reduced on the device."""
    import torch

    pd = getattr(state, which)
    grid = device_grid(pd.spec)
    p, d = pd.ensure_device(), geo.dual_volumes.ensure_device()
    work = torch.empty(1025, dtype=torch.float64, device=grid.device)
    _lib.call("tsg_total_mass", grid.handle, _lib.ptr(p), _lib.ptr(d), _lib.ptr(work[:1024]),
              _lib.ptr(work[1024:]), _lib.stream_handle())
    return float(work[1024].item())
