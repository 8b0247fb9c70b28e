"""The nine structured neighbour relations and their flat tables (mirrors
tristencil.connectivity, connectivity.py:36-205).

``OFFSET_TABLES`` is the frozen canonical data: per source colour an ordered
list of ``(drow, target colour, dcol)``; the slot order fixes every
floating-point summation order downstream.  The same table is compiled into
the device constant ``c_offsets`` (csrc/tsg_offsets.cuh); the structured
kernels never materialise neighbour tables.

Flat tables (for the indirect / Atlas-style path and for callers) and the
edge-orientation signs are generated on the device by ``tsg_build_neighbor_table``
and ``tsg_edge_signs`` and returned as numpy arrays (``as_tensor=True`` keeps
them on the device).
"""

from __future__ import annotations

import csv
from dataclasses import dataclass

import numpy as np

from .topology import LocationType, PatchSpec, as_location, element_count

_V, _C, _E = LocationType.VERTICES, LocationType.CELLS, LocationType.EDGES

OFFSET_TABLES = {
    (_E, _V): (((0, 0, 0), (0, 0, 1)), ((0, 0, 0), (1, 0, 1)), ((0, 0, 0), (1, 0, 0))),
    (_E, _C): (((0, 0, 0), (-1, 1, 0)), ((0, 0, 0), (0, 1, 0)), ((0, 1, 0), (0, 0, -1))),
    (_E, _E): (((0, 1, 0), (0, 2, 1), (-1, 2, 0), (-1, 1, 0)),
               ((0, 0, 0), (0, 2, 1), (0, 2, 0), (1, 0, 0)),
               ((0, 1, 0), (1, 0, 0), (0, 0, -1), (0, 1, -1))),
    (_C, _V): (((0, 0, 0), (0, 0, 1), (1, 0, 1)), ((0, 0, 0), (1, 0, 0), (1, 0, 1))),
    (_C, _E): (((0, 0, 0), (0, 1, 0), (0, 2, 1)), ((0, 2, 0), (0, 1, 0), (1, 0, 0))),
    (_C, _C): (((0, 1, 0), (-1, 1, 0), (0, 1, 1)), ((0, 0, 0), (0, 0, -1), (1, 0, 0))),
    (_V, _V): (((0, 0, 1), (1, 0, 1), (1, 0, 0), (0, 0, -1), (-1, 0, -1), (-1, 0, 0)),),
    (_V, _E): (((0, 0, 0), (0, 1, 0), (0, 2, 0), (0, 0, -1), (-1, 1, -1), (-1, 2, 0)),),
    (_V, _C): (((0, 0, 0), (0, 1, 0), (0, 0, -1), (-1, 1, -1), (-1, 0, -1), (-1, 1, 0)),),
}


@dataclass(frozen=True)
class StructuredOffsets:
    from_loc: LocationType
    to_loc: LocationType
    color: int
    entries: tuple

    def __len__(self) -> int:
        return len(self.entries)


def _table(from_loc, to_loc):
    key = (as_location(from_loc), as_location(to_loc))
    try:
        return OFFSET_TABLES[key]
    except KeyError:
        raise ValueError(f"no structured relation {key[0].value} -> {key[1].value}") from None


def neighbor_len(from_loc, to_loc) -> int:
    return len(_table(from_loc, to_loc)[0])


def structured_offsets(from_loc, to_loc, color: int) -> StructuredOffsets:
    table = _table(from_loc, to_loc)
    f, t = as_location(from_loc), as_location(to_loc)
    if not 0 <= color < f.colors:
        raise ValueError(f"color {color} out of range for {f.value} (0..{f.colors - 1})")
    return StructuredOffsets(f, t, color, table[color])


@dataclass(frozen=True)
class NeighborTable:
    """Flat (n_from, width) rank table of one relation (connectivity.py:110-127)."""

    from_loc: LocationType
    to_loc: LocationType
    ids: object  # numpy int64 array (or a CUDA tensor when built with as_tensor=True)

    def __post_init__(self):
        if self.ids.ndim != 2 or self.ids.shape[1] != neighbor_len(self.from_loc, self.to_loc):
            raise ValueError(f"bad neighbor table shape {tuple(self.ids.shape)}")


def build_neighbor_table(spec: PatchSpec, from_loc, to_loc, perm_from=None, perm_to=None,
                         as_tensor: bool = False) -> NeighborTable:
    """One relation as a flat table under optional numberings, built on the device."""
    import torch

    from . import _lib
    from .device import require_cuda

    f, t = as_location(from_loc), as_location(to_loc)
    width = neighbor_len(f, t)
    n_from, n_to = element_count(spec, f), element_count(spec, t)
    if perm_from is not None and len(perm_from) != n_from:
        raise ValueError(f"perm_from sized {len(perm_from)}, expected {n_from} {f.value}")
    if perm_to is not None and len(perm_to) != n_to:
        raise ValueError(f"perm_to sized {len(perm_to)}, expected {n_to} {t.value}")
    dev = require_cuda()
    inv = None if perm_from is None else torch.as_tensor(perm_from.inverse, device=dev)
    fwd = None if perm_to is None else torch.as_tensor(perm_to.forward, device=dev)
    out = torch.empty((n_from, width), dtype=torch.int64, device=dev)
    _lib.call("tsg_build_neighbor_table", spec.rows, spec.cols, f.code, t.code, _lib.ptr(inv),
              _lib.ptr(fwd), _lib.ptr(out), _lib.stream_handle())
    return NeighborTable(f, t, out if as_tensor else out.cpu().numpy())


def edge_signs_table(spec: PatchSpec, as_tensor: bool = False):
    """(n_vertices, 6) orientation signs, +1 where the vertex is the edge's lower id."""
    import torch

    from . import _lib
    from .device import require_cuda

    dev = require_cuda()
    out = torch.empty((spec.rows * spec.cols, 6), dtype=torch.float64, device=dev)
    _lib.call("tsg_edge_signs", spec.rows, spec.cols, _lib.ptr(out), _lib.stream_handle())
    return out if as_tensor else out.cpu().numpy()


def dump_tables(spec: PatchSpec, stream) -> None:
    """All nine tables as CSV rows (connectivity.py:197-205)."""
    writer = csv.writer(stream)
    writer.writerow(["from_loc", "to_loc", "element", "slot", "neighbor"])
    for f, t in sorted(OFFSET_TABLES, key=lambda p: (p[0].value, p[1].value)):
        ids = build_neighbor_table(spec, f, t).ids
        for eid, row in enumerate(ids.tolist()):
            for slot, nid in enumerate(row):
                writer.writerow([f.value, t.value, eid, slot, nid])


def offset_array() -> np.ndarray:
    """OFFSET_TABLES as a dense int8 [9][3][6][3] array in the device constant's order."""
    arr = np.zeros((9, 3, 6, 3), dtype=np.int8)
    for (f, t), per_color in OFFSET_TABLES.items():
        for c, entries in enumerate(per_color):
            for s, e in enumerate(entries):
                arr[f.code * 3 + t.code, c, s] = e
    return arr
