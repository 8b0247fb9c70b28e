"""Patch geometry: location types, the periodic parallelogram patch, canonical ids.

Mirrors the public names of ``tristencil.topology`` (topology.py:27-109) so
callers switch by changing the import.  A patch is a doubly periodic
parallelogram of ``rows x cols`` diamonds; per diamond there is 1 vertex,
2 cells (colour 0 = down, 1 = up) and 3 edges (0 horizontal, 1 diagonal,
2 vertical).  Canonical id: ``(row * colors + color) * cols + col``.

On the device the same (row, colour, column) indexing is the storage order
(include/tsg.h), so a canonical id is also the structured storage order.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass

import numpy as np


class LocationType(enum.Enum):
    VERTICES = "vertices"
    CELLS = "cells"
    EDGES = "edges"

    @property
    def colors(self) -> int:
        return {"vertices": 1, "cells": 2, "edges": 3}[self.value]

    @property
    def code(self) -> int:
        """Location code of the C ABI (include/tsg.h: 0 = V, 1 = C, 2 = E)."""
        return {"vertices": 0, "cells": 1, "edges": 2}[self.value]


def as_location(loc) -> LocationType:
    """Accept our enum, the reference's enum (by ``.value``) or a name."""
    if isinstance(loc, LocationType):
        return loc
    if isinstance(loc, (int, np.integer)) and not isinstance(loc, bool):
        return (LocationType.VERTICES, LocationType.CELLS, LocationType.EDGES)[int(loc)]
    return LocationType(getattr(loc, "value", loc))


@dataclass(frozen=True)
class PatchSpec:
    """Dimensions of one periodic parallelogram patch (topology.py:44-83)."""

    rows: int
    cols: int
    levels: int
    halo: int = 1

    def __post_init__(self):
        for name in ("rows", "cols", "levels", "halo"):
            value = getattr(self, name)
            if isinstance(value, bool) or not isinstance(value, (int, np.integer)):
                raise ValueError(f"{name} must be an integer, got {value!r}")
        if self.rows < 2 or self.cols < 2:
            raise ValueError(f"rows and cols must each be >= 2, got {self.rows}x{self.cols}")
        if self.levels < 1:
            raise ValueError(f"levels must be >= 1, got {self.levels}")
        if self.halo < 1:
            raise ValueError(f"halo must be >= 1, got {self.halo}")
        if self.halo > min(self.rows, self.cols):
            raise ValueError(f"halo {self.halo} exceeds patch extent {self.rows}x{self.cols}; "
                             "periodic wrap would alias")

    @property
    def diamonds(self) -> int:
        return self.rows * self.cols

    def wrap(self, i: int, j: int) -> tuple[int, int]:
        return i % self.rows, j % self.cols


def element_count(spec: PatchSpec, loc) -> int:
    return spec.diamonds * as_location(loc).colors


def element_id(spec: PatchSpec, loc, i: int, c: int, j: int) -> int:
    loc = as_location(loc)
    if not 0 <= c < loc.colors:
        raise ValueError(f"color {c} out of range for {loc.value} (0..{loc.colors - 1})")
    i, j = spec.wrap(i, j)
    return (i * loc.colors + c) * spec.cols + j


def element_coord(spec: PatchSpec, loc, eid: int) -> tuple[int, int, int]:
    loc = as_location(loc)
    n = element_count(spec, loc)
    if not 0 <= eid < n:
        raise ValueError(f"element id {eid} out of range for {loc.value} (0..{n - 1})")
    rest, j = divmod(eid, spec.cols)
    i, c = divmod(rest, loc.colors)
    return i, c, j
