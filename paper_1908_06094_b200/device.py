"""Device plumbing: grid handles, structured device fields, streams.

PyTorch provides device memory and streams only; all compute is in libtsg.so.
A :class:`DeviceGrid` wraps the C ABI's opaque ``tsg_grid`` (include/tsg.h)
and allocates structured fields in the device layout
``[rows+2][colors][cols+2][pitch(inner)]`` (level innermost, one-ring halo).
"""

from __future__ import annotations

import ctypes

import torch

from . import _lib
from .topology import PatchSpec, as_location

PERIODIC_ROWS = 1
PERIODIC_COLS = 2


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1908_06094_b200 computes on a CUDA device (sm_100a); "
                           "no GPU is visible and there is no CPU fallback")
    _lib.lib()
    return torch.device("cuda", torch.cuda.current_device())


def inner_pitch(inner: int) -> int:
    """Padded innermost extent (tsg_inner_pitch): 1 stays 1, even below 64, else a multiple of 16."""
    if inner <= 1:
        return 1
    return (inner + 1) // 2 * 2 if inner < 64 else (inner + 15) // 16 * 16


class DeviceGrid:
    """Owner of one ``tsg_grid`` handle: a (strip of a) patch on the current device."""

    def __init__(self, rows: int, cols: int, levels: int, flags: int = PERIODIC_ROWS | PERIODIC_COLS,
                 row0: int = 0, global_rows: int | None = None):
        require_cuda()
        handle = ctypes.c_void_p()
        _lib.call("tsg_grid_create", rows, cols, levels, flags, ctypes.byref(handle))
        self.handle = handle
        self.rows, self.cols, self.levels, self.flags = rows, cols, levels, flags
        self.device = torch.device("cuda", torch.cuda.current_device())
        if global_rows is not None:
            _lib.call("tsg_grid_set_origin", handle, row0, global_rows)
        self.row0 = row0
        self.global_rows = global_rows if global_rows is not None else rows

    @classmethod
    def for_spec(cls, spec: PatchSpec) -> "DeviceGrid":
        return cls(spec.rows, spec.cols, spec.levels)

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value and _lib._lib is not None:
            _lib._lib.tsg_grid_destroy(h)
            self.handle = None

    def field_shape(self, loc, inner: int) -> tuple[int, int, int, int]:
        loc = as_location(loc)
        return (self.rows + 2, loc.colors, self.cols + 2, inner_pitch(inner))

    def empty(self, loc, inner: int) -> torch.Tensor:
        """A zeroed structured field (padding stays zero)."""
        return torch.zeros(self.field_shape(loc, inner), dtype=torch.float64, device=self.device)
