"""Location-typed fields with a host ("primary") and a device ("mirror") space.

Mirrors tristencil.storage (storage.py:27-376).  In the reference the
"mirror" buffer is an explicit stand-in for device memory; here
it IS device memory: a CUDA tensor in the structured layout of
include/tsg.h (``[rows+2][colors][cols+2][pitch]``, level innermost).

* ``primary`` keeps the reference's host layout (LayoutSpec / LinearLayout)
  so host views, offsets and ``core()`` copies behave as before.
* ``sync(field, "mirror")`` uploads the raw host buffer and reorders it on the
  GPU (``tsg_pack_strided``); ``sync(field, "primary")`` reorders on the GPU
  (``tsg_unpack_strided``, halo cells as periodic images) and downloads.
* Staleness / divergence contracts are the reference's: reading a space while
  the other holds newer data raises :class:`StalenessError`; syncing when both
  were written raises :class:`DivergenceError`.

The reference's per-element traffic counters (a CPU instrumentation model) are
replaced by their closed form: every run records on its fields what those
counters would hold (``Field.counters``, filled by traffic.record_run and read
through ``RunStats.traffic()``); the GPU's own bytes are measured with ncu
(profiles/).

Host buffers are allocated in page-locked memory when a GPU is present, so the
primary <-> mirror copies of ``sync`` are DMA transfers straight from / into them.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .layouts import AXES, LayoutSpec, LinearLayout
from .topology import PatchSpec, as_location
from .traffic import TrafficReport, TrafficRow  # noqa: F401  (storage.py:410-479 of the reference)

SPACES = ("primary", "mirror")


class StorageError(RuntimeError):
    pass


class StalenessError(StorageError):
    """A space was read while the opposite space held newer data."""


class DivergenceError(StorageError):
    """Both spaces were written since the last sync; neither may win."""


@dataclass(frozen=True)
class Selector:
    row: bool = True
    color: bool = True
    column: bool = True
    level: bool = True
    extra: bool = False


@dataclass(frozen=True)
class FieldMeta:
    name: str
    location: object
    selector: Selector
    levels: int
    extra_len: int
    layout: LayoutSpec


_GRIDS: dict = {}


def device_grid(spec: PatchSpec):
    """The shared DeviceGrid of a patch on the current device (one tsg_grid per
    (rows, cols, levels, device): a handle binds to the device it was created on)."""
    import torch

    from .device import DeviceGrid, require_cuda

    require_cuda()
    key = (spec.rows, spec.cols, spec.levels, torch.cuda.current_device())
    g = _GRIDS.get(key)
    if g is None:
        g = _GRIDS[key] = DeviceGrid.for_spec(spec)
    return g


def _host_zeros(n: int) -> np.ndarray:
    """A zeroed float64 host buffer, page-locked when a GPU is present (the torch tensor
    owning the memory stays alive as the array's base)."""
    try:
        import torch

        if torch.cuda.is_available():
            return torch.zeros(n, dtype=torch.float64, pin_memory=True).numpy()
    except (ImportError, RuntimeError):
        pass
    return np.zeros(n, dtype=np.float64)


class Field:
    """One storage with its host buffer and device mirror (storage.py:71-285)."""

    def __init__(self, spec: PatchSpec, meta: FieldMeta):
        self.spec = spec
        self.meta = meta
        sizes = {
            "row": spec.rows + 2 * spec.halo,
            "color": meta.location.colors,
            "column": spec.cols + 2 * spec.halo,
            "level": meta.levels if meta.selector.level else 1,
            "extra": meta.extra_len if meta.selector.extra else 1,
        }
        self.linear = LinearLayout(meta.layout, sizes, spec.halo)
        self.shape = tuple(sizes[a] for a in AXES)
        self._primary = None  # numpy, allocated on first use (zeros)
        self._mirror = None   # torch CUDA tensor, allocated on first use (zeros)
        self.dirty = {"primary": False, "mirror": False}
        self.sync_count = 0
        # phase -> [distinct_reads, distinct_writes, raw_reads, raw_writes] (traffic.py)
        self.counters = {}

    # -- identity ---------------------------------------------------------------------
    @property
    def name(self) -> str:
        return self.meta.name

    @property
    def has_levels(self) -> bool:
        return self.meta.selector.level

    @property
    def has_extra(self) -> bool:
        return self.meta.selector.extra

    @property
    def inner(self) -> int:
        """Contiguous values per element on the device: levels, extra, or 1."""
        if self.has_levels and self.has_extra:
            raise ValueError(f"field {self.name!r}: level and extra axes together are not "
                             "supported on the device")
        if self.has_levels:
            return self.meta.levels
        return self.meta.extra_len if self.has_extra else 1

    @property
    def loc_code(self) -> int:
        return self.meta.location.code

    # -- buffers -----------------------------------------------------------------------
    def buffer(self, space: str):
        self._check_space(space)
        if space == "primary":
            if self._primary is None:
                self._primary = _host_zeros(self.linear.total)
            return self._primary
        if self._mirror is None:
            self._mirror = device_grid(self.spec).empty(self.meta.location, self.inner)
        return self._mirror

    def device(self):
        """The device tensor ([rows+2][colors][cols+2][pitch]); checks staleness."""
        self._check_stale("mirror")
        return self.buffer("mirror")

    def _logical(self, space: str):
        buf = self.buffer(space)
        if space == "primary":
            shape, strides = self.linear.view_shape_strides()
            return np.lib.stride_tricks.as_strided(
                buf[self.linear.front_pad:], shape=shape,
                strides=tuple(s * buf.itemsize for s in strides))
        import torch

        R, C, W, P = buf.shape
        lev = self.meta.levels if self.has_levels else 1
        ext = self.meta.extra_len if self.has_extra else 1
        sl = (P, 1, 0) if self.has_levels else (P, 0, 1)
        return torch.as_strided(buf, (R, C, W, lev, ext), (C * W * P, W * P, sl[0], sl[1], sl[2]))

    def array(self, space: str = "primary", mode: str = "r"):
        """Uncounted bulk view; 'rw' marks the space dirty (storage.py:130-145)."""
        self._check_stale(space)
        view = self._logical(space)
        if mode == "rw":
            self.dirty[space] = True
        elif mode == "r":
            if space == "primary":
                view = view.view()
                view.flags.writeable = False
        else:
            raise ValueError(f"mode must be 'r' or 'rw', got {mode!r}")
        return view

    def core(self, space: str = "primary"):
        """Copy of the interior (halo stripped)."""
        if space == "primary":
            h = self.spec.halo
            return self.array(space)[h:h + self.spec.rows, :, h:h + self.spec.cols].copy()
        full = self.array(space)
        return full[1:1 + self.spec.rows, :, 1:1 + self.spec.cols].clone()

    def current_space(self) -> str:
        """Where the newest data lives ('mirror' only when the device copy is newer)."""
        return "mirror" if self.dirty["mirror"] else "primary"

    # -- bookkeeping -------------------------------------------------------------------
    def _check_space(self, space: str) -> None:
        if space not in SPACES:
            raise ValueError(f"unknown space {space!r}, expected one of {SPACES}")

    def _check_stale(self, space: str) -> None:
        self._check_space(space)
        other = "mirror" if space == "primary" else "primary"
        if self.dirty[other]:
            raise StalenessError(f"field {self.name!r}: {space} is stale, {other} holds newer "
                                 "data; sync() first")

    def ensure_device(self):
        """Upload if the host copy is newer; return the device tensor."""
        if self.dirty["primary"]:
            sync(self, "mirror")
        return self.buffer("mirror")

    def mark_device_written(self) -> None:
        """A kernel overwrote the whole device copy (interior and halo)."""
        self.dirty["primary"] = False
        self.dirty["mirror"] = True


def make_storage(spec: PatchSpec, loc, name: str, selector: Selector | None = None,
                 extra_len: int = 0, levels: int | None = None,
                 layout: LayoutSpec | None = None) -> Field:
    """Allocate a field on one location type (storage.py:316-357)."""
    loc = as_location(loc)
    if selector is None:
        selector = Selector(extra=extra_len > 0)
    if loc.colors > 1 and not selector.color:
        raise ValueError(f"storage {name!r}: selector flag 'color' is required on {loc.value} "
                         "(multiple colors per diamond)")
    if not (selector.row and selector.column):
        flag = "row" if not selector.row else "column"
        raise ValueError(f"storage {name!r}: selector flag {flag!r} must be set")
    if selector.extra != (extra_len > 0):
        raise ValueError(f"storage {name!r}: selector flag 'extra' inconsistent with "
                         f"extra_len={extra_len}")
    if extra_len < 0:
        raise ValueError(f"storage {name!r}: extra_len must be >= 0")
    meta = FieldMeta(name=name, location=loc, selector=selector,
                     levels=spec.levels if levels is None else int(levels),
                     extra_len=extra_len, layout=layout if layout is not None else LayoutSpec())
    if meta.selector.level and meta.levels < 1:
        raise ValueError(f"storage {name!r}: levels must be >= 1")
    return Field(spec, meta)


def sync(field: Field, to_space: str) -> None:
    """Reconcile the two spaces by copying into ``to_space`` (storage.py:360-376)."""
    import torch

    from . import _lib

    field._check_space(to_space)
    src = "mirror" if to_space == "primary" else "primary"
    if field.dirty["primary"] and field.dirty["mirror"]:
        raise DivergenceError(f"field {field.name!r}: both spaces modified since last sync")
    if field.dirty[src]:
        grid = device_grid(field.spec)
        lay = field.linear.layout6()
        if not field.has_levels:
            lay[4] = 0  # the device inner axis runs along `extra` (or is a scalar)
        lay_p = lay.ctypes.data_as(_lib.ctypes.POINTER(_lib.ctypes.c_int64))
        host = torch.from_numpy(field.buffer("primary"))
        if to_space == "mirror":
            staging = host.to(grid.device, non_blocking=host.is_pinned())
            _lib.call("tsg_pack_strided", grid.handle, field.loc_code, field.inner,
                      _lib.ptr(staging), lay_p, field.spec.halo, _lib.ptr(field.buffer("mirror")),
                      _lib.stream_handle())
            torch.cuda.current_stream().synchronize()
        else:
            staging = torch.zeros(field.linear.total, dtype=torch.float64, device=grid.device)
            _lib.call("tsg_unpack_strided", grid.handle, field.loc_code, field.inner,
                      _lib.ptr(field.buffer("mirror")), lay_p, field.spec.halo, _lib.ptr(staging),
                      _lib.stream_handle())
            host.copy_(staging)  # straight into the (page-locked) host buffer
    field.dirty = {"primary": False, "mirror": False}
    field.sync_count += 1


def reset_counters(fields) -> None:
    """Clear the recorded traffic of ``fields`` (storage.py:380-382)."""
    for f in fields:
        f.counters.clear()


def plane_access_total(counts: dict, coefficients: dict) -> int:
    """Per-plane access model sum(count * (reads + writes)) (storage.py:470-479)."""
    missing = set(coefficients) - set(counts)
    if missing:
        raise ValueError(f"no element counts for groups {sorted(missing)}")
    return sum(counts[g] * (r + w) for g, (r, w) in coefficients.items())
