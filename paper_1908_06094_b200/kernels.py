"""Neighbour-reduction kernels: Table-1 indexing study and the 9-relation reduce.

Mirrors tristencil.kernels (kernels.py:27-155):

* direct (structured) access -- ``build_kernel`` / :func:`build_reduce` return a
  computation executed by :func:`executors.run_gpu` through
  ``tsg_neighbor_reduce`` (offset arithmetic on the (row, colour, column)
  layout, no tables);
* indirect access -- :func:`run_neighbor_sum` / :func:`run_neighbor_sum_scaled`
  gather through a flat int64 neighbour table in any numbering
  (``tsg_neighbor_reduce_indirect``);
* :func:`field_to_flat` / :func:`flat_to_field` convert between Fields and
  flat ``[element, level]`` arrays in any numbering; when the data lives on
  the device the reorder runs there (``tsg_unpack`` / ``tsg_pack``).

Both access methods fold neighbours in canonical slot order from 0.0
(``acc = a[nbr] + acc``), so results agree bitwise across numberings.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .layouts import Permutation
from .stencil import CompositionError
from .storage import Field, Selector, device_grid, make_storage
from .topology import LocationType, PatchSpec, as_location, element_count

_C = LocationType.CELLS


class ReduceComputation:
    """dst[from, k] = sum over canonical neighbours of src (times scale[from])."""

    kind = "reduce"

    def __init__(self, patch: PatchSpec, from_loc, to_loc, src: Field, dst: Field,
                 scale: Field | None = None, name: str = "reduce"):
        self.patch = patch
        self.from_loc, self.to_loc = as_location(from_loc), as_location(to_loc)
        if src.meta.location is not self.to_loc or dst.meta.location is not self.from_loc:
            raise CompositionError("src must live on to_loc and dst on from_loc")
        if src.inner != dst.inner:
            raise CompositionError("src and dst must have the same number of levels")
        if scale is not None and (scale.meta.location is not self.from_loc or scale.inner != 1):
            raise CompositionError("scale must be a 2-D field on from_loc")
        self.src, self.dst, self.scale, self.name = src, dst, scale, name
        self.bindings = {"a": src, "b": dst}
        if scale is not None:
            self.bindings["fac"] = scale

    def fields(self):
        return list(self.bindings.values())

    def stage_updates(self) -> dict:
        return {self.name: element_count(self.patch, self.from_loc) * self.dst.inner}

    def algorithmic_bytes(self) -> int:
        """(n_from + n_to) * K * 8 (+ n_from * 8 for the scale), SURVEY 8(d)."""
        nf = element_count(self.patch, self.from_loc)
        nt = element_count(self.patch, self.to_loc)
        return 8 * ((nf + nt) * self.dst.inner + (nf if self.scale is not None else 0))

    def total_updates(self) -> int:
        return sum(self.stage_updates().values())


def build_reduce(spec: PatchSpec, from_loc, to_loc, src: Field, dst: Field,
                 scale: Field | None = None) -> ReduceComputation:
    """Any of the nine relations through the structured reduce (stencil.py:404-408)."""
    return ReduceComputation(spec, from_loc, to_loc, src, dst, scale)


def make_kernel_fields(spec: PatchSpec, layout=None) -> dict:
    return {
        "a": make_storage(spec, _C, "a", layout=layout),
        "b": make_storage(spec, _C, "b", layout=layout),
        "fac": make_storage(spec, _C, "fac", Selector(level=False), layout=layout),
    }


def build_kernel(spec: PatchSpec, fields: dict, scaled: bool) -> ReduceComputation:
    """k1: b = sum_nbr a; k2: b = (sum_nbr a) * fac (kernels.py:70-76)."""
    name = "neighbor_sum_scaled" if scaled else "neighbor_sum"
    return ReduceComputation(spec, _C, _C, fields["a"], fields["b"],
                             fields["fac"] if scaled else None, name)


# ---------------------------------------------------------------------------
# indirect (table-driven) runners over flat arrays


def _as_device(x, dtype):
    import torch

    from .device import require_cuda

    dev = require_cuda()
    if isinstance(x, torch.Tensor):
        return x.to(device=dev, dtype=dtype).contiguous(), True
    return torch.as_tensor(np.ascontiguousarray(x), dtype=dtype, device=dev), False


def _indirect(table, a, fac):
    import torch

    ids = getattr(table, "ids", table)
    t, _ = _as_device(ids, torch.int64)
    av, on_dev = _as_device(a, torch.float64)
    if av.ndim != 2:
        raise ValueError("a must be (n_elements, levels)")
    if t.ndim != 2:
        raise ValueError("the neighbour table must be (n_rows, width)")
    check_ids(t, av.shape[0], "neighbour table")
    fv = None
    if fac is not None:
        fv, _ = _as_device(fac, torch.float64)
        fv = fv.reshape(-1)
        if fv.numel() != t.shape[0]:
            raise ValueError("fac must hold one factor per table row")
    out = torch.empty((t.shape[0], av.shape[1]), dtype=torch.float64, device=av.device)
    _lib.call("tsg_neighbor_reduce_indirect", _lib.ptr(t), t.shape[0], t.shape[1], av.shape[1],
              _lib.ptr(av), _lib.ptr(fv), _lib.ptr(out), _lib.stream_handle())
    return out if on_dev else out.cpu().numpy()


def check_ids(ids, n: int, what: str) -> None:
    """IndexError unless every id of a device index table lies in [0, n) -- the kernels
    gather without bounds checks, where numpy would raise (reference.py:137-145)."""
    if ids.numel() == 0:
        return
    lo, hi = (int(v) for v in torch_aminmax(ids))
    if lo < 0 or hi >= n:
        raise IndexError(f"{what}: index {lo if lo < 0 else hi} is out of bounds for {n} elements")


def torch_aminmax(t):
    import torch

    mm = torch.aminmax(t)
    return torch.stack([mm.min, mm.max]).cpu().tolist()


def run_neighbor_sum(table, a):
    """Flat indirect sweep (kernels.py:83-92); numpy in -> numpy out, CUDA tensor stays."""
    return _indirect(table, a, None)


def run_neighbor_sum_scaled(table, a, fac):
    return _indirect(table, a, fac)


def field_to_flat(field: Field, perm: Permutation | None = None):
    """Interior as (n_elements, levels) in canonical or rank order (kernels.py:107-117)."""
    if field.has_extra:
        raise ValueError(f"field {field.name!r} has an extra axis")
    if field.current_space() == "mirror":
        import torch

        grid = device_grid(field.spec)
        n = element_count(field.spec, field.meta.location)
        out = torch.empty((n, field.inner), dtype=torch.float64, device=grid.device)
        fwd = None if perm is None else torch.as_tensor(perm.forward, device=grid.device)
        _lib.call("tsg_unpack", grid.handle, field.loc_code, field.inner,
                  _lib.ptr(field.buffer("mirror")), _lib.ptr(fwd), _lib.ptr(out),
                  _lib.stream_handle())
        return out.cpu().numpy()
    core = field.core()
    flat = core[:, :, :, :, 0].reshape(-1, core.shape[3])
    return flat if perm is None else flat[perm.inverse]


def flat_to_field(values, field: Field, perm: Permutation | None = None) -> None:
    """Scatter (n_elements, levels) values into a field (kernels.py:120-127).

    CUDA-tensor input is reordered into the device copy by tsg_pack (halo
    images included); host input is written into the host copy.
    """
    import torch

    if isinstance(values, torch.Tensor) and values.is_cuda:
        grid = device_grid(field.spec)
        v = values.to(torch.float64).contiguous()
        fwd = None if perm is None else torch.as_tensor(perm.forward, device=grid.device)
        _lib.call("tsg_pack", grid.handle, field.loc_code, field.inner, _lib.ptr(v), _lib.ptr(fwd),
                  _lib.ptr(field.buffer("mirror")), _lib.stream_handle())
        field.mark_device_written()
        return
    spec = field.spec
    h = spec.halo
    canonical = values if perm is None else values[perm.forward]
    shaped = np.asarray(canonical).reshape(spec.rows, field.shape[1], spec.cols, field.shape[3])
    # a newer device copy is not silently dropped: array('primary', 'rw') raises
    # StalenessError as the reference does (storage.py:130-145); sync first
    field.array("primary", "rw")[h:h + spec.rows, :, h:h + spec.cols, :, 0] = shaped


def gather_groups(table, width: int, own_reads: int = 0) -> list:
    """Warp address groups of one indirect sweep over a neighbour table (kernels.py:137-155):
    per warp of ``width`` consecutive ranks one gather group per neighbour slot, then
    ``own_reads`` own-rank read groups and the own-rank write group."""
    if width < 1:
        raise ValueError(f"width must be >= 1, got {width}")
    ids = getattr(table, "ids", table)
    if hasattr(ids, "cpu"):
        ids = ids.cpu().numpy()
    ids = np.asarray(ids)
    groups = []
    for r0 in range(0, ids.shape[0], width):
        rows = ids[r0:r0 + width]
        chunk = np.arange(r0, r0 + rows.shape[0])
        groups.extend(rows[:, s].copy() for s in range(ids.shape[1]))
        groups.extend(chunk for _ in range(own_reads + 1))  # own reads, then the write
    return groups


def unpermute(values, perm: Permutation | None):
    """Rank-ordered rows back to canonical element order."""
    if perm is None:
        return values
    return values[perm.forward]
