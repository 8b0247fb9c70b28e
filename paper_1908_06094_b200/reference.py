"""GPU drop-in for ``tristencil.reference`` (reference.py:1-160): the flat, table-driven
formulation of the transport step and its stages, over ``[element, level]`` arrays in any
element numbering, with the reference's function names, argument order and errors.

Each function runs one CUDA kernel of ``libtsg.so`` (``tsg_flat_*``,
``tsg_transport_indirect``, ``tsg_neighbor_reduce_indirect``) with the reference's
operation order, so results are bitwise equal to it.  numpy inputs return numpy outputs
(host <-> device copies included); CUDA tensors stay on the device.  A one-dimensional
data array (no level axis) is treated as one level, as numpy broadcasting does there.
Tables are checked for ids outside ``[0, n)`` (IndexError) before any launch: the
kernels gather without bounds checks where numpy would raise.
"""

from __future__ import annotations

from . import _lib
from .flat import _FLUX_CODE, _dev
from .flat import transport_step as transport_step  # reference.py:93-116
from .kernels import check_ids

__all__ = ["upwind_flux", "centred_flux", "upwind_fluz", "flux_divergence", "advance_density",
           "transport_step", "cell_divergence", "neighbor_sum", "neighbor_sum_scaled"]


def _levels(t):
    """(tensor as [n, levels], original shape) -- 1-D arrays are one level."""
    if t.ndim == 1:
        return t.reshape(-1, 1), tuple(t.shape)
    if t.ndim != 2:
        raise ValueError(f"expected an [element, level] array, got shape {tuple(t.shape)}")
    return t, tuple(t.shape)


def _table(table, width=None, what="table"):
    import torch

    t, _ = _dev(getattr(table, "ids", table), torch.int64)
    if t.ndim != 2 or (width is not None and t.shape[1] != width):
        want = f"(n, {width})" if width is not None else "(n, width)"
        raise ValueError(f"{what} must be {want}, got {tuple(t.shape)}")
    return t


def _back(t, shape, on_dev):
    t = t.reshape(shape)
    return t if on_dev else t.cpu().numpy()


def _edge_flux(e2v, vn, pd, op):
    import torch

    vn_t, on_dev = _dev(vn, torch.float64)
    pd_t, _ = _dev(pd, torch.float64)
    v2, shape = _levels(vn_t)
    p2, _ = _levels(pd_t)
    if p2.shape[1] != v2.shape[1]:
        raise ValueError(f"pd levels {p2.shape[1]} do not match vn levels {v2.shape[1]}")
    t = _table(e2v, 2, "e2v")
    if t.shape[0] != v2.shape[0]:
        raise ValueError(f"e2v has {t.shape[0]} rows for {v2.shape[0]} edges")
    check_ids(t, p2.shape[0], "e2v")
    out = torch.empty_like(v2)
    _lib.call("tsg_flat_flux", _lib.ptr(t), _lib.ptr(p2), _lib.ptr(v2), v2.shape[0], v2.shape[1],
              _FLUX_CODE[op], _lib.ptr(out), _lib.stream_handle())
    return _back(out, shape, on_dev)


def upwind_flux(e2v, vn, pd):
    """Donor-cell edge flux: the upwind endpoint supplies the density (reference.py:18-26)."""
    return _edge_flux(e2v, vn, pd, "upwind")


def centred_flux(e2v, vn, pd):
    """Arithmetic-mean edge flux (reference.py:29-35)."""
    return _edge_flux(e2v, vn, pd, "centred")


def upwind_fluz(wn, pd, pivbz: float):
    """Vertical interface flux with scaled-copy boundaries (reference.py:38-60)."""
    import torch

    pd_t, on_dev = _dev(pd, torch.float64)
    wn_t, _ = _dev(wn, torch.float64)
    n, levels = pd_t.shape if pd_t.ndim == 2 else (pd_t.shape[0], 1)
    if levels < 2:
        raise ValueError(f"need at least 2 levels, got {levels}")
    if tuple(wn_t.shape) != (n, levels + 1):
        raise ValueError(f"wn must be staggered: expected {(n, levels + 1)}, got {tuple(wn_t.shape)}")
    out = torch.empty_like(wn_t)
    _lib.call("tsg_flat_fluz", _lib.ptr(pd_t), _lib.ptr(wn_t), n, levels, float(pivbz), _lib.ptr(out),
              _lib.stream_handle())
    return out if on_dev else out.cpu().numpy()


def flux_divergence(v2e, signs, dual_volumes, flux, fluz):
    """Signed flux sum per dual volume, horizontal then vertical (reference.py:63-79)."""
    import torch

    fz, on_dev = _dev(fluz, torch.float64)
    if fz.ndim != 2 or fz.shape[1] < 2:
        raise ValueError(f"fluz must be (n, levels + 1), got {tuple(fz.shape)}")
    n, levels = fz.shape[0], fz.shape[1] - 1
    fl, _ = _dev(flux, torch.float64)
    fl, _ = _levels(fl)
    if fl.shape[1] != levels:
        raise ValueError(f"flux levels {fl.shape[1]} do not match fluz levels {levels}")
    t = _table(v2e, what="v2e")
    if t.shape[0] != n:
        raise ValueError(f"v2e has {t.shape[0]} rows for {n} vertices")
    sg, _ = _dev(signs, torch.float64)
    if tuple(sg.shape) != tuple(t.shape):
        raise ValueError(f"signs must be {tuple(t.shape)}, got {tuple(sg.shape)}")
    du, _ = _dev(dual_volumes, torch.float64)
    du = du.reshape(-1)
    if du.numel() != n:
        raise ValueError(f"dual_volumes must hold {n} values, got {du.numel()}")
    check_ids(t, fl.shape[0], "v2e")
    out = torch.empty((n, levels), dtype=torch.float64, device=fz.device)
    _lib.call("tsg_flat_divergence", _lib.ptr(t), t.shape[1], _lib.ptr(sg), _lib.ptr(du), _lib.ptr(fl),
              _lib.ptr(fz), n, levels, _lib.ptr(out), _lib.stream_handle())
    return out if on_dev else out.cpu().numpy()


def advance_density(pd, div, rho, dt: float):
    """Explicit Euler: density minus dt times divergence over rho (reference.py:82-90)."""
    import torch

    pd_t, on_dev = _dev(pd, torch.float64)
    dv, _ = _dev(div, torch.float64)
    rh, _ = _dev(rho, torch.float64)
    if not (tuple(pd_t.shape) == tuple(dv.shape) == tuple(rh.shape)):
        raise ValueError(f"pd, div and rho shapes differ: {tuple(pd_t.shape)}, {tuple(dv.shape)}, "
                         f"{tuple(rh.shape)}")
    out = torch.empty_like(pd_t)
    _lib.call("tsg_flat_advance", _lib.ptr(pd_t), _lib.ptr(dv), _lib.ptr(rh), pd_t.numel(), float(dt),
              _lib.ptr(out), _lib.stream_handle())
    return out if on_dev else out.cpu().numpy()


def cell_divergence(c2e, vn, edge_length, cell_area):
    """Per-cell divergence: length-weighted normal velocities over the area
    (reference.py:119-134)."""
    import torch

    vn_t, on_dev = _dev(vn, torch.float64)
    v2, shape = _levels(vn_t)
    t = _table(c2e, what="c2e")
    ln, _ = _dev(edge_length, torch.float64)
    ar, _ = _dev(cell_area, torch.float64)
    ln, ar = ln.reshape(-1), ar.reshape(-1)
    if ln.numel() != v2.shape[0]:
        raise ValueError(f"edge_length must hold one value per edge ({v2.shape[0]}), got {ln.numel()}")
    if ar.numel() != t.shape[0]:
        raise ValueError(f"cell_area must hold one value per cell ({t.shape[0]}), got {ar.numel()}")
    check_ids(t, v2.shape[0], "c2e")
    out = torch.empty((t.shape[0], v2.shape[1]), dtype=torch.float64, device=v2.device)
    _lib.call("tsg_flat_cell_divergence", _lib.ptr(t), t.shape[1], _lib.ptr(v2), _lib.ptr(ln), _lib.ptr(ar),
              t.shape[0], v2.shape[1], _lib.ptr(out), _lib.stream_handle())
    return _back(out, (t.shape[0],) + shape[1:], on_dev)


def _neighbor(table, a, fac):
    import torch

    a_t, on_dev = _dev(a, torch.float64)
    a2, shape = _levels(a_t)
    t = _table(table, what="neighbour table")
    check_ids(t, a2.shape[0], "neighbour table")
    fv = None
    if fac is not None:
        fv, _ = _dev(fac, torch.float64)
        fv = fv.reshape(-1)
        if fv.numel() != t.shape[0]:
            raise ValueError("fac must hold one factor per table row")
    out = torch.zeros((t.shape[0], a2.shape[1]), dtype=torch.float64, device=a2.device)
    if t.shape[1] == 0:  # an empty neighbourhood sums to 0.0 (times fac)
        if fv is not None:
            out *= fv.reshape(-1, 1)
        return _back(out, (t.shape[0],) + shape[1:], on_dev)
    _lib.call("tsg_neighbor_reduce_indirect", _lib.ptr(t), t.shape[0], t.shape[1], a2.shape[1],
              _lib.ptr(a2), _lib.ptr(fv), _lib.ptr(out), _lib.stream_handle())
    return _back(out, (t.shape[0],) + shape[1:], on_dev)


def neighbor_sum(table, a):
    """Plain neighbourhood sum in table order, slot 0 first (reference.py:137-145)."""
    return _neighbor(table, a, None)


def neighbor_sum_scaled(table, a, fac):
    """Neighbourhood sum times a per-element factor (reference.py:148-157)."""
    return _neighbor(table, a, fac)
