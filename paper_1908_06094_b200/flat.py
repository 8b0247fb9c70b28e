"""Flat-array entry points with the reference oracle's signatures.

* :func:`transport_step` -- ``reference.transport_step`` (reference.py:93-116):
  flat ``[element, level]`` arrays and explicit neighbour tables in ANY
  numbering, executed by the table-driven ("indirect", Atlas-style) kernels
  ``tsg_transport_indirect``.
* :func:`neighbor_sum` / :func:`neighbor_sum_scaled` -- reference.py:137-157.
* :class:`StructuredStepper` -- the fast path for flat data: flat arrays (any
  numbering given as permutations) are reordered on the GPU into the
  structured (row, colour, column) layout (``tsg_pack``), advanced by the
  fused single-pass kernel (``tsg_mpdata_step``) and reordered back
  (``tsg_unpack``).  This is the "Atlas -> structured" drop-in of the
  north star; bench.py times it end to end from pinned host buffers.

numpy inputs return numpy outputs (host<->device copies included); CUDA
tensors stay on the device.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .device import DeviceGrid, require_cuda
from .topology import PatchSpec

_FLUX_CODE = {"upwind": 0, "centred": 1}


def _dev(x, dtype):
    import torch

    dev = require_cuda()
    if isinstance(x, torch.Tensor):
        return x.to(device=dev, dtype=dtype).contiguous(), x.is_cuda
    return torch.as_tensor(np.ascontiguousarray(x), dtype=dtype, device=dev), False


def transport_step(e2v, v2e, signs, dual_volumes, pd, vn, wn, rho, dt, pivbz, flux_op="upwind"):
    """One transport step over flat arrays; returns {'flux','fluz','div','pd_out'}."""
    import torch

    if flux_op not in _FLUX_CODE:
        raise ValueError(f"unknown flux operator {flux_op!r}")
    pd_t, on_dev = _dev(pd, torch.float64)
    n, levels = pd_t.shape
    if levels < 2:
        raise ValueError(f"need at least 2 levels, got {levels}")
    wn_t, _ = _dev(wn, torch.float64)
    if tuple(wn_t.shape) != (n, levels + 1):
        raise ValueError(f"wn must be staggered: expected {(n, levels + 1)}, got {tuple(wn_t.shape)}")
    e2v_t, _ = _dev(e2v, torch.int64)
    v2e_t, _ = _dev(v2e, torch.int64)
    sg_t, _ = _dev(signs, torch.float64)
    du_t, _ = _dev(dual_volumes, torch.float64)
    vn_t, _ = _dev(vn, torch.float64)
    rho_t, _ = _dev(rho, torch.float64)
    # the kernels index without bounds checks: validate every shape and id first, raising
    # what numpy raises in the reference for the same inputs (reference.py:93-116)
    if vn_t.ndim != 2 or vn_t.shape[1] != levels:
        raise ValueError(f"vn must be (n_edges, {levels}), got {tuple(vn_t.shape)}")
    ne = vn_t.shape[0]
    if tuple(rho_t.shape) != (n, levels):
        raise ValueError(f"rho must be {(n, levels)}, got {tuple(rho_t.shape)}")
    if tuple(e2v_t.shape) != (ne, 2) or tuple(v2e_t.shape) != (n, 6):
        raise ValueError("e2v must be (n_edges, 2) and v2e (n_vertices, 6)")
    if tuple(sg_t.shape) != (n, 6):
        raise ValueError(f"signs must be {(n, 6)}, got {tuple(sg_t.shape)}")
    if du_t.numel() != n:
        raise ValueError(f"dual_volumes must hold {n} values, got {du_t.numel()}")
    from .kernels import check_ids

    check_ids(e2v_t, n, "e2v")
    check_ids(v2e_t, ne, "v2e")
    out = {"flux": torch.empty((ne, levels), dtype=torch.float64, device=pd_t.device),
           "fluz": torch.empty((n, levels + 1), dtype=torch.float64, device=pd_t.device),
           "div": torch.empty((n, levels), dtype=torch.float64, device=pd_t.device),
           "pd_out": torch.empty((n, levels), dtype=torch.float64, device=pd_t.device)}
    _lib.call("tsg_transport_indirect", _lib.ptr(e2v_t), _lib.ptr(v2e_t), _lib.ptr(sg_t),
              _lib.ptr(du_t.reshape(-1)), _lib.ptr(pd_t), _lib.ptr(vn_t), _lib.ptr(wn_t),
              _lib.ptr(rho_t), n, ne, levels, float(dt), float(pivbz), _FLUX_CODE[flux_op],
              _lib.ptr(out["flux"]), _lib.ptr(out["fluz"]), _lib.ptr(out["div"]),
              _lib.ptr(out["pd_out"]), _lib.stream_handle())
    if on_dev:
        return out
    return {k: v.cpu().numpy() for k, v in out.items()}


def neighbor_sum(table, a):
    from .kernels import run_neighbor_sum

    return run_neighbor_sum(table, a)


def neighbor_sum_scaled(table, a, fac):
    from .kernels import run_neighbor_sum_scaled

    return run_neighbor_sum_scaled(table, a, fac)


class StructuredStepper:
    """Flat arrays in -> fused structured step -> flat arrays out, with resident buffers.

    ``perm_v`` / ``perm_e`` (layouts.Permutation or forward arrays) give the
    numbering of the flat vertex / edge arrays (None = structured numbering).
    Geometry (signs, dual) is uploaded once by :meth:`set_geometry`.
    """

    def __init__(self, spec: PatchSpec, perm_v=None, perm_e=None):
        import torch

        self.spec = spec
        self.grid = DeviceGrid.for_spec(spec)
        dev = self.grid.device
        K = spec.levels
        g = self.grid
        self.pd = g.empty(0, K)
        self.pd_out = g.empty(0, K)
        self.vn = g.empty(2, K)
        self.wn = g.empty(0, K + 1)
        self.rho = g.empty(0, K)
        self.signs = g.empty(0, 6)
        self.dual = g.empty(0, 1)

        def fwd(p):
            if p is None:
                return None
            f = getattr(p, "forward", p)
            return torch.as_tensor(np.asarray(f), dtype=torch.int64, device=dev)

        self.fwd_v, self.fwd_e = fwd(perm_v), fwd(perm_e)
        nv, ne = spec.rows * spec.cols, 3 * spec.rows * spec.cols
        self.in_bufs = {
            "pd": torch.empty((nv, K), dtype=torch.float64, device=dev),
            "vn": torch.empty((ne, K), dtype=torch.float64, device=dev),
            "wn": torch.empty((nv, K + 1), dtype=torch.float64, device=dev),
            "rho": torch.empty((nv, K), dtype=torch.float64, device=dev),
        }
        self.out_buf = torch.empty((nv, K), dtype=torch.float64, device=dev)

    def _pack(self, loc, inner, flat, fwd, field, stream):
        _lib.call("tsg_pack", self.grid.handle, loc, inner, _lib.ptr(flat), _lib.ptr(fwd),
                  _lib.ptr(field), _lib.stream_handle(stream))

    def set_geometry(self, signs, dual, stream=None):
        import torch

        sg, _ = _dev(signs, torch.float64)
        du, _ = _dev(dual, torch.float64)
        self._pack(0, 6, sg, self.fwd_v, self.signs, stream)
        self._pack(0, 1, du.reshape(-1, 1).contiguous(), self.fwd_v, self.dual, stream)

    def upload(self, pd, vn, wn, rho, stream=None):
        """Pinned host (or device) flat inputs -> structured device fields."""
        import torch

        src = {"pd": pd, "vn": vn, "wn": wn, "rho": rho}
        with torch.cuda.stream(stream if stream is not None else torch.cuda.current_stream()):
            for name, buf in self.in_bufs.items():
                x = src[name]
                if isinstance(x, np.ndarray):
                    x = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64))
                buf.copy_(x, non_blocking=True)
        K = self.spec.levels
        self._pack(0, K, self.in_bufs["pd"], self.fwd_v, self.pd, stream)
        self._pack(2, K, self.in_bufs["vn"], self.fwd_e, self.vn, stream)
        self._pack(0, K + 1, self.in_bufs["wn"], self.fwd_v, self.wn, stream)
        self._pack(0, K, self.in_bufs["rho"], self.fwd_v, self.rho, stream)

    def step(self, dt, pivbz, flux_op="upwind", stream=None):
        """Fused step on the resident fields: pd -> pd_out (halo images included)."""
        _lib.call("tsg_mpdata_step", self.grid.handle, _lib.ptr(self.pd), _lib.ptr(self.vn),
                  _lib.ptr(self.wn), _lib.ptr(self.rho), _lib.ptr(self.signs),
                  _lib.ptr(self.dual), _lib.ptr(self.pd_out), float(dt), float(pivbz),
                  _FLUX_CODE[flux_op], _lib.stream_handle(stream))

    def step_unfused(self, dt, pivbz, flux_op="upwind", stream=None):
        """Four-kernel step materialising flux / fluz / divvd (run_naive analogue)."""
        g, K = self.grid, self.spec.levels
        if not hasattr(self, "flux"):
            self.flux, self.fluz, self.divvd = g.empty(2, K), g.empty(0, K + 1), g.empty(0, K)
        _lib.call("tsg_mpdata_step_unfused", g.handle, _lib.ptr(self.pd), _lib.ptr(self.vn),
                  _lib.ptr(self.wn), _lib.ptr(self.rho), _lib.ptr(self.signs),
                  _lib.ptr(self.dual), _lib.ptr(self.flux), _lib.ptr(self.fluz),
                  _lib.ptr(self.divvd), _lib.ptr(self.pd_out), float(dt), float(pivbz),
                  _FLUX_CODE[flux_op], _lib.stream_handle(stream))

    def fetch(self, name, stream=None):
        """Any resident structured field as a flat numpy array (canonical numbering)."""
        import torch

        field = getattr(self, name)
        loc = 2 if name in ("vn", "flux") else 0
        inner = {"wn": self.spec.levels + 1, "fluz": self.spec.levels + 1, "signs": 6,
                 "dual": 1}.get(name, self.spec.levels)
        n = (3 if loc == 2 else 1) * self.spec.rows * self.spec.cols
        out = torch.empty((n, inner), dtype=torch.float64, device=self.grid.device)
        _lib.call("tsg_unpack", self.grid.handle, loc, inner, _lib.ptr(field), None,
                  _lib.ptr(out), _lib.stream_handle(stream))
        return out.cpu().numpy()

    def swap(self):
        """Time loop: the new density becomes the next step's input (no copy)."""
        self.pd, self.pd_out = self.pd_out, self.pd

    def run(self, steps, dt, pivbz, flux_op="upwind", stream=None):
        """``steps`` fused steps with fixed vn / wn / rho (bench.py:398-403), ping-ponging
        the two density buffers on the device (tsg_mpdata_run).  Afterwards ``pd_out``
        holds the newest density and ``pd`` the state before the last step, exactly as
        after ``steps`` calls of step(); swap()."""
        steps = int(steps)
        if steps < 0:
            raise ValueError(f"steps must be >= 0, got {steps}")
        _lib.call("tsg_mpdata_run", self.grid.handle, _lib.ptr(self.pd), _lib.ptr(self.pd_out),
                  _lib.ptr(self.vn), _lib.ptr(self.wn), _lib.ptr(self.rho), _lib.ptr(self.signs),
                  _lib.ptr(self.dual), float(dt), float(pivbz), _FLUX_CODE[flux_op], steps,
                  _lib.stream_handle(stream))
        if steps and steps % 2 == 0:
            self.swap()  # the newest density landed in the input buffer

    def download(self, out=None, stream=None):
        """Structured pd_out -> flat (numbering of perm_v) -> host ``out`` (pinned) or numpy."""
        _lib.call("tsg_unpack", self.grid.handle, 0, self.spec.levels, _lib.ptr(self.pd_out),
                  _lib.ptr(self.fwd_v), _lib.ptr(self.out_buf), _lib.stream_handle(stream))
        if out is None:
            return self.out_buf.cpu().numpy()
        out.copy_(self.out_buf, non_blocking=True)
        return out

    def run_pipelined(self, inputs, outputs, dt, pivbz, flux_op="upwind"):
        """Many independent host-fed steps with copies overlapped (PCIe is full duplex).

        ``inputs[n]`` = (pd, vn, wn, rho) pinned host tensors of step n, ``outputs[n]`` a
        pinned host tensor receiving that step's pd_out.  A ``None`` entry keeps that field's
        resident value (the reference's time loop holds vn / wn / rho fixed, bench.py:398-403:
        ``(pd, None, None, None)`` moves only the state).  Three streams: the H2D copy of
        step n+1 runs while step n is reordered / advanced on the GPU and step n-1's result
        is copied back; flat staging buffers are double-buffered and guarded by events.
        Returns (start_event, end_event) bracketing all the work.
        """
        import torch

        K = self.spec.levels
        if not hasattr(self, "_pipe"):
            dev = self.grid.device
            self._pipe = {
                "h2d": torch.cuda.Stream(), "comp": torch.cuda.Stream(), "d2h": torch.cuda.Stream(),
                "in": [{k: torch.empty_like(v) for k, v in self.in_bufs.items()} for _ in range(2)],
                "out": [torch.empty_like(self.out_buf) for _ in range(2)],
            }
        P = self._pipe
        ev = lambda: torch.cuda.Event(enable_timing=False)  # noqa: E731
        # the private streams start after everything already queued on the caller's stream
        # (set_geometry / upload / the resident fields' zero fill) ...
        cur = torch.cuda.current_stream()
        for st in (P["h2d"], P["comp"], P["d2h"]):
            st.wait_stream(cur)
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        start.record(P["h2d"])
        packed = [None, None]    # staging set b free again (its pack kernels finished)
        fetched = [None, None]   # output buffer b free again (its D2H finished)
        last = None
        for n, (src, dst) in enumerate(zip(inputs, outputs)):
            b = n % 2
            h2d, comp, d2h = P["h2d"], P["comp"], P["d2h"]
            if packed[b] is not None:
                h2d.wait_event(packed[b])
            names = ("pd", "vn", "wn", "rho")
            with torch.cuda.stream(h2d):
                for k, t in zip(names, src):
                    if t is not None:
                        P["in"][b][k].copy_(t, non_blocking=True)
            landed = ev()
            landed.record(h2d)
            comp.wait_event(landed)
            ib = P["in"][b]
            given = dict(zip(names, (t is not None for t in src)))
            for k, loc, inner, fwd, field in (("pd", 0, K, self.fwd_v, self.pd),
                                              ("vn", 2, K, self.fwd_e, self.vn),
                                              ("wn", 0, K + 1, self.fwd_v, self.wn),
                                              ("rho", 0, K, self.fwd_v, self.rho)):
                if given[k]:
                    self._pack(loc, inner, ib[k], fwd, field, comp)
            packed[b] = ev()
            packed[b].record(comp)
            self.step(dt, pivbz, flux_op, stream=comp)
            if fetched[b] is not None:
                comp.wait_event(fetched[b])
            _lib.call("tsg_unpack", self.grid.handle, 0, K, _lib.ptr(self.pd_out), _lib.ptr(self.fwd_v),
                      _lib.ptr(P["out"][b]), _lib.stream_handle(comp))
            ready = ev()
            ready.record(comp)
            d2h.wait_event(ready)
            with torch.cuda.stream(d2h):
                dst.copy_(P["out"][b], non_blocking=True)
            fetched[b] = ev()
            fetched[b].record(d2h)
            last = fetched[b]
        P["d2h"].wait_event(last)
        P["d2h"].wait_stream(P["comp"])
        end.record(P["d2h"])
        # ... and the caller's stream continues after all of it
        cur.wait_stream(P["d2h"])
        return start, end

    def __call__(self, pd, vn, wn, rho, dt, pivbz, flux_op="upwind"):
        self.upload(pd, vn, wn, rho)
        self.step(dt, pivbz, flux_op)
        return self.download()


def transport_step_structured(spec: PatchSpec, signs, dual, pd, vn, wn, rho, dt, pivbz,
                              flux_op="upwind", perm_v=None, perm_e=None):
    """One fused structured step on flat arrays (any numbering); returns pd_out."""
    st = StructuredStepper(spec, perm_v, perm_e)
    st.set_geometry(signs, dual)
    return st(pd, vn, wn, rho, dt, pivbz, flux_op)
