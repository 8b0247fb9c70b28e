"""Reference-side binding of libtsg.so with nothing but ctypes + libcudart (no torch).

This is the stub a ``tristencil`` maintainer would add next to reference.py to route
``reference.transport_step`` (reference.py:93-116) and ``reference.neighbor_sum``
(reference.py:137-145) to the B200 kernels.  It owns device memory through the CUDA
runtime directly, so it shows the C ABI is usable without PyTorch.
quotes it; tests/test_integration.py runs it on the GPU against the oracle.
"""

from __future__ import annotations

import ctypes
import ctypes.util
import glob
import os
from pathlib import Path

import numpy as np

LIBTSG = Path(__file__).resolve().parents[1] / "paper_1908_06094_b200" / "libtsg.so"


def _cudart():
    cands = glob.glob("/usr/local/cuda/lib64/libcudart.so*") + \
        glob.glob(os.path.join(os.path.dirname(np.__file__), "..", "nvidia", "cuda_runtime", "lib",
                               "libcudart.so*"))
    for c in cands:
        try:
            return ctypes.CDLL(c)
        except OSError:
            continue
    return ctypes.CDLL(ctypes.util.find_library("cudart"))


class Tsg:
    """Minimal ctypes facade: device buffers + the flat transport step + neighbour sum."""

    H2D, D2H = 1, 2

    def __init__(self):
        self.rt = _cudart()
        self.lib = ctypes.CDLL(str(LIBTSG))
        self.lib.tsg_last_error.restype = ctypes.c_char_p
        self.rt.cudaMalloc.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_size_t]
        self.rt.cudaMemcpy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
        self.rt.cudaFree.argtypes = [ctypes.c_void_p]
        self._bufs = []

    def _check(self, rc):
        if rc:
            raise RuntimeError(self.lib.tsg_last_error().decode())

    def put(self, a: np.ndarray) -> ctypes.c_void_p:
        a = np.ascontiguousarray(a)
        p = ctypes.c_void_p()
        assert self.rt.cudaMalloc(ctypes.byref(p), max(a.nbytes, 8)) == 0
        assert self.rt.cudaMemcpy(p, a.ctypes.data, a.nbytes, self.H2D) == 0
        self._bufs.append(p)
        return p

    def empty(self, nbytes: int) -> ctypes.c_void_p:
        p = ctypes.c_void_p()
        assert self.rt.cudaMalloc(ctypes.byref(p), max(nbytes, 8)) == 0
        self._bufs.append(p)
        return p

    def get(self, p, shape) -> np.ndarray:
        out = np.empty(shape, dtype=np.float64)
        assert self.rt.cudaMemcpy(out.ctypes.data, p, out.nbytes, self.D2H) == 0
        return out

    def free(self):
        for p in self._bufs:
            self.rt.cudaFree(p)
        self._bufs = []

    def transport_step(self, e2v, v2e, signs, dual, pd, vn, wn, rho, dt, pivbz, flux_op="upwind"):
        """Drop-in for reference.transport_step: numpy in, numpy out."""
        nv, K = pd.shape
        ne = vn.shape[0]
        d = [self.put(np.asarray(x, dtype=np.int64)) for x in (e2v, v2e)]
        d += [self.put(np.asarray(x, dtype=np.float64)) for x in (signs, dual, pd, vn, wn, rho)]
        outs = [self.empty(ne * K * 8), self.empty(nv * (K + 1) * 8), self.empty(nv * K * 8),
                self.empty(nv * K * 8)]
        f = self.lib.tsg_transport_indirect
        f.argtypes = [ctypes.c_void_p] * 8 + [ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
                                              ctypes.c_double, ctypes.c_double, ctypes.c_int] + \
            [ctypes.c_void_p] * 5
        self._check(f(*d, nv, ne, K, dt, pivbz, {"upwind": 0, "centred": 1}[flux_op], *outs, None))
        res = {"flux": self.get(outs[0], (ne, K)), "fluz": self.get(outs[1], (nv, K + 1)),
               "div": self.get(outs[2], (nv, K)), "pd_out": self.get(outs[3], (nv, K))}
        self.free()
        return res

    def neighbor_sum(self, table, a):
        """Drop-in for reference.neighbor_sum."""
        t = self.put(np.asarray(table, dtype=np.int64))
        src = self.put(np.asarray(a, dtype=np.float64))
        out = self.empty(table.shape[0] * a.shape[1] * 8)
        f = self.lib.tsg_neighbor_reduce_indirect
        f.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                      ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        self._check(f(t, table.shape[0], table.shape[1], a.shape[1], src, None, out, None))
        res = self.get(out, (table.shape[0], a.shape[1]))
        self.free()
        return res
