"""ctypes binding of oracle/c/libtsg_oracle.so -- TEST/BASELINE INFRASTRUCTURE ONLY."""

from __future__ import annotations

import ctypes
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent / "c"
LIB_PATH = HERE / "build" / "libtsg_oracle.so"
_lib = None

_D = ctypes.POINTER(ctypes.c_double)
_I = ctypes.POINTER(ctypes.c_int64)


def build() -> Path:
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        _lib = ctypes.CDLL(str(LIB_PATH))
        _lib.tsgo_transport_step.restype = ctypes.c_int
        _lib.tsgo_transport_step.argtypes = [_I, _I, _D, _D, _D, _D, _D, _D, ctypes.c_int64,
                                             ctypes.c_int64, ctypes.c_int, ctypes.c_double,
                                             ctypes.c_double, ctypes.c_int, _D, _D, _D, _D]
        _lib.tsgo_neighbor_sum.restype = ctypes.c_int
        _lib.tsgo_neighbor_sum.argtypes = [_I, ctypes.c_int64, ctypes.c_int, _D, ctypes.c_int, _D, _D]
        _lib.tsgo_threads.restype = ctypes.c_int
    return _lib


def _d(a):
    return a.ctypes.data_as(_D)


def _i(a):
    return a.ctypes.data_as(_I)


def threads() -> int:
    return lib().tsgo_threads()


def set_threads(n: int) -> None:
    lib().tsgo_set_threads(ctypes.c_int(n))


def transport_step(e2v, v2e, signs, dual, pd, vn, wn, rho, dt, pivbz, flux_op="upwind", out=None):
    arrs = [np.ascontiguousarray(x, dtype=np.int64) for x in (e2v, v2e)]
    f = [np.ascontiguousarray(x, dtype=np.float64) for x in (signs, dual, pd, vn, wn, rho)]
    nv, K = f[2].shape
    ne = f[3].shape[0]
    if out is None:
        out = {"flux": np.empty((ne, K)), "fluz": np.empty((nv, K + 1)),
               "div": np.empty((nv, K)), "pd_out": np.empty((nv, K))}
    rc = lib().tsgo_transport_step(_i(arrs[0]), _i(arrs[1]), *[_d(x) for x in f], nv, ne, K,
                                   float(dt), float(pivbz), 0 if flux_op == "upwind" else 1,
                                   _d(out["flux"]), _d(out["fluz"]), _d(out["div"]), _d(out["pd_out"]))
    if rc:
        raise ValueError("levels must be >= 2")
    return out


def neighbor_sum(table, a, fac=None):
    t = np.ascontiguousarray(table, dtype=np.int64)
    a = np.ascontiguousarray(a, dtype=np.float64)
    out = np.empty((t.shape[0], a.shape[1]))
    facp = None
    if fac is not None:
        fac = np.ascontiguousarray(fac, dtype=np.float64).reshape(-1)
        facp = _d(fac)
    lib().tsgo_neighbor_sum(_i(t), t.shape[0], t.shape[1], _d(a), a.shape[1], facp, _d(out))
    return out
