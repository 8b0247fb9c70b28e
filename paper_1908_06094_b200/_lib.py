"""ctypes binding of libtsg.so (the C ABI declared in include/tsg.h).

The library is built in-tree (``paper_1908_06094_b200/libtsg.so``) by
``__graft_entry__.build()`` / ``make -C paper_1908_06094_b200/csrc``.  There is
no CPU fallback: every compute entry point of this package calls into this
library, and importing it without the built ``.so`` raises immediately.
Status codes map onto the reference's exception types (include/tsg.h).
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

# TSG_LIBRARY overrides the in-tree build (A/B timing of two builds of the same ABI)
LIB_PATH = Path(os.environ.get("TSG_LIBRARY") or Path(__file__).resolve().with_name("libtsg.so"))

_c_int, _c_i64, _c_dbl, _c_u64 = ctypes.c_int, ctypes.c_int64, ctypes.c_double, ctypes.c_uint64
_p = ctypes.c_void_p

# name -> (restype, argtypes); mirrors include/tsg.h one to one
SIGNATURES = {
    "tsg_last_error": (ctypes.c_char_p, []),
    "tsg_abi_version": (_c_int, []),
    "tsg_grid_create": (_c_int, [_c_int, _c_int, _c_int, _c_int, ctypes.POINTER(_p)]),
    "tsg_grid_destroy": (_c_int, [_p]),
    "tsg_grid_set_origin": (_c_int, [_p, _c_int, _c_int]),
    "tsg_inner_pitch": (_c_i64, [_c_int]),
    "tsg_field_elems": (_c_i64, [_p, _c_int, _c_int]),
    "tsg_halo_update": (_c_int, [_p, _c_int, _c_int, _p, _p]),
    "tsg_pack": (_c_int, [_p, _c_int, _c_int, _p, _p, _p, _p]),
    "tsg_unpack": (_c_int, [_p, _c_int, _c_int, _p, _p, _p, _p]),
    "tsg_pack_strided": (_c_int, [_p, _c_int, _c_int, _p, ctypes.POINTER(_c_i64), _c_int, _p, _p]),
    "tsg_unpack_strided": (_c_int, [_p, _c_int, _c_int, _p, ctypes.POINTER(_c_i64), _c_int, _p, _p]),
    "tsg_pack_strided_rows": (_c_int, [_p, _c_int, _c_int, _p, ctypes.POINTER(_c_i64), _c_int, _c_int, _c_int,
                                       _p, _p]),
    "tsg_unpack_strided_rows": (_c_int, [_p, _c_int, _c_int, _p, ctypes.POINTER(_c_i64), _c_int, _c_int,
                                         _c_int, _p, _p]),
    "tsg_memcpy2d": (_c_int, [_p, _c_i64, _p, _c_i64, _c_i64, _c_i64, _c_int, _p]),
    "tsg_mpdata_step": (_c_int, [_p, _p, _p, _p, _p, _p, _p, _p, _c_dbl, _c_dbl, _c_int, _p]),
    "tsg_mpdata_step_rows": (_c_int, [_p, _p, _p, _p, _p, _p, _p, _p, _c_dbl, _c_dbl, _c_int, _c_int,
                                      _c_int, _p]),
    "tsg_mpdata_step_rows_peer": (_c_int, [_p, _p, _p, _p, _p, _p, _p, _p, _c_dbl, _c_dbl, _c_int,
                                           _c_int, _c_int, _p, _p, _p]),
    "tsg_mpdata_step_strip": (_c_int, [_p, _p, _p, _p, _p, _p, _p, _p, _c_dbl, _c_dbl, _c_int,
                                       _p, _p, _p, _p, _p, _c_i64, _p, _c_int, _p, _p, _p]),
    "tsg_mpdata_run_strip": (_c_int, [_p, _p, _p, _p, _p, _p, _p, _p, _c_dbl, _c_dbl, _c_int,
                                      _p, _p, _p, _p, _p, _p, _p, _p, _c_int, _p, _p, _c_int, _p]),
    "tsg_malloc": (_c_int, [_c_i64, ctypes.POINTER(_p)]),
    "tsg_free": (_c_int, [_p]),
    "tsg_ipc_handle": (_c_int, [_p, ctypes.c_char_p]),
    "tsg_ipc_open": (_c_int, [ctypes.c_char_p, ctypes.POINTER(_p)]),
    "tsg_ipc_close": (_c_int, [_p]),
    "tsg_signal_peers": (_c_int, [_p, _p, _c_i64, _p]),
    "tsg_wait_flags": (_c_int, [_p, _c_i64, _c_int, _p, _p]),
    "tsg_mpdata_step_unfused": (_c_int, [_p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _c_dbl,
                                         _c_dbl, _c_int, _p]),
    "tsg_transport_indirect": (_c_int, [_p, _p, _p, _p, _p, _p, _p, _p, _c_i64, _c_i64, _c_int,
                                        _c_dbl, _c_dbl, _c_int, _p, _p, _p, _p, _p]),
    "tsg_mpdata_run": (_c_int, [_p] + [_p] * 7 + [_c_dbl, _c_dbl, _c_int, _c_int, _p]),
    "tsg_set_fused_variant": (_c_int, [_c_int]),
    "tsg_set_reduce_variant": (_c_int, [_c_int]),
    "tsg_set_point_limit": (_c_int, [_c_i64]),
    "tsg_fused_variant_of": (_c_int, [_p, _c_int, _c_int]),
    "tsg_fused_band_of": (_c_int, [_p, _c_int, _c_int]),
    "tsg_set_fused_band": (_c_int, [_c_int]),
    "tsg_set_fused_schedule": (_c_int, [_c_int]),
    "tsg_fused_wait_error": (_c_int, [_p, ctypes.POINTER(_c_int)]),
    "tsg_fused_loop_launches": (_c_int, [_p, _c_int]),
    "tsg_time_loop_graphs_built": (_c_int, []),
    "tsg_launch_cache_stats": (_c_int, [_p, ctypes.POINTER(_c_i64), ctypes.POINTER(_c_i64)]),
    "tsg_debug_trace": (_c_int, [_p]),
    "tsg_fused_variant_info": (_c_int, [_c_int] + [ctypes.POINTER(_c_int)] * 6),
    "tsg_neighbor_reduce": (_c_int, [_p, _c_int, _c_int, _c_int, _p, _p, _p, _p]),
    "tsg_neighbor_reduce_indirect": (_c_int, [_p, _c_i64, _c_int, _c_int, _p, _p, _p, _p]),
    "tsg_flat_flux": (_c_int, [_p, _p, _p, _c_i64, _c_int, _c_int, _p, _p]),
    "tsg_flat_fluz": (_c_int, [_p, _p, _c_i64, _c_int, _c_dbl, _p, _p]),
    "tsg_flat_divergence": (_c_int, [_p, _c_int, _p, _p, _p, _p, _c_i64, _c_int, _p, _p]),
    "tsg_flat_advance": (_c_int, [_p, _p, _p, _c_i64, _c_dbl, _p, _p]),
    "tsg_flat_cell_divergence": (_c_int, [_p, _c_int, _p, _p, _p, _c_i64, _c_int, _p, _p]),
    "tsg_cell_divergence": (_c_int, [_p, _c_int, _p, _p, _p, _p, _p, _p]),
    "tsg_cell_weights": (_c_int, [_p, _p, _p, _p, _p]),
    "tsg_build_neighbor_table": (_c_int, [_c_int, _c_int, _c_int, _c_int, _p, _p, _p, _p]),
    "tsg_edge_signs": (_c_int, [_c_int, _c_int, _p, _p]),
    "tsg_make_permutation": (_c_int, [_c_int, _c_int, _c_int, _c_int, _p, _p, _p]),
    "tsg_permutation_work_elems": (_c_i64, [_c_int, _c_int, _c_int]),
    "tsg_total_mass": (_c_int, [_p, _p, _p, _p, _p, _p]),
    "tsg_fill_hash": (_c_int, [_p, _c_int, _c_int, _c_u64, _c_dbl, _c_dbl, _p, _p]),
}

_lib = None


class LibraryMissing(ImportError):
    """libtsg.so is not built; there is deliberately no CPU fallback."""


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise LibraryMissing(
                f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
                "or `make -C paper_1908_06094_b200/csrc` (this package has no CPU fallback)")
        handle = ctypes.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            if "TSG_LIBRARY" in os.environ and not hasattr(handle, name):
                continue  # an older build under A/B timing
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


_ERRORS = {1: ValueError, 2: IndexError}


def check(rc: int) -> None:
    """Raise the reference's exception type for a non-zero tsg status."""
    if rc:
        msg = lib().tsg_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, RuntimeError)(msg)


def call(name: str, *args):
    check(getattr(lib(), name)(*args))


def ptr(t) -> ctypes.c_void_p | None:
    """Raw device pointer of a CUDA tensor (None passes NULL)."""
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError("expected a contiguous tensor")
    return ctypes.c_void_p(t.data_ptr())


def stream_handle(stream=None) -> ctypes.c_void_p:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)
