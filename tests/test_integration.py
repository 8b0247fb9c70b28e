"""The reference-side ctypes binding (tools/ctypes_binding.py, quoted in INTEGRATION.md)
drives libtsg.so with plain ctypes + libcudart -- no torch -- and matches the oracle."""

import numpy as np
import pytest

from oracle import tsg_oracle as O

pytestmark = pytest.mark.gpu


def test_ctypes_binding_transport_and_neighbor_sum(cuda_ok, golden, golden_hashes):
    from tools.ctypes_binding import Tsg

    tsg = Tsg()
    for meta in golden_hashes["small_transport"][:6]:
        k = meta["key"]
        r, c, _ = meta["shape"]
        out = tsg.transport_step(O.neighbor_table(r, c, "edges", "vertices"),
                                 O.neighbor_table(r, c, "vertices", "edges"),
                                 golden[f"{k}_signs"], golden[f"{k}_dual"], golden[f"{k}_pd"],
                                 golden[f"{k}_vn"], golden[f"{k}_wn"], golden[f"{k}_rho"],
                                 meta["dt"], meta["pivbz"], meta["flux_op"])
        for name in ("flux", "fluz", "div", "pd_out"):
            assert np.array_equal(out[name], golden[f"{k}_{name}"]), (k, name)
    t = O.neighbor_table(16, 8, "cells", "cells")
    assert np.array_equal(tsg.neighbor_sum(t, golden["k_16x8x2_a"]), golden["k_16x8x2_k1"])
