"""Synthetic workloads of the reference's benchmark, as flat canonical arrays.

``transport_inputs`` reproduces ``bench._transport_setup`` (bench.py:293-303)
and the tests' ``_transport_case`` (tests/test_acceptance.py:81-92) draw for
draw with numpy's generators, so the same seed yields bitwise the same
inputs as the reference (pinned by tests/golden).  Signs come from the
device kernel ``tsg_edge_signs``.

``CONFIGS`` realises BASELINE.json's named grids as periodic patches
(SURVEY.md 8(d)).
"""

from __future__ import annotations

import zlib

import numpy as np

from .mpdata import UNIT_CELL_AREA, UNIT_DUAL_VOLUME, UNIT_EDGE_LENGTH

CONFIGS = {
    "cfg1": dict(rows=44, cols=72, levels=10, label="O24-size patch, 10 levels"),
    "cfg2": dict(rows=128, cols=128, levels=80, label="128x128x80 octahedral patch (Table 1)"),
    "cfg3": dict(rows=279, cols=256, levels=80,
                 label="71424 nodes / 214272 edges / 80 levels (paper Fig. 15 grid size)"),
    "cfg4": dict(rows=256, cols=256, levels=80, label="9 stencil types, 256x256x80"),
    "cfg5": dict(rows=2560, cols=2576, levels=137, label="O1280-size patch, 137 levels"),
}


def _core(rows, cols, colors, levels):
    return (rows, colors, cols, levels, 1)


def transport_inputs(rows: int, cols: int, levels: int, seed: int = 0, geometry: str = "uniform",
                     preset: str = "gaussian-bump", rho: str = "one", signs: bool = True) -> dict:
    """Flat [element, level] inputs of one transport step (canonical numbering).

    ``signs=False`` skips the device-built orientation signs (host-only use).
    """
    from .connectivity import edge_signs_table
    from .topology import PatchSpec

    if geometry == "uniform":
        dual = np.full(rows * cols, UNIT_DUAL_VOLUME)
        length = np.full(3 * rows * cols, UNIT_EDGE_LENGTH)
        area = np.full(2 * rows * cols, UNIT_CELL_AREA)
    elif geometry == "random":
        g = np.random.default_rng(seed)  # lengths, areas, volumes (mpdata.py:127-131)
        length = (UNIT_EDGE_LENGTH * (0.5 + g.random((rows, 3, cols)))).reshape(-1)
        area = (UNIT_CELL_AREA * (0.5 + g.random((rows, 2, cols)))).reshape(-1)
        dual = (UNIT_DUAL_VOLUME * (0.5 + g.random((rows, 1, cols)))).reshape(-1)
    else:
        raise ValueError(f"unknown geometry mode {geometry!r}")
    shape = _core(rows, cols, 1, levels)
    if preset == "uniform":
        pd = np.ones(shape)
    elif preset == "gaussian-bump":
        sigma = max(rows, cols) / 6.0
        di = np.arange(rows)[:, None] - rows / 2.0
        dj = np.arange(cols)[None, :] - cols / 2.0
        bump = np.exp(-(di ** 2 + dj ** 2) / (2.0 * sigma ** 2))
        pd = np.broadcast_to(bump[:, None, :, None, None], shape).copy()
    elif preset == "random":
        pd = np.random.default_rng([seed, zlib.crc32(b"pd_in")]).random(shape)
    else:
        raise ValueError(f"unknown preset {preset!r}")
    rng = np.random.default_rng(seed)
    vn = -0.5 + (0.5 - -0.5) * rng.random(_core(rows, cols, 3, levels))
    wn = -0.5 + (0.5 - -0.5) * rng.random(_core(rows, cols, 1, levels + 1))
    if rho == "one":
        rho_v = np.ones(shape)
    elif rho == "random":
        rho_v = 0.5 + (1.5 - 0.5) * rng.random(shape)
    else:
        raise ValueError(f"unknown rho mode {rho!r}")
    nv = rows * cols
    out = {
        "pd": pd.reshape(nv, levels), "vn": vn.reshape(3 * nv, levels),
        "wn": wn.reshape(nv, levels + 1), "rho": rho_v.reshape(nv, levels),
        "dual": dual, "length": length, "area": area,
    }
    if signs:
        out["signs"] = edge_signs_table(PatchSpec(rows, cols, levels))
    return out


def mpdata_algorithmic_bytes(rows: int, cols: int, levels: int) -> int:
    """B_comp: pd r + vn r + wn interfaces 1..K-1 r + rho r + pd_out w."""
    v = rows * cols
    return 8 * (v * levels + 3 * v * levels + v * (levels - 1) + v * levels + v * levels)


def mpdata_2d_bytes(rows: int, cols: int) -> int:
    """Per-vertex 2-D inputs read once per step: 6 signs + dual."""
    return 8 * 7 * rows * cols


def paper_model_bytes(rows: int, cols: int, levels: int) -> int:
    """Table-2 fused count: nodes (4r + 1w) per plane x levels x 8 B."""
    return 5 * rows * cols * levels * 8
