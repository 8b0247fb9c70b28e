"""Numpy restatement of the reference MPDATA path -- TEST INFRASTRUCTURE ONLY.

Imported only by ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
CPU-baseline legs.  Never imported by the product package.

Each function restates one reference function (``/root/reference`` paths
relative to ``pkg/src/tristencil``).  The reference loops over elements and
vectorises over levels; here the loops run over neighbour *slots* and
vectorise over elements and levels.  The per-element floating-point
operation sequence is unchanged, so results are bitwise identical (pinned by
``tests/golden``).
"""

from __future__ import annotations

import zlib

import numpy as np

COLORS = {"vertices": 1, "cells": 2, "edges": 3}

# connectivity.py:36-68 -- per source colour, ordered (drow, target colour, dcol)
OFFSETS = {
    ("edges", "vertices"): (((0, 0, 0), (0, 0, 1)),
                            ((0, 0, 0), (1, 0, 1)),
                            ((0, 0, 0), (1, 0, 0))),
    ("edges", "cells"): (((0, 0, 0), (-1, 1, 0)),
                         ((0, 0, 0), (0, 1, 0)),
                         ((0, 1, 0), (0, 0, -1))),
    ("edges", "edges"): (((0, 1, 0), (0, 2, 1), (-1, 2, 0), (-1, 1, 0)),
                         ((0, 0, 0), (0, 2, 1), (0, 2, 0), (1, 0, 0)),
                         ((0, 1, 0), (1, 0, 0), (0, 0, -1), (0, 1, -1))),
    ("cells", "vertices"): (((0, 0, 0), (0, 0, 1), (1, 0, 1)),
                            ((0, 0, 0), (1, 0, 0), (1, 0, 1))),
    ("cells", "edges"): (((0, 0, 0), (0, 1, 0), (0, 2, 1)),
                         ((0, 2, 0), (0, 1, 0), (1, 0, 0))),
    ("cells", "cells"): (((0, 1, 0), (-1, 1, 0), (0, 1, 1)),
                         ((0, 0, 0), (0, 0, -1), (1, 0, 0))),
    ("vertices", "vertices"): (((0, 0, 1), (1, 0, 1), (1, 0, 0),
                                (0, 0, -1), (-1, 0, -1), (-1, 0, 0)),),
    ("vertices", "edges"): (((0, 0, 0), (0, 1, 0), (0, 2, 0),
                             (0, 0, -1), (-1, 1, -1), (-1, 2, 0)),),
    ("vertices", "cells"): (((0, 0, 0), (0, 1, 0), (0, 0, -1),
                             (-1, 1, -1), (-1, 0, -1), (-1, 1, 0)),),
}

UNIT_EDGE_LENGTH = 1.0
UNIT_CELL_AREA = np.sqrt(3.0) / 4.0      # mpdata.py:53-55
UNIT_DUAL_VOLUME = np.sqrt(3.0) / 2.0


# ---------------------------------------------------------------------------
# ids, tables, numberings


def coords(rows, cols, loc):
    """(i, c, j) of every canonical id -- topology.py:100-109 (inverse of :91-97)."""
    n = rows * COLORS[loc] * cols
    ids = np.arange(n, dtype=np.int64)
    j = ids % cols
    rest = ids // cols
    return rest // COLORS[loc], rest % COLORS[loc], j


def ids_of(rows, cols, loc, i, c, j):
    """Canonical id with periodic wrap -- topology.py:91-97."""
    return ((np.mod(i, rows) * COLORS[loc] + c) * cols + np.mod(j, cols)).astype(np.int64)


def neighbor_table(rows, cols, from_loc, to_loc, fwd_from=None, fwd_to=None):
    """Flat (n_from, width) rank table -- connectivity.py:130-161.

    ``fwd_*`` are forward permutations (id -> rank); row r describes the
    from-element of rank r, entries are target ranks.
    """
    i, c, j = coords(rows, cols, from_loc)
    table = OFFSETS[(from_loc, to_loc)]
    width = len(table[0])
    out = np.empty((i.size, width), dtype=np.int64)
    for slot in range(width):
        di = np.array([table[cc][slot][0] for cc in range(COLORS[from_loc])])[c]
        tc = np.array([table[cc][slot][1] for cc in range(COLORS[from_loc])])[c]
        dj = np.array([table[cc][slot][2] for cc in range(COLORS[from_loc])])[c]
        out[:, slot] = ids_of(rows, cols, to_loc, i + di, tc, j + dj)
    if fwd_to is not None:
        out = np.asarray(fwd_to)[out]
    if fwd_from is not None:
        inv = np.empty_like(fwd_from)
        inv[fwd_from] = np.arange(len(fwd_from))
        out = out[inv]
    return out


def edge_signs(rows, cols):
    """+1 where the vertex is the lower endpoint id -- connectivity.py:184-194."""
    v2e = neighbor_table(rows, cols, "vertices", "edges")
    e2v = neighbor_table(rows, cols, "edges", "vertices")
    lower = e2v.min(axis=1)
    own = np.arange(v2e.shape[0])[:, None]
    return np.where(lower[v2e] == own, 1.0, -1.0).astype(np.float64)


def un_forward(rows, cols, loc):
    """Colour-interleaved rank (i*cols + j)*colors + c -- layouts.py:258-264."""
    i, c, j = coords(rows, cols, loc)
    return ((i * cols + j) * COLORS[loc] + c).astype(np.int64)


def hilbert_xy(n, d):
    """Vectorised inverse Hilbert map -- layouts.py:201-218."""
    d = np.asarray(d, dtype=np.int64)
    x = np.zeros_like(d)
    y = np.zeros_like(d)
    t = d.copy()
    s = 1
    while s < n:
        rx = 1 & (t // 2)
        ry = 1 & (t ^ rx)
        flip = (ry == 0) & (rx == 1)
        x = np.where(flip, s - 1 - x, x)
        y = np.where(flip, s - 1 - y, y)
        swap = ry == 0
        x, y = np.where(swap, y, x), np.where(swap, x, y)
        x = x + s * rx
        y = y + s * ry
        t = t // 4
        s *= 2
    return x, y


def hilbert_rank(n, x, y):
    """Hilbert rank of (x, y) -- layouts.py:183-198 (scalar)."""
    rank = 0
    s = n // 2
    while s > 0:
        rx = 1 if x & s else 0
        ry = 1 if y & s else 0
        rank += s * s * ((3 * rx) ^ ry)
        if ry == 0:
            if rx == 1:
                x, y = s - 1 - x, s - 1 - y
            x, y = y, x
        s //= 2
    return rank


def hn_forward(rows, cols, loc):
    """Hilbert numbering over the quad embedding -- layouts.py:221-279."""
    if loc == "vertices":
        gx, gy = rows, cols
    elif loc == "cells":
        gx, gy = rows, 2 * cols
    else:
        raise ValueError("hn numbering is not defined for edges")
    side = 2
    while side < max(gx, gy):
        side *= 2
    x, y = hilbert_xy(side, np.arange(side * side))
    keep = (x < gx) & (y < gy)
    x, y = x[keep], y[keep]
    if loc == "vertices":
        ids = ids_of(rows, cols, loc, x, 0, y)
    else:
        ids = ids_of(rows, cols, loc, x, y % 2, y // 2)
    fwd = np.empty(ids.size, dtype=np.int64)
    fwd[ids] = np.arange(ids.size)
    return fwd


# ---------------------------------------------------------------------------
# the flat transport step -- reference.py:18-116


def upwind_flux(e2v, vn, pd):
    return pd[e2v[:, 0]] * np.maximum(vn, 0.0) + pd[e2v[:, 1]] * np.minimum(vn, 0.0)


def centred_flux(e2v, vn, pd):
    return 0.5 * vn * (pd[e2v[:, 0]] + pd[e2v[:, 1]])


def upwind_fluz(wn, pd, pivbz):
    n, levels = pd.shape
    if levels < 2:
        raise ValueError(f"need at least 2 levels, got {levels}")
    if wn.shape != (n, levels + 1):
        raise ValueError("wn must be staggered")
    w = wn[:, 1:levels]
    fluz = np.empty_like(wn)
    fluz[:, 1:levels] = np.maximum(w, 0.0) * pd[:, : levels - 1] + np.minimum(w, 0.0) * pd[:, 1:]
    fluz[:, 0] = pivbz * fluz[:, 1]
    fluz[:, levels] = pivbz * fluz[:, levels - 1]
    return fluz


def flux_divergence(v2e, signs, dual, flux, fluz):
    acc = 0.0
    for slot in range(v2e.shape[1]):
        acc = signs[:, slot, None] * flux[v2e[:, slot]] + acc
    acc = acc + (fluz[:, 1:] - fluz[:, :-1])
    return acc / dual[:, None]


def advance_density(pd, div, rho, dt):
    slope = dt * div
    slope = slope / rho
    return pd - slope


def transport_step(e2v, v2e, signs, dual, pd, vn, wn, rho, dt, pivbz, flux_op="upwind"):
    if flux_op == "upwind":
        flux = upwind_flux(e2v, vn, pd)
    elif flux_op == "centred":
        flux = centred_flux(e2v, vn, pd)
    else:
        raise ValueError(f"unknown flux operator {flux_op!r}")
    fluz = upwind_fluz(wn, pd, pivbz)
    div = flux_divergence(v2e, signs, dual, flux, fluz)
    return {"flux": flux, "fluz": fluz, "div": div,
            "pd_out": advance_density(pd, div, rho, dt)}


def neighbor_sum(table, a):
    """reference.py:137-145 (``acc = a[nbr] + acc`` from 0.0)."""
    acc = 0.0
    for slot in range(table.shape[1]):
        acc = a[table[:, slot]] + acc
    return acc


def neighbor_sum_scaled(table, a, fac):
    """reference.py:148-157."""
    return neighbor_sum(table, a) * fac


def cell_divergence(c2e, vn, length, area):
    """reference.py:119-134."""
    acc = 0.0
    for slot in range(c2e.shape[1]):
        e = c2e[:, slot]
        acc = vn[e] * length[e, None] + acc
    return acc / area[:, None]


def weighted_divergence(c2e, vn, weights):
    """mpdata.py:372-376: ``acc = vn(e_n) * w[c, n] + acc`` (no division)."""
    acc = 0.0
    for slot in range(c2e.shape[1]):
        acc = vn[c2e[:, slot]] * weights[:, slot, None] + acc
    return acc


# ---------------------------------------------------------------------------
# input generation -- mpdata.py:106-169, :423-451; bench.py:188-194, :293-303


def geometry(rows, cols, mode="uniform", seed=0):
    """Flat geometry arrays (length[E], area[C], dual[V], weights[C,3], signs[V,6])."""
    if mode == "uniform":
        lengths = np.full((rows, 3, cols), UNIT_EDGE_LENGTH)
        areas = np.full((rows, 2, cols), UNIT_CELL_AREA)
        volumes = np.full((rows, 1, cols), UNIT_DUAL_VOLUME)
    elif mode == "random":
        rng = np.random.default_rng(seed)
        lengths = UNIT_EDGE_LENGTH * (0.5 + rng.random((rows, 3, cols)))
        areas = UNIT_CELL_AREA * (0.5 + rng.random((rows, 2, cols)))
        volumes = UNIT_DUAL_VOLUME * (0.5 + rng.random((rows, 1, cols)))
    else:
        raise ValueError(f"unknown geometry mode {mode!r}")
    length = lengths.reshape(-1)
    area = areas.reshape(-1)
    c2e = neighbor_table(rows, cols, "cells", "edges")
    return {
        "length": length,
        "area": area,
        "dual": volumes.reshape(-1),
        "weights": length[c2e] / area[:, None],
        "signs": edge_signs(rows, cols),
    }


def preset(rows, cols, colors, levels, name, kind, seed=0):
    """init_preset on a (rows, colors, cols, levels, 1) core -> flat [n, levels]."""
    shape = (rows, colors, cols, levels, 1)
    if kind == "uniform":
        values = np.ones(shape)
    elif kind == "gaussian-bump":
        sigma = max(rows, cols) / 6.0
        di = np.arange(rows)[:, None] - rows / 2.0
        dj = np.arange(cols)[None, :] - cols / 2.0
        bump = np.exp(-(di**2 + dj**2) / (2.0 * sigma**2))
        values = np.broadcast_to(bump[:, None, :, None, None], shape).copy()
    elif kind == "random":
        values = np.random.default_rng([seed, zlib.crc32(name.encode())]).random(shape)
    else:
        raise ValueError(f"unknown preset {kind!r}")
    return values.reshape(rows * colors * cols, levels)


def fill(rng, rows, cols, colors, levels, lo, hi):
    """bench._fill_random on a (rows, colors, cols, levels, 1) core."""
    values = lo + (hi - lo) * rng.random((rows, colors, cols, levels, 1))
    return values.reshape(rows * colors * cols, levels)


def transport_inputs(rows, cols, levels, seed=0, geometry_mode="uniform",
                     pd_preset="gaussian-bump", rho_mode="one"):
    """Flat inputs of one transport step.

    ``rho_mode='one'`` is bench._transport_setup (bench.py:293-303);
    ``rho_mode='random'`` is the acceptance/unit-test variant
    (tests/test_acceptance.py:81-92) that draws rho ~ U[0.5, 1.5) after wn.
    """
    geo = geometry(rows, cols, geometry_mode, seed)
    rng = np.random.default_rng(seed)
    pd = preset(rows, cols, 1, levels, "pd_in", pd_preset, seed)
    vn = fill(rng, rows, cols, 3, levels, -0.5, 0.5)
    wn = fill(rng, rows, cols, 1, levels + 1, -0.5, 0.5)
    if rho_mode == "one":
        rho = np.ones((rows * cols, levels))
    elif rho_mode == "random":
        rho = fill(rng, rows, cols, 1, levels, 0.5, 1.5)
    elif rho_mode == "uniform":
        rho = np.ones((rows * cols, levels))
    else:
        raise ValueError(rho_mode)
    return dict(pd=pd, vn=vn, wn=wn, rho=rho, **geo)


def step_inputs(rows, cols, inputs, dt, pivbz, flux_op="upwind"):
    """Run one oracle transport step on ``transport_inputs`` output."""
    e2v = neighbor_table(rows, cols, "edges", "vertices")
    v2e = neighbor_table(rows, cols, "vertices", "edges")
    return transport_step(e2v, v2e, inputs["signs"], inputs["dual"], inputs["pd"],
                          inputs["vn"], inputs["wn"], inputs["rho"], dt, pivbz, flux_op)


def total_mass(pd, dual):
    """mpdata.py:496-500 on flat arrays."""
    return float(np.sum(pd * dual[:, None]))
