"""Host memory layouts and element numberings (mirrors tristencil.layouts).

* :class:`LayoutSpec` / :class:`LinearLayout` describe the host ("primary")
  buffer of a Field exactly like layouts.py:27-104, so host views and offsets
  are unchanged for callers.  The device copy always uses the structured
  layout of include/tsg.h; ``tsg_pack_strided`` reorders between the two on
  the GPU.
* Numberings (layouts.py:134-279): ``sn`` identity, ``un`` colour-interleaved
  ``(i*cols + j)*colors + c``, ``hn`` Hilbert walk.  :func:`make_permutation`
  builds them with the ``tsg_make_permutation`` kernels (block-scan
  compaction of the Hilbert walk), so O1280-sized numberings cost
  milliseconds instead of a Python loop over ids.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass

import numpy as np

from .topology import PatchSpec, as_location, element_count, element_id

AXES = ("row", "color", "column", "level", "extra")
DEFAULT_DIM_ORDER = ("extra", "level", "row", "color", "column")


@dataclass(frozen=True)
class LayoutSpec:
    """Memory nesting order (outermost first) and innermost-axis alignment."""

    dim_order: tuple = DEFAULT_DIM_ORDER
    alignment: int = 8

    def __post_init__(self):
        if sorted(self.dim_order) != sorted(AXES):
            raise ValueError(f"dim_order must be a permutation of {AXES}, got {self.dim_order}")
        if self.alignment < 1:
            raise ValueError(f"alignment must be >= 1, got {self.alignment}")

    @property
    def innermost(self) -> str:
        return self.dim_order[-1]


class LinearLayout:
    """Strides, innermost padding and front pad of one host buffer (layouts.py:55-104)."""

    def __init__(self, spec: LayoutSpec, sizes: dict, halo: int):
        if set(sizes) != set(AXES):
            raise ValueError(f"sizes must cover axes {AXES}, got {sorted(sizes)}")
        self.spec = spec
        self.sizes = dict(sizes)
        self.halo = halo
        inner = spec.innermost
        a = spec.alignment
        self.padded = {ax: (-(-n // a) * a if ax == inner else n) for ax, n in sizes.items()}
        strides, run = {}, 1
        for ax in spec.dim_order[::-1]:
            strides[ax] = run
            run *= self.padded[ax]
        self.strides = strides
        self.front_pad = (-halo * strides["column"]) % a
        self.total = self.front_pad + run

    def offset(self, i: int, c: int, j: int, k: int = 0, x: int = 0) -> int:
        idx = {"row": i + self.halo, "color": c, "column": j + self.halo, "level": k, "extra": x}
        for ax in AXES:
            if not 0 <= idx[ax] < self.sizes[ax]:
                raise IndexError(f"{ax} index out of range: storage index {idx[ax]} not in "
                                 f"[0, {self.sizes[ax]})")
        return self.front_pad + sum(idx[ax] * self.strides[ax] for ax in AXES)

    def view_shape_strides(self):
        return tuple(self.sizes[a] for a in AXES), tuple(self.strides[a] for a in AXES)

    def layout6(self) -> np.ndarray:
        """{front_pad, row, color, column, level, extra} strides for tsg_pack_strided."""
        return np.array([self.front_pad] + [self.strides[a] for a in AXES], dtype=np.int64)


def sn_offset(layout: LayoutSpec, spec: PatchSpec, loc, i, c, j, k=0, x=0, levels=None, extra=1) -> int:
    loc = as_location(loc)
    sizes = {"row": spec.rows + 2 * spec.halo, "color": loc.colors,
             "column": spec.cols + 2 * spec.halo,
             "level": spec.levels if levels is None else levels, "extra": extra}
    return LinearLayout(layout, sizes, spec.halo).offset(i, c, j, k, x)


class Numbering(enum.Enum):
    SN = "sn"
    UN = "un"
    HN = "hn"


class AccessMethod(enum.Enum):
    DIRECT = "direct"
    INDIRECT = "indirect"


def check_access_combo(numbering: Numbering, access: AccessMethod) -> None:
    if access is AccessMethod.DIRECT and numbering is not Numbering.SN:
        raise ValueError(f"direct access requires sn numbering, got {numbering.value}")


@dataclass(frozen=True)
class Permutation:
    """Bijection canonical id <-> storage rank (layouts.py:153-180)."""

    forward: np.ndarray
    inverse: np.ndarray

    def __post_init__(self):
        n = len(self.forward)
        if len(self.inverse) != n:
            raise ValueError("forward/inverse length mismatch")
        if not np.array_equal(self.inverse[self.forward], np.arange(n)):
            raise ValueError("permutation is not a bijection")

    def __len__(self) -> int:
        return len(self.forward)

    @classmethod
    def from_forward(cls, forward) -> "Permutation":
        forward = np.asarray(forward, dtype=np.int64)
        inverse = np.empty_like(forward)
        inverse[forward] = np.arange(len(forward), dtype=np.int64)
        return cls(forward=forward, inverse=inverse)

    @classmethod
    def identity(cls, n: int) -> "Permutation":
        ids = np.arange(n, dtype=np.int64)
        return cls(forward=ids, inverse=ids.copy())


def _check_pow2(n: int) -> None:
    if not (n >= 2 and n & (n - 1) == 0):
        raise ValueError(f"n must be a power of two >= 2, got {n}")


def hilbert_rank(n: int, x: int, y: int) -> int:
    """Rank of (x, y) on the n x n Hilbert curve; (0,0),(0,1),(1,1),(1,0) for n = 2."""
    _check_pow2(n)
    if not (0 <= x < n and 0 <= y < n):
        raise ValueError(f"cell ({x}, {y}) outside the {n} x {n} grid")
    rank, s = 0, n >> 1
    while s:
        qx, qy = int(bool(x & s)), int(bool(y & s))
        rank += s * s * ((3 * qx) ^ qy)
        if not qy:
            if qx:
                x, y = s - 1 - x, s - 1 - y
            x, y = y, x
        s >>= 1
    return rank


def hilbert_xy(n: int, rank: int) -> tuple[int, int]:
    """Inverse of :func:`hilbert_rank` (same quadrant rotation as tsg hilbert_xy)."""
    _check_pow2(n)
    if not 0 <= rank < n * n:
        raise ValueError(f"rank {rank} out of range [0, {n * n})")
    x = y = 0
    t, s = rank, 1
    while s < n:
        qx = 1 & (t >> 1)
        qy = 1 & (t ^ qx)
        if not qy:
            if qx:
                x, y = s - 1 - x, s - 1 - y
            x, y = y, x
        x, y = x + s * qx, y + s * qy
        t >>= 2
        s <<= 1
    return x, y


_NUMBERING_CODE = {Numbering.SN: 0, Numbering.UN: 1, Numbering.HN: 2}


def make_permutation(numbering, patch, loc) -> Permutation:
    """Permutation of a numbering scheme, built on the device (tsg_make_permutation)."""
    import torch

    from . import _lib
    from .device import require_cuda

    numbering = Numbering(getattr(numbering, "value", numbering))
    spec: PatchSpec = getattr(patch, "spec", patch)
    loc = as_location(loc)
    n = element_count(spec, loc)
    if numbering is Numbering.SN:
        return Permutation.identity(n)
    if numbering is Numbering.HN and loc.value == "edges":
        raise ValueError("hn numbering is not defined for edges")
    dev = require_cuda()
    fwd = torch.empty(n, dtype=torch.int64, device=dev)
    work = None
    if numbering is Numbering.HN:
        nwork = _lib.lib().tsg_permutation_work_elems(spec.rows, spec.cols, loc.code)
        work = torch.empty(nwork, dtype=torch.int64, device=dev)
    _lib.call("tsg_make_permutation", spec.rows, spec.cols, loc.code, _NUMBERING_CODE[numbering],
              _lib.ptr(fwd), _lib.ptr(work), _lib.stream_handle())
    return Permutation.from_forward(fwd.cpu().numpy())


def un_rank(spec: PatchSpec, loc, i: int, c: int, j: int) -> int:
    """UN rank of one element (layouts.py:258-264), for tests and tools."""
    loc = as_location(loc)
    element_id(spec, loc, i, c, j)
    return (i * spec.cols + j) * loc.colors + c


# ---------------------------------------------------------------------------
# Coalescing model of the reference's Table-1 study (layouts.py:282-326): which warp
# address groups of a sweep form one contiguous range.  Host analysis only; the B200
# sweeps' real sector efficiency comes from ncu (profiles/).


def coalescing_fraction(groups) -> float:
    """Fraction of access groups whose addresses are distinct and cover [min, min + len)
    (order inside a group does not matter; width-1 groups are trivially coalesced)."""
    groups = list(groups)
    if not groups:
        raise ValueError("no access groups given")
    hits = 0
    for g in groups:
        a = np.sort(np.asarray(g, dtype=np.int64).reshape(-1))
        if a.size == 0:
            raise ValueError("empty access group")
        hits += bool(np.all(np.diff(a) == 1))
    return hits / len(groups)


def direct_sweep_groups(layout: LayoutSpec, spec: PatchSpec, loc, width: int) -> list:
    """Warp address groups of a direct column sweep of one structured field: each
    interior (row, colour, level) line of columns chopped into groups of ``width``
    (the last group of a line may be shorter), lines in (row, colour, level) order."""
    if width < 1:
        raise ValueError(f"width must be >= 1, got {width}")
    loc = as_location(loc)
    sizes = {"row": spec.rows + 2 * spec.halo, "color": loc.colors,
             "column": spec.cols + 2 * spec.halo, "level": spec.levels, "extra": 1}
    lay = LinearLayout(layout, sizes, spec.halo)
    st = lay.strides
    i = np.arange(spec.rows)[:, None, None, None]
    c = np.arange(loc.colors)[None, :, None, None]
    k = np.arange(spec.levels)[None, None, :, None]
    j = np.arange(spec.cols)[None, None, None, :]
    off = (lay.front_pad + (i + spec.halo) * st["row"] + c * st["color"]
           + (j + spec.halo) * st["column"] + k * st["level"])
    lines = off.reshape(-1, spec.cols)
    return [line[s:s + width].tolist() for line in lines for s in range(0, spec.cols, width)]
