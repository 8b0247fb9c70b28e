"""GPU runners behind the reference's executor protocol ``runner(comp) -> RunStats``.

The reference runs stage bodies through ``run_naive`` / ``run_fused``
(executors.py:213-316); time_computation takes any such runner
(executors.py:390-414).  Here:

* :func:`run_gpu` executes a computation on the device.  ``fused=True`` is the
  single-pass TMA kernel (``tsg_mpdata_step``); ``fused=False`` is the
  four-kernel path that materialises flux / fluz / divvd like ``run_naive``.
* :func:`run_naive` / :func:`run_fused` keep the reference's signatures so
  existing call sites work unchanged.  ``TileSpec`` is validated like the
  reference's (a tile smaller than the largest stage reach raises the same
  ``ValueError``) and sets the reported stage updates (the fused plan's apron
  recompute); the device tiling is the kernel's own.
* ``RunStats.traffic()`` returns the reference's ``TrafficReport`` (per field
  and phase, distinct and raw accesses), filled from the closed form of what
  the reference's counters record (traffic.py).

Inputs are uploaded on demand (primary -> mirror, reordered on the GPU);
outputs are written on the device and, with ``download=True`` (default, the
reference's semantics: results are readable from the Field afterwards),
synced back to the host.  ``download=False`` leaves them device-resident.
"""

from __future__ import annotations

import statistics
import time
from dataclasses import dataclass, field as dc_field

from . import _lib
from .storage import Field, device_grid, sync
from .traffic import TrafficReport, record_run, required_tile

_FLUX_CODE = {"upwind": 0, "centred": 1}


@dataclass(frozen=True)
class TileSpec:
    tile_i: int
    tile_j: int
    workers: int = 1

    def __post_init__(self):
        if self.tile_i < 1 or self.tile_j < 1:
            raise ValueError(f"tile sizes must be >= 1, got {self.tile_i}x{self.tile_j}")
        if self.workers < 1:
            raise ValueError(f"workers must be >= 1, got {self.workers}")


@dataclass
class RunStats:
    """Device times and update counts of one run (executors.py:48-71).

    ``wall_times`` holds the CUDA-event device time of the launch sequence in
    seconds; ``traffic()`` is the reference's per-field access report under the
    ``"{tag}/"`` phase prefix; ``bytes_moved`` the algorithmic HBM bytes.
    """

    tag: str
    executor: str
    fields: list = dc_field(default_factory=list)
    wall_times: dict = dc_field(default_factory=dict)
    stage_updates: dict = dc_field(default_factory=dict)
    bytes_moved: int = 0

    @property
    def total_wall(self) -> float:
        return sum(self.wall_times.values())

    @property
    def total_updates(self) -> int:
        return sum(self.stage_updates.values())

    def traffic(self) -> TrafficReport:
        return TrafficReport.gather(self.fields, prefix=f"{self.tag}/")


def halo_update(field: Field, space: str = "primary") -> None:
    """Refresh the periodic halo (executors.py:74-86); 'mirror' runs tsg_halo_update."""
    if space == "mirror":
        grid = device_grid(field.spec)
        t = field.buffer("mirror")
        _lib.call("tsg_halo_update", grid.handle, field.loc_code, field.inner, _lib.ptr(t),
                  _lib.stream_handle())
        field.dirty["mirror"] = True
        return
    spec = field.spec
    h, rows, cols = spec.halo, spec.rows, spec.cols
    arr = field.array(space, "rw")
    arr[:h] = arr[rows:rows + h]
    arr[h + rows:] = arr[h:2 * h]
    arr[:, :, :h] = arr[:, :, cols:cols + h]
    arr[:, :, h + cols:] = arr[:, :, h:2 * h]


def mpdata_bytes(rows: int, cols: int, levels: int, fused: bool = True) -> int:
    """Algorithmic HBM bytes of one step (SURVEY 8(d) B_comp; unfused: DISTINCT model)."""
    v, e = rows * cols, 3 * rows * cols
    if fused:
        return 8 * (v * levels + e * levels + v * (levels - 1) + v * levels + v * levels)
    # flux: pd r, vn r, flux w; fluz: pd r, wn r, fluz w; div: flux r, fluz r, div w;
    # advance: pd r, div r, rho r, pd_out w
    return 8 * (3 * e * levels + 7 * v * levels + 2 * v * (levels + 1) + v * (levels - 1))


def _launch(comp, fused: bool, stream):
    import torch

    grid = device_grid(comp.patch)
    s = _lib.stream_handle(stream)
    if comp.kind == "mpdata":
        st, geo, p = comp.state, comp.geo, comp.params
        ins = [st.pd_in.ensure_device(), st.vn.ensure_device(), st.wn.ensure_device(),
               st.rho.ensure_device(), geo.edge_signs.ensure_device(),
               geo.dual_volumes.ensure_device()]
        outs = [st.pd_out] if fused else [st.flux, st.fluz, st.divvd, st.pd_out]
        optrs = [_lib.ptr(f.buffer("mirror")) for f in outs]
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        start.record(stream)
        if fused:
            _lib.call("tsg_mpdata_step", grid.handle, *[_lib.ptr(t) for t in ins], *optrs,
                      float(p.dt), float(p.pivbz), _FLUX_CODE[comp.flux_op], s)
        else:
            _lib.call("tsg_mpdata_step_unfused", grid.handle, *[_lib.ptr(t) for t in ins], *optrs,
                      float(p.dt), float(p.pivbz), _FLUX_CODE[comp.flux_op], s)
        end.record(stream)
        nbytes = mpdata_bytes(comp.patch.rows, comp.patch.cols, comp.patch.levels, fused)
    elif comp.kind == "divergence":
        g = comp.geo
        vn = comp.state.vn.ensure_device()
        if comp.weighted:
            length = area = None
            w = g.weights.ensure_device()
        else:
            length, area, w = g.edge_length.ensure_device(), g.cell_area.ensure_device(), None
        outs = [comp.out]
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        start.record(stream)
        _lib.call("tsg_cell_divergence", grid.handle, int(comp.weighted), _lib.ptr(vn),
                  _lib.ptr(length), _lib.ptr(area), _lib.ptr(w),
                  _lib.ptr(comp.out.buffer("mirror")), s)
        end.record(stream)
        nbytes = 8 * comp.patch.rows * comp.patch.cols * comp.patch.levels * 5
    elif comp.kind == "reduce":
        src = comp.src.ensure_device()
        scale = comp.scale.ensure_device() if comp.scale is not None else None
        outs = [comp.dst]
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        start.record(stream)
        _lib.call("tsg_neighbor_reduce", grid.handle, comp.from_loc.code, comp.to_loc.code,
                  comp.dst.inner, _lib.ptr(src), _lib.ptr(scale),
                  _lib.ptr(comp.dst.buffer("mirror")), s)
        end.record(stream)
        nbytes = comp.algorithmic_bytes()
    else:
        raise TypeError(f"cannot run computation of kind {getattr(comp, 'kind', None)!r}")
    for f in outs:
        f.mark_device_written()
    return outs, (start, end), nbytes


# Streamed host step (run_fused on host Fields, the reference's loop of bench.py:398-403):
# when the density is the only host-side input, it goes up, through the fused step and
# back down band by band of rows on three streams, so the upload of band b+1, the step of
# band b and the download of band b-1 overlap (PCIe is full duplex) instead of running one
# after the other over the whole field.  279x256x80: 1.59 ms per run_fused (device 1.47)
# against 2.02 ms unstreamed (tools/streamed_probe.py; 2 / 4 / 8 / 12 bands: 1.77 / 1.62 /
# 1.60 / 1.65 ms).  A row band of the level-outer host layout is a strided (2-D) copy, and
# concurrent 2-D copies in both directions move ~20 % less than 1-D ones
# (tools/dma2d_probe.py: 1.19 vs 0.99 ms for the field both ways in 6 bands), which is
# what keeps it above the ~1.0 ms of the link.
_STREAM_BANDS = 6
_STREAM_MIN_ROWS = 24


def _band_plan(field):
    """(front, row stride, level stride, level planes outermost) when every band of host
    storage rows of ``field`` is one 2-D copy, else None.  Elements, not bytes."""
    lay = [int(x) for x in field.linear.layout6()]  # front, row, color, column, level, extra
    front, s_row, s_col, s_cl, s_lev = lay[0], lay[1], lay[2], lay[3], lay[4]
    spec, meta = field.spec, field.meta
    rows_st, cols_st = spec.rows + 2 * spec.halo, spec.cols + 2 * spec.halo
    if meta.selector.extra or s_row <= 0 or s_lev <= 0:
        return None
    span_row = (meta.location.colors - 1) * s_col + (cols_st - 1) * s_cl + 1  # one row, one level
    if span_row <= s_row and s_lev >= rows_st * s_row:
        return front, s_row, s_lev, True  # level planes outermost: a band = one run per level
    if span_row + (meta.levels - 1) * s_lev <= s_row:
        return front, s_row, s_lev, False  # rows outermost: a band is contiguous
    return None


def _band_copy(field, buf, staging, rows_lo: int, rows_hi: int, h2d: bool, stream) -> None:
    """Copy host storage rows [rows_lo, rows_hi) of ``field`` between its page-locked host
    buffer ``buf`` and the device ``staging`` image of that buffer (one cudaMemcpy2DAsync)."""
    front, s_row, s_lev, planes = _band_plan(field)
    nrow = rows_hi - rows_lo
    if nrow <= 0:
        return
    host = buf.ctypes.data + 8 * (front + rows_lo * s_row)
    dev = staging.data_ptr() + 8 * (front + rows_lo * s_row)
    width = 8 * nrow * s_row
    height, pitch = (field.meta.levels, 8 * s_lev) if planes else (1, width)
    _lib.call("tsg_memcpy2d", _lib.ctypes.c_void_p(dev if h2d else host), pitch,
              _lib.ctypes.c_void_p(host if h2d else dev), pitch, width, height, 1 if h2d else 2,
              _lib.stream_handle(stream))


def _streamable(comp, fused: bool, download: bool) -> bool:
    if not (fused and download and comp.kind == "mpdata"):
        return False
    st, geo = comp.state, comp.geo
    pd = st.pd_in
    rest = (st.vn, st.wn, st.rho, geo.edge_signs, geo.dual_volumes)
    if not pd.dirty["primary"] or any(f.dirty["primary"] or f._mirror is None for f in rest):
        return False
    if st.pd_out.dirty["mirror"] or pd.has_extra or not pd.has_levels or pd.spec.rows < _STREAM_MIN_ROWS:
        return False
    import numpy as np

    if not np.array_equal(pd.linear.layout6(), st.pd_out.linear.layout6()):
        return False
    return _band_plan(pd) is not None and pd.buffer("primary").ctypes.data % 16 == 0


_STREAMS = {}


def _stream_set(device):
    """Three side streams per device for the streamed host step (created once)."""
    import torch

    key = str(device)
    if key not in _STREAMS:
        _STREAMS[key] = tuple(torch.cuda.Stream(device=device) for _ in range(3))
    return _STREAMS[key]


def _run_streamed(comp, stream):
    """pd_in host -> device -> fused step -> pd_out device -> host, in bands of rows."""
    import torch

    st, geo, p = comp.state, comp.geo, comp.params
    spec = comp.patch
    grid = device_grid(spec)
    R, h, K = spec.rows, spec.halo, spec.levels
    pd_in, pd_out = st.pd_in, st.pd_out
    lay = pd_in.linear.layout6()
    lay_p = lay.ctypes.data_as(_lib.ctypes.POINTER(_lib.ctypes.c_int64))
    host_in, host_out = pd_in.buffer("primary"), pd_out.buffer("primary")
    dev_in, dev_out = pd_in.buffer("mirror"), pd_out.buffer("mirror")
    stage_in = torch.empty(pd_in.linear.total, dtype=torch.float64, device=grid.device)
    stage_out = torch.empty(pd_out.linear.total, dtype=torch.float64, device=grid.device)
    ins = [dev_in, st.vn.buffer("mirror"), st.wn.buffer("mirror"), st.rho.buffer("mirror"),
           geo.edge_signs.buffer("mirror"), geo.dual_volumes.buffer("mirror")]
    B = _STREAM_BANDS
    cuts = [R * b // B for b in range(B + 1)]
    cur = torch.cuda.current_stream() if stream is None else stream
    s_up, s_comp, s_down = _stream_set(grid.device)
    for s in (s_up, s_comp, s_down):
        s.wait_stream(cur)
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record(s_up)
    def up(lo, hi):  # upload interior rows [lo, hi) and pack them (with their halo images)
        _band_copy(pd_in, host_in, stage_in, h + lo, h + hi, True, s_up)
        ev = torch.cuda.Event()
        ev.record(s_up)
        s_comp.wait_event(ev)
        _lib.call("tsg_pack_strided_rows", grid.handle, pd_in.loc_code, K, _lib.ptr(stage_in), lay_p, h, lo, hi,
                  _lib.ptr(dev_in), _lib.stream_handle(s_comp))

    def step_down(lo, hi):  # the fused step over rows [lo, hi), then unpack + download them
        _lib.call("tsg_mpdata_step_rows", grid.handle, *[_lib.ptr(t) for t in ins], _lib.ptr(dev_out),
                  float(p.dt), float(p.pivbz), _FLUX_CODE[comp.flux_op], lo, hi, _lib.stream_handle(s_comp))
        _lib.call("tsg_unpack_strided_rows", grid.handle, pd_out.loc_code, K, _lib.ptr(dev_out), lay_p, h,
                  h + lo, h + hi, _lib.ptr(stage_out), _lib.stream_handle(s_comp))
        ev = torch.cuda.Event()
        ev.record(s_comp)
        s_down.wait_event(ev)
        _band_copy(pd_out, host_out, stage_out, h + lo, h + hi, False, s_down)

    # rows of band b need rows lo-1 .. hi: the last row first (its image is row -1 of the
    # periodic patch), then each band with one extra row below it, so band b steps as soon
    # as its own upload has landed
    up(R - 1, R)
    for b in range(B):
        lo, hi = cuts[b], cuts[b + 1]
        up(lo, min(hi + 1, R))
        step_down(lo, hi)
    # the host halo rows are images of rows R-1 and 0, final only now
    _lib.call("tsg_unpack_strided_rows", grid.handle, pd_out.loc_code, K, _lib.ptr(dev_out), lay_p, h, 0, h,
              _lib.ptr(stage_out), _lib.stream_handle(s_comp))
    _lib.call("tsg_unpack_strided_rows", grid.handle, pd_out.loc_code, K, _lib.ptr(dev_out), lay_p, h,
              R + h, R + 2 * h, _lib.ptr(stage_out), _lib.stream_handle(s_comp))
    ev = torch.cuda.Event()
    ev.record(s_comp)
    s_down.wait_event(ev)
    _band_copy(pd_out, host_out, stage_out, 0, h, False, s_down)
    _band_copy(pd_out, host_out, stage_out, R + h, R + 2 * h, False, s_down)
    s_down.wait_stream(s_comp)
    s_down.wait_stream(s_up)
    end.record(s_down)
    cur.wait_stream(s_down)
    end.synchronize()
    del stage_in, stage_out
    pd_in.dirty = {"primary": False, "mirror": False}
    pd_in.sync_count += 1
    pd_out.dirty = {"primary": False, "mirror": False}
    pd_out.sync_count += 1
    return [pd_out], (start, end), mpdata_bytes(R, spec.cols, K, True)


def run_gpu(comp, fused: bool = True, run_tag: str = "gpu", download: bool = True,
            stream=None, tiles: "TileSpec | None" = None) -> RunStats:
    """Execute ``comp`` on the current CUDA device; returns RunStats."""
    if _streamable(comp, fused, download):
        outs, (start, end), nbytes = _run_streamed(comp, stream)
        download = False  # pd_out is already on the host
    else:
        outs, (start, end), nbytes = _launch(comp, fused, stream)
    end.synchronize()
    updates = record_run(comp, run_tag, fused, tiles)
    if tiles is None:  # useful updates (run_naive's count); a TileSpec adds the apron recompute
        updates = comp.stage_updates()
    stats = RunStats(tag=run_tag, executor="gpu-fused" if fused else "gpu-unfused",
                     fields=comp.fields(), stage_updates=updates, bytes_moved=nbytes)
    stats.wall_times["ms0"] = start.elapsed_time(end) / 1e3
    if download:
        for f in outs:
            sync(f, "primary")
    return stats


def run_naive(comp, run_tag: str = "naive") -> RunStats:
    """Stage-by-stage device execution materialising every intermediate (executors.py:213)."""
    return run_gpu(comp, fused=comp.kind != "mpdata", run_tag=run_tag)


def run_fused(comp, tiles: TileSpec | None = None, run_tag: str = "fused") -> RunStats:
    """Single-pass fused device execution (executors.py:266-316).

    ``tiles`` is checked against the largest stage reach as the reference does
    (executors.py:276-282) and sets the reported flux updates (each tile recomputes
    its apron); the device tiling itself is the kernel's own.  ``None`` = one tile.
    """
    if tiles is not None and not isinstance(tiles, TileSpec):
        raise TypeError("tiles must be a TileSpec")
    if tiles is None:
        tiles = TileSpec(comp.patch.rows, comp.patch.cols)
    ri, rj = required_tile(comp)
    if tiles.tile_i < ri or tiles.tile_j < rj:
        raise ValueError(f"tile {tiles.tile_i}x{tiles.tile_j} smaller than the largest "
                         f"stage reach {ri}x{rj}")
    return run_gpu(comp, fused=True, run_tag=run_tag, tiles=tiles)


def run_time_loop(comp, steps: int, fused: bool = True, run_tag: str = "loop",
                  download: bool = True, stream=None) -> RunStats:
    """The reference's multi-step loop (bench.py:398-403: ``if step: copy pd_out -> pd_in``,
    then run the step) on the device without the copy: the density ping-pongs between the
    pd_in / pd_out device buffers (tsg_mpdata_run for the fused step).  Afterwards pd_out
    holds the final density and pd_in the state before the last step, as in the reference;
    velocities, rho and the geometry stay fixed, as in the reference."""
    import torch

    if getattr(comp, "kind", None) != "mpdata":
        raise TypeError("run_time_loop needs an MPDATA computation")
    steps = int(steps)
    if steps < 1:
        raise ValueError(f"steps must be >= 1, got {steps}")
    grid = device_grid(comp.patch)
    s = _lib.stream_handle(stream)
    st, geo, p = comp.state, comp.geo, comp.params
    a, b = st.pd_in.ensure_device(), st.pd_out.buffer("mirror")
    rest = [st.vn.ensure_device(), st.wn.ensure_device(), st.rho.ensure_device(),
            geo.edge_signs.ensure_device(), geo.dual_volumes.ensure_device()]
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record(stream)
    if fused:
        _lib.call("tsg_mpdata_run", grid.handle, _lib.ptr(a), _lib.ptr(b), *[_lib.ptr(t) for t in rest],
                  float(p.dt), float(p.pivbz), _FLUX_CODE[comp.flux_op], steps, s)
    else:
        mids = [_lib.ptr(f.buffer("mirror")) for f in (st.flux, st.fluz, st.divvd)]
        src, dst = a, b
        for _ in range(steps):
            _lib.call("tsg_mpdata_step_unfused", grid.handle, _lib.ptr(src), *[_lib.ptr(t) for t in rest],
                      *mids, _lib.ptr(dst), float(p.dt), float(p.pivbz), _FLUX_CODE[comp.flux_op], s)
            src, dst = dst, src
    end.record(stream)
    if steps % 2 == 0:  # the final density landed in pd_in's buffer: exchange the buffers
        st.pd_in._mirror, st.pd_out._mirror = st.pd_out._mirror, st.pd_in._mirror
    outs = [st.pd_in, st.pd_out] + ([] if fused else [st.flux, st.fluz, st.divvd])
    for f in outs:
        f.mark_device_written()
    end.synchronize()
    nbytes = steps * mpdata_bytes(comp.patch.rows, comp.patch.cols, comp.patch.levels, fused)
    for _ in range(steps):
        record_run(comp, run_tag, fused)
    stats = RunStats(tag=run_tag, executor="gpu-fused" if fused else "gpu-unfused",
                     fields=comp.fields(),
                     stage_updates={k: steps * v for k, v in comp.stage_updates().items()},
                     bytes_moved=nbytes)
    stats.wall_times["ms0"] = start.elapsed_time(end) / 1e3
    if download:
        for f in outs:
            sync(f, "primary")
    return stats


@dataclass
class TimingResult:
    median_seconds: float
    seconds_per_update: float
    times: list
    updates: int


def time_computation(comp, runner, reps: int = 10, warmup: int = 1) -> TimingResult:
    """Median wall time of ``runner(comp)`` (device work included) after warm-up."""
    import torch

    if reps < 1:
        raise ValueError(f"reps must be >= 1, got {reps}")
    stats = None
    for _ in range(warmup):
        stats = runner(comp)
    torch.cuda.synchronize()
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        stats = runner(comp)
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
    updates = stats.total_updates
    median = statistics.median(times)
    return TimingResult(median, median / updates if updates else float("nan"), times, updates)
