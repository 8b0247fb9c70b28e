"""Row-strip domain decomposition of the periodic patch across GPUs.

The reference runs on one process and refreshes its periodic halo in place
(executors.py:74-86; SPEC.md:8 replaces MPI with that copy).  Here the patch
is cut into P row strips; each strip is itself a parallelogram,
keeps every column (column periodicity stays local) and needs one halo row of
``pd`` from each ring neighbour per step.  ``vn``/``wn``/``rho``/signs/dual
are static inputs: their halo rows are exchanged once at setup.

* :class:`RowStrips` -- balanced decomposition (first ``rows % P`` strips get
  one extra row).
* :func:`exchange_halo_rows` -- one grouped send/recv per step: a strip's first
  interior storage row goes to the strip above (its bottom halo row), its last
  to the strip below (its top halo row).  Storage rows are contiguous, so the
  transfer is zero-copy into the neighbour's halo.  Works on any backend
  (NCCL over NVLink on GPUs; gloo on CPU tensors in the tests).
* :class:`StripStepper` -- one rank's device state: interior rows are computed
  while the previous step's halo rows are in flight, then the two boundary rows.
  Results are bitwise identical to the single-GPU step (same per-point
  arithmetic; signs come from global canonical ids).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist

from . import _lib
from .device import PERIODIC_COLS, PERIODIC_ROWS, DeviceGrid


@dataclass(frozen=True)
class RowStrips:
    rows: int
    world: int

    def __post_init__(self):
        if self.world < 1 or self.rows < 2 * self.world:
            raise ValueError(f"cannot cut {self.rows} rows into {self.world} strips of >= 2 rows")

    def strip(self, rank: int) -> tuple[int, int]:
        """(first global row, number of rows) of ``rank``'s strip."""
        base, extra = divmod(self.rows, self.world)
        row0 = rank * base + min(rank, extra)
        return row0, base + (1 if rank < extra else 0)

    def up(self, rank: int) -> int:
        return (rank - 1) % self.world

    def down(self, rank: int) -> int:
        return (rank + 1) % self.world


def exchange_halo_rows(field: torch.Tensor, nrows: int, rank: int, world: int, group=None):
    """Fill storage rows 0 and nrows+1 of ``field`` ([nrows+2, ...]) from the ring neighbours.

    Message order per peer is fixed (send to down, send to up; receive from up,
    receive from down) so a 2-rank ring, where up == down, still matches each send
    with the right receive.
    """
    if world == 1:
        return []
    up, down = (rank - 1) % world, (rank + 1) % world
    ops = [dist.P2POp(dist.isend, field[nrows], down, group),   # last interior -> down's top halo
           dist.P2POp(dist.isend, field[1], up, group),         # first interior -> up's bottom halo
           dist.P2POp(dist.irecv, field[0], up, group),         # top halo <- up's last interior
           dist.P2POp(dist.irecv, field[nrows + 1], down, group)]  # bottom halo <- down's first
    return dist.batch_isend_irecv(ops)


def wait_all(reqs) -> None:
    for r in reqs:
        r.wait()


class StripStepper:
    """One rank's strip of a (global_rows x cols x K) patch, stepped on the device.

    Inputs are synthetic (on-device counter hash of global ids, identical for every
    decomposition) unless loaded with :meth:`load_flat`.  ``world == 1`` degenerates to
    the periodic single-patch step.
    """

    def __init__(self, global_rows: int, cols: int, levels: int, rank: int, world: int,
                 seed: int = 0, group=None, flux_op: str = "upwind", exchange=None):
        self.strips = RowStrips(global_rows, world)
        self.rank, self.world, self.group = rank, world, group
        self.row0, self.nrows = self.strips.strip(rank)
        self.cols, self.K = cols, levels
        flags = PERIODIC_COLS | (PERIODIC_ROWS if world == 1 else 0)
        self.grid = DeviceGrid(self.nrows, cols, levels, flags, self.row0, global_rows)
        self.flux_code = {"upwind": 0, "centred": 1}[flux_op]
        g, K = self.grid, levels
        self.pd, self.pd_out = g.empty(0, K), g.empty(0, K)
        self.vn, self.wn, self.rho = g.empty(2, K), g.empty(0, K + 1), g.empty(0, K)
        self.signs, self.dual = g.empty(0, 6), g.empty(0, 1)
        self.comm = torch.cuda.Stream()
        self.pending = []
        # exchange(field, nrows, rank, world, group) -> requests; replaceable for in-process use
        self.exchange = exchange or exchange_halo_rows
        self._fill_synthetic(seed)

    def _fill_synthetic(self, seed: int) -> None:
        s = _lib.stream_handle()
        for k, (f, loc, inner, lo, hi) in enumerate(((self.pd, 0, self.K, 0.0, 1.0),
                                                     (self.vn, 2, self.K, -0.5, 0.5),
                                                     (self.wn, 0, self.K + 1, -0.5, 0.5),
                                                     (self.dual, 0, 1, 0.5, 1.5))):
            _lib.call("tsg_fill_hash", self.grid.handle, loc, inner, seed * 16 + k, lo, hi, _lib.ptr(f), s)
        self.rho.fill_(1.0)
        # orientation signs of the global patch, this strip's rows (+ halo rows)
        gl = self.strips.rows
        flat = torch.empty((gl * self.cols, 6), dtype=torch.float64, device=self.grid.device)
        _lib.call("tsg_edge_signs", gl, self.cols, _lib.ptr(flat), s)
        rows = torch.arange(self.row0 - 1, self.row0 + self.nrows + 1, device=flat.device) % gl
        strip = flat.view(gl, self.cols, 6)[rows]              # [nrows+2, cols, 6]
        self.signs[:, 0, 1:-1, :] = strip
        self.signs[:, 0, 0, :] = strip[:, -1, :]
        self.signs[:, 0, -1, :] = strip[:, 0, :]
        self._exchange_static()

    def _exchange_static(self) -> None:
        """Halo rows of the static inputs (and of pd for the first step), once."""
        for f in (self.pd, self.vn, self.wn, self.rho, self.dual):
            wait_all(self.exchange(f, self.nrows, self.rank, self.world, self.group))
        torch.cuda.current_stream().synchronize()

    def _launch(self, row_lo: int, row_hi: int, dt: float, pivbz: float, stream) -> None:
        _lib.call("tsg_mpdata_step_rows", self.grid.handle, _lib.ptr(self.pd), _lib.ptr(self.vn),
                  _lib.ptr(self.wn), _lib.ptr(self.rho), _lib.ptr(self.signs), _lib.ptr(self.dual),
                  _lib.ptr(self.pd_out), float(dt), float(pivbz), self.flux_code, row_lo, row_hi,
                  _lib.stream_handle(stream))

    def step(self, dt: float, pivbz: float) -> None:
        """pd -> pd_out for this strip; starts pd_out's halo exchange on the comm stream."""
        main = torch.cuda.current_stream()
        if self.world == 1:
            self._launch(0, self.nrows, dt, pivbz, main)
            return
        # interior rows need no halo: overlap them with the previous exchange
        self._launch(1, self.nrows - 1, dt, pivbz, main)
        wait_all(self.pending)  # makes `main` wait for the halo rows of pd
        self.pending = []
        self._launch(0, 1, dt, pivbz, main)
        self._launch(self.nrows - 1, self.nrows, dt, pivbz, main)
        done = torch.cuda.Event()
        done.record(main)
        self.comm.wait_event(done)
        with torch.cuda.stream(self.comm):
            self.pending = self.exchange(self.pd_out, self.nrows, self.rank, self.world, self.group)

    def swap(self) -> None:
        self.pd, self.pd_out = self.pd_out, self.pd

    def finish(self) -> None:
        wait_all(self.pending)
        self.pending = []

    def interior(self, name: str = "pd") -> torch.Tensor:
        """This strip's interior rows of a field, [nrows, colors, cols, inner]."""
        f = getattr(self, name)
        return f[1:self.nrows + 1, :, 1:self.cols + 1]
