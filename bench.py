#!/usr/bin/env python
"""Benchmark of the MPDATA transport step on B200 (contract: one JSON line on rank 0).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[2], the grid of the paper's Fig. 15): one
fused MPDATA transport step on the periodic 279 x 256 x 80 patch
(71,424 vertices = the paper's node count, 214,272 edges, 80 levels), fp64,
inputs as the reference's ``_transport_setup`` (gaussian-bump density,
U[-0.5,0.5) velocities, rho = 1, uniform geometry, dt = 0.1, pivbz = 1).

* value: grid-point updates/s (V*K per step / device time), inputs resident in
  HBM, every rank stepping its 279-row strip of a (279*N) x 256 x 80 patch
  through ``StripStepper`` (N = 1: the periodic patch; N > 1: row strips with
  the per-step halo exchange) -- the same code path and the same per-strip
  inputs at every N (weak scaling).  The timed region is the reference's time
  loop (bench.py:398-403): K dependent steps, each consuming the previous
  step's density (``StripStepper.run``: one persistent multi-step launch per
  rank, halo exchange inside it for N > 1), bracketed by a barrier + device
  synchronize and CUDA events on the launching stream; no L2 flush between the
  steps -- every step streams 320 MB per rank through a 126 MB L2 -- and a
  256 MiB L2 flush before the region.
* step_flushed: the same step timed one launch at a time, each preceded
  (outside its events) by the L2 flush: per-step spread, and the cold-cache
  single-step figure (round 1's headline protocol).
* o1280_strong: configs[4], the 2560 x 2576 x 137 patch cut into N strips
  through the same StripStepper path (on-device counter-hash inputs), for the
  strong-scaling efficiency T1 / (N * T_N) against the N = 1 run's record.
* e2e: independent host-fed steps through the flat-array API
  (StructuredStepper.run_pipelined): per step H2D of pd from pinned memory,
  reorder, fused step, reorder, D2H of pd_out, overlapped across steps; at N > 1
  every rank feeds its own 279 x 256 x 80 patch (max over ranks).  N = 1 only:
  ``e2e_all_inputs``: the same with every input (pd / vn / wn / rho) copied per
  step.  ``e2e_time_loop``: the reference's dependent loop (bench.py:398-403):
  ``_copy_core(pd_out, pd_in)`` on the host Fields, then ``run_fused(comp,
  TileSpec)`` -- no overlap possible, step n+1 consumes step n's output.
* roofline: algorithmic bytes B_comp per step / average step time, against
  the measured HBM copy bandwidth (MEASURED_PEAKS.json).
* sustained (N = 1, last, outside the clock sampling): the headline loop kept
  busy for --sustained-seconds, the step time it settles to under the board's
  power cap, with the board power and updates per joule.
* cpu_baseline / --impl reference: the reference algorithm restated in C
  (oracle/c, bitwise equal to the reference, OpenMP over all host cores),
  median step of the same sampling protocol in both arms (the repo arm checks the
  benchmarked kernel's result against the sample's own output, bitwise); the
  reference arm also times the reference package itself (``run_fused``,
  ``run_naive``, ``reference.transport_step``; baseline/_ref) when installed.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "MPDATA grid-point updates/s & effective HBM GB/s (frac of peak) at 1/2/4/8 B200"
UNIT = "grid-point updates/s"
DT, PIVBZ = 0.1, 1.0
# BASELINE.json configs[2] (the headline, weak-scaled over GPUs) and configs[4] (O1280-class,
# strong-scaled); SURVEY 8(d) realises both as periodic patches
WORKLOADS = {
    "cfg3": dict(rows=279, cols=256, levels=80, scaling="weak", cpu_rows=279,
                 label="MPDATA full step, 71424-node/214272-edge/80-level periodic patch "
                       "(279x256x80 per GPU), fp64"),
    "o1280": dict(rows=2560, cols=2576, levels=137, scaling="strong", cpu_rows=320,
                  label="MPDATA full step, O1280-class periodic patch 2560x2576x137 "
                        "(6,594,560 vertices), row strips across GPUs, fp64"),
}
SLEEP_CYCLES = 200_000  # ~100 us at 1.965 GHz: the host enqueues flush + events + step meanwhile


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy, burst)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def workload_config(w: dict, world: int) -> dict:
    """The ``config`` both arms print for one workload at N ranks (identical dicts)."""
    rows = w["rows"] * world if w["scaling"] == "weak" else w["rows"]
    return {"workload": w["label"], "rows": rows, "cols": w["cols"], "levels": w["levels"],
            "l2": "inputs larger than L2: every step streams the whole state (>= 320 MB per GPU) "
                  "through the 126 MB L2; one 256 MiB L2 flush before the timed region"}


def step_stats(ms: list) -> dict:
    s = sorted(ms)
    return {"min": s[0], "median": statistics.median(s), "p90": s[min(len(s) - 1, int(0.9 * len(s)))],
            "max": s[-1], "mean": sum(s) / len(s), "n": len(s)}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled while the GPU works."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.12)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU baselines (the reference algorithm restated in C; test/baseline infrastructure)


def cpu_port_sample(rows: int, cols: int, levels: int, warmup: int, steps: int | None = None,
                    budget_s: float | None = None):
    """Step times of the C port on every host core: ``warmup`` untimed steps, then
    ``steps`` timed ones or as many as fit in ``budget_s`` (at least 3).  Both arms use
    this and report the median."""
    from oracle import c_oracle
    from oracle import tsg_oracle as O

    # every host core this process may run on (torchrun exports OMP_NUM_THREADS=1 per rank)
    c_oracle.set_threads(len(os.sched_getaffinity(0)))
    inp = O.transport_inputs(rows, cols, levels, 0, "uniform", "gaussian-bump", "one")
    e2v = O.neighbor_table(rows, cols, "edges", "vertices")
    v2e = O.neighbor_table(rows, cols, "vertices", "edges")
    args = (e2v, v2e, inp["signs"], inp["dual"], inp["pd"], inp["vn"], inp["wn"], inp["rho"], DT, PIVBZ)
    out = None
    for _ in range(max(warmup, 1)):
        out = c_oracle.transport_step(*args, out=out)
    times = []
    t_begin = time.perf_counter()
    while True:
        t0 = time.perf_counter()
        out = c_oracle.transport_step(*args, out=out)
        times.append(time.perf_counter() - t0)
        if steps is not None and len(times) >= steps:
            break
        if budget_s is not None and time.perf_counter() - t_begin > budget_s and len(times) >= 3:
            break
    return times, c_oracle.threads(), out["pd_out"].copy()


def cpu_record(w: dict, times, threads) -> dict:
    r, c, k = w["cpu_rows"], w["cols"], w["levels"]
    t = statistics.median(times)
    part = "" if r == w["rows"] else f" (1/{w['rows'] // r} of the per-job patch; updates/s is size-independent)"
    return {"value": r * c * k / t, "unit": UNIT, "cores": threads, "kind": "port",
            "ms_per_step": t * 1e3,
            "sample": f"{r}x{c}x{k} periodic patch{part}, median of {len(times)} steps, "
                      "reference.transport_step restated in C (oracle/c), OpenMP"}


def reference_python_record(w: dict, reps: int) -> dict | None:
    """The reference package itself (baseline/_ref, unmodified), its three CPU paths on
    ``_transport_setup`` inputs (bench.py:293-303, :375-427): the
    fastest, ``run_fused(comp, TileSpec(R, C, 1))`` via its own ``time_computation``
    (median of ``reps``), plus ``run_naive`` and the flat oracle ``reference.transport_step``
    (one timed run each after one warm-up; table building outside the timing)."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "tristencil").is_dir():
        return None
    sys.path.insert(0, str(ref))
    try:
        from tristencil import mpdata as rmp
        from tristencil import reference as rref
        from tristencil.bench import BenchConfig, _transport_setup
        from tristencil.connectivity import build_neighbor_table, edge_signs_table
        from tristencil.executors import TileSpec, time_computation, run_fused, run_naive
        from tristencil.kernels import field_to_flat
        from tristencil.topology import LocationType
    finally:
        sys.path.remove(str(ref))
    r, c, k = w["cpu_rows"], w["cols"], w["levels"]
    cfg = BenchConfig(rows=r, cols=c, levels=k, tile_i=r, tile_j=c, workers=1)
    spec = cfg.patch()
    state, geo, params = _transport_setup(cfg, spec)
    comp = rmp.build_mpdata(spec, state, geo, params)
    tiles = TileSpec(r, c, 1)
    timing = time_computation(comp, lambda cc: run_fused(cc, tiles), reps=reps, warmup=1)
    naive = time_computation(comp, run_naive, reps=1, warmup=1)
    E, V = LocationType.EDGES, LocationType.VERTICES
    args = (build_neighbor_table(spec, E, V).ids, build_neighbor_table(spec, V, E).ids, edge_signs_table(spec),
            field_to_flat(geo.dual_volumes)[:, 0], field_to_flat(state.pd_in), field_to_flat(state.vn),
            field_to_flat(state.wn), field_to_flat(state.rho), params.dt, params.pivbz)
    rref.transport_step(*args)
    t0 = time.perf_counter()
    rref.transport_step(*args)
    t_oracle = time.perf_counter() - t0
    vk = r * c * k
    return {"value": vk / timing.median_seconds, "unit": UNIT, "cores": 1,
            "kind": "reference-python", "ms_per_step": timing.median_seconds * 1e3,
            "reference_updates_per_second": 1.0 / timing.seconds_per_update,
            "sample": f"{r}x{c}x{k} patch, tristencil.run_fused(comp, TileSpec({r}, {c}, 1)) "
                      f"(its fastest path), median of {reps} via its time_computation",
            "run_naive": {"value": vk / naive.median_seconds, "ms_per_step": naive.median_seconds * 1e3},
            "transport_step": {"value": vk / t_oracle, "ms_per_step": t_oracle * 1e3,
                               "note": "reference.transport_step, the flat oracle (tables built outside)"}}


CPU_PD_OUT = {}


def cpu_baseline(args, w: dict) -> dict:
    """The one CPU-baseline protocol both arms use: the C port on every host core,
    ``--warmup`` untimed steps, then ``--steps`` timed ones (3 for the O1280 sample) capped
    at ``--cpu-seconds``, median; run before any CUDA work in the process."""
    steps = args.steps if args.workload == "cfg3" else min(args.steps, 3)
    times, threads, pd_out = cpu_port_sample(w["cpu_rows"], w["cols"], w["levels"], args.warmup, steps=steps,
                                             budget_s=args.cpu_seconds)
    rec = cpu_record(w, times, threads)
    rec["steps"] = len(times)
    CPU_PD_OUT[args.workload] = pd_out  # the sample's own result: the GPU's is checked against it
    return rec


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    w = WORKLOADS[args.workload]
    cpu = cpu_baseline(args, w)
    value = cpu["value"]
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": cpu["steps"], "warmup": args.warmup, "ms_per_step": cpu["ms_per_step"],
        "higher_is_better": True, "scaling": w["scaling"], "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": workload_config(w, world),
        "cpu_baseline": cpu,
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    # the package itself on the cfg3 patch only: its O1280 sample (a 320-row strip) would
    # take ~80 s per step in pure Python
    if not args.no_python_ref and args.workload == "cfg3":
        try:
            line["reference_python"] = reference_python_record(w, args.python_ref_reps)
        except Exception as e:  # the record is informational: never lose the line over it
            line["reference_python"] = {"unavailable": f"{type(e).__name__}: {e}"}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm


def _exchange_mode(requested: str, rank: int, world: int, local: int, shared: bool):
    """p2p only when both ring neighbours (global rank +- 1) are on this host with peer
    access from this device; otherwise every rank takes the NCCL exchange."""
    import torch
    import torch.distributed as dist

    if world == 1 or shared:
        return requested, None
    info = [None] * world
    dist.all_gather_object(info, (socket.gethostname(), local))
    host = info[rank][0]
    note = None
    mode = requested
    if requested == "p2p":
        for nb in {(rank - 1) % world, (rank + 1) % world} - {rank}:
            h, dev = info[nb]
            if h != host:
                note = f"ring neighbour rank {nb} is on host {h}: NCCL exchange"
            elif not torch.cuda.can_device_access_peer(local, dev):
                note = f"no peer access from cuda:{local} to cuda:{dev}: NCCL exchange"
        flag = torch.tensor([note is not None], dtype=torch.int32, device="cuda")
        dist.all_reduce(flag, op=dist.ReduceOp.MAX)  # every rank takes the same exchange
        if flag.item():
            mode = "nccl"
            note = note or "a rank cannot reach its neighbours peer to peer: NCCL exchange"
    return mode, note


def _timed_steps(stepper, steps, stream, flush_l2=None):
    """Per-step device times (ms) of ``steps`` step+swap pairs on ``stream``."""
    import torch

    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(steps)]
    for s in range(steps):
        torch.cuda._sleep(SLEEP_CYCLES)  # keeps the launch queue ahead of the GPU
        if flush_l2 is not None:
            flush_l2()  # evict the previous step's data from L2 (outside the events)
        evs[s][0].record(stream)
        stepper.step(DT, PIVBZ)
        evs[s][1].record(stream)
        stepper.swap()
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in evs]


def _timed_run(stepper, steps, stream) -> float:
    """Device time (s) of ``stepper.run(steps)`` -- one persistent launch -- between CUDA
    events on ``stream``; a device sleep queued first keeps the host's launch preparation
    off the measured interval (the GPU is busy until the launch is queued)."""
    import torch

    torch.cuda._sleep(SLEEP_CYCLES)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    stepper.run(steps, DT, PIVBZ)
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3


def _max_over_ranks(x: float, world: int, shared: bool) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cpu" if shared else "cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _sm_clock_mhz(index: int):
    """The SM clock now (NVML), or None."""
    try:
        import pynvml

        pynvml.nvmlInit()
        return pynvml.nvmlDeviceGetClockInfo(pynvml.nvmlDeviceGetHandleByIndex(index), pynvml.NVML_CLOCK_SM)
    except Exception:  # informational only
        return None


def _power_w(index: int):
    """The board power now (NVML, W), or None."""
    try:
        import pynvml

        pynvml.nvmlInit()
        return pynvml.nvmlDeviceGetPowerUsage(pynvml.nvmlDeviceGetHandleByIndex(index)) / 1e3
    except Exception:  # informational only
        return None


def o1280_strong(args, rank, world, shared, barrier, peak):
    """configs[4] strong scaling: the O1280-class patch in `world` strips, same path."""
    import torch

    from paper_1908_06094_b200.distributed import StripStepper
    from paper_1908_06094_b200.workloads import mpdata_algorithmic_bytes

    w = WORKLOADS["o1280"]
    R, C, K = w["rows"], w["cols"], w["levels"]
    st = StripStepper(R, C, K, rank, world, seed=0, mode=args.exchange)
    st.run(3, DT, PIVBZ)
    torch.cuda.synchronize()
    if world > 1:
        st.check()
    barrier()
    t_run = _timed_run(st, args.o1280_steps, torch.cuda.current_stream())  # the dependent loop
    barrier()
    if world > 1:
        st.finish()
        st.check()
    t = _max_over_ranks(t_run, world, shared) / args.o1280_steps
    sm_after = _sm_clock_mhz(0 if shared else torch.cuda.current_device())
    # the same step isolated: 200 ms idle before each (the SM clock back at its boost
    # value), so the power-capped sustained loop above can be read against it
    iso = []
    for _ in range(3):
        time.sleep(0.2)
        barrier()
        iso.append(_timed_run(st, 1, torch.cuda.current_stream()))
    barrier()
    if world > 1:
        st.finish()
        st.check()
    t_iso = _max_over_ranks(statistics.median(iso), world, shared)
    mine = mpdata_algorithmic_bytes(st.nrows, C, K)
    rec = {"value": R * C * K / t, "unit": UNIT, "n_gpus": world, "scaling": "strong",
           "ms_per_step": t * 1e3, "steps": args.o1280_steps,
           "config": workload_config(w, world), "rows_per_gpu": st.nrows,
           "effective_gbs": mine / t / 1e9, "roofline_frac": mine / t / 1e9 / peak,
           "path": f"StripStepper ({'periodic patch' if world == 1 else st.mode + ' exchange'})",
           "inputs": "on-device counter hash of global ids (identical for every N)",
           "l2": "no flush: per-GPU state >= 6.3 GB",
           "efficiency": "T1 / (N * T_N) with T1 = the N = 1 run's o1280_strong.ms_per_step",
           "sm_mhz_after_loop": sm_after,
           "isolated_step": {"ms_per_step": t_iso * 1e3, "roofline_frac": mine / t_iso / 1e9 / peak,
                             "how": "one step after 200 ms idle, median of 3 (SM clock at boost; the "
                                    "loop above runs long enough to reach the power cap)"}}
    del st
    torch.cuda.empty_cache()
    return rec


def e2e_time_loop(w: dict, steps: int) -> dict:
    """The reference's dependent time loop through the drop-in API on host Fields."""
    from paper_1908_06094_b200 import (MpdataParams, PatchSpec, TileSpec, build_geometry, build_mpdata,
                                       build_state, flat_to_field, halo_update, run_fused)
    from paper_1908_06094_b200.workloads import transport_inputs

    R, C, K = w["rows"], w["cols"], w["levels"]
    spec = PatchSpec(R, C, K)
    inp = transport_inputs(R, C, K, 0, "uniform", "gaussian-bump", "one", signs=False)
    state = build_state(spec)
    geo = build_geometry(spec, "uniform", seed=0)
    for name in ("pd_in", "vn", "wn", "rho"):
        f = getattr(state, name)
        flat_to_field(inp[{"pd_in": "pd"}.get(name, name)], f)
        halo_update(f)
    comp = build_mpdata(spec, state, geo, MpdataParams(DT, PIVBZ))
    tiles = TileSpec(R, C, 1)
    h = spec.halo

    def copy_core(src, dst):  # the reference's bench._copy_core (bench.py:430-435)
        values = src.array("primary", "r")[h:h + R, :, h:h + C, :, :]
        dst.array("primary", "rw")[h:h + R, :, h:h + C, :, :] = values
        halo_update(dst)

    times = []
    for step in range(steps + 2):  # two untimed warm-up steps
        t0 = time.perf_counter()
        if step:
            copy_core(state.pd_out, state.pd_in)
        run_fused(comp, tiles)
        times.append(time.perf_counter() - t0)
    times = times[2:]
    t = statistics.median(times)
    nb = state.pd_in.linear.total * 8
    return {"value": R * C * K / t, "unit": UNIT, "h2d_bytes_per_step": nb, "d2h_bytes_per_step": nb,
            "ms_per_step": t * 1e3, "step_ms": step_stats([x * 1e3 for x in times]),
            "api": f"reference loop (bench.py:398-403): _copy_core(pd_out, pd_in) on the host Fields, "
                   f"then run_fused(comp, TileSpec({R}, {C}, 1)); per step the pd_in host buffer "
                   "(page-locked LinearLayout) H2D + device reorder, fused step, reorder + pd_out D2H "
                   "into its host buffer, host core copy + halo refresh; dependent steps, no overlap"}


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1908_06094_b200 import PatchSpec, StructuredStepper, _lib
    from paper_1908_06094_b200.distributed import StripStepper
    from paper_1908_06094_b200.workloads import (mpdata_2d_bytes, mpdata_algorithmic_bytes,
                                                 paper_model_bytes, transport_inputs)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # the host baseline (N = 1 only), first, so it sees the same process state as the
    # reference arm's identical sample
    cpu = cpu_baseline(args, WORKLOADS[args.workload]) if not args.no_cpu and world == 1 else None
    # TSG_SHARE_ONE_GPU=1: every rank on cuda:0 with gloo -- exercises the N>1 code path on
    # a one-GPU box (not a performance configuration)
    shared = os.environ.get("TSG_SHARE_ONE_GPU") == "1"
    torch.cuda.set_device(0 if shared else local)
    if world > 1:
        dist.init_process_group("gloo" if shared else "nccl")
    if args.variant:
        _lib.call("tsg_set_fused_variant", args.variant)
    if args.no_band:
        _lib.call("tsg_set_fused_band", 0)

    def barrier():
        if world > 1:
            dist.barrier()

    args.exchange, exchange_note = _exchange_mode(args.exchange, rank, world, local, shared)
    w = WORKLOADS[args.workload]
    K, cols = w["levels"], w["cols"]
    cfg = workload_config(w, world)
    global_rows = cfg["rows"]
    GV = global_rows * cols  # vertices of the whole job
    peak, peak_src = _peaks()
    stream = torch.cuda.current_stream()
    with ClockSampler(0 if shared else local) as clocks:
        # every rank steps its strip through the same path at every N; the cfg3 strips carry
        # the reference's _transport_setup fields of one 279x256x80 patch each
        stepper = StripStepper(global_rows, cols, K, rank, world, seed=0, mode=args.exchange)
        if world > 1 and stepper.mode != args.exchange:  # peer mapping failed on some rank
            args.exchange, exchange_note = stepper.mode, stepper.fallback
        my_rows = stepper.nrows
        inp = None
        if args.workload == "cfg3":
            inp = transport_inputs(w["rows"], cols, K, 0, "uniform", "gaussian-bump", "one", signs=False)
            stepper.load_flat(inp["pd"], inp["vn"], inp["wn"], inp["rho"], inp["dual"].reshape(-1, 1))
        # L2 flush by READING 256 MiB (> 126 MB L2): leaves only clean lines behind, so the
        # timed step pays no write-back of someone else's dirty data
        flush = torch.ones(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
        flush_sink = torch.empty(1, dtype=torch.float64, device="cuda")

        def flush_l2():
            flush_sink.copy_(flush.sum().reshape(1))

        # warm-up: the timed loop itself (W dependent steps), then one flushed step sequence
        stepper.run(args.warmup, DT, PIVBZ)
        if world > 1:
            stepper.check()  # a broken exchange fails here, not after every timed step has timed out
        flush_l2()
        barrier()
        torch.cuda.synchronize()
        barrier()
        t_wall0 = time.perf_counter()
        t_run = _timed_run(stepper, args.steps, stream)  # the timed region: K dependent steps
        barrier()
        t_wall = time.perf_counter() - t_wall0
        if world > 1:
            stepper.finish()
            stepper.check()
        total_s = _max_over_ranks(t_run, world, shared)
        mean_step = total_s / args.steps
        value = GV * K / mean_step
        loop_launches = (_lib.lib().tsg_fused_loop_launches(stepper.grid.handle, args.steps)
                         if world == 1 or args.exchange == "p2p" else 3 * args.steps)
        # the flushed single-step sequence (round 1's protocol): per-step spread
        _timed_steps(stepper, min(args.warmup, 5), stream, flush_l2)
        if world > 1:
            stepper.check()
        barrier()
        step_ms = _timed_steps(stepper, args.flushed_steps, stream, flush_l2)
        barrier()
        if world > 1:
            stepper.finish()
            stepper.check()
        flushed_s = _max_over_ranks(sum(step_ms) / 1e3, world, shared) / len(step_ms)
        variant = _lib.lib().tsg_fused_variant_of(stepper.grid.handle, 0, my_rows)
        band = world == 1 and _lib.lib().tsg_fused_band_of(stepper.grid.handle, 0, my_rows) == 1
        hits = _lib.ctypes.c_int64()
        misses = _lib.ctypes.c_int64()
        _lib.call("tsg_launch_cache_stats", stepper.grid.handle, _lib.ctypes.byref(hits),
                  _lib.ctypes.byref(misses))
        del stepper
        torch.cuda.empty_cache()

        host_fed = args.workload == "cfg3"  # e2e at every N; the other host-fed records at N = 1
        e2e = e2e_all = loop = e2e_loop = None
        if host_fed:
            V = my_rows * cols
            st = StructuredStepper(PatchSpec(w["rows"], cols, K))
            sig = transport_inputs(w["rows"], cols, K, 0, "uniform", "gaussian-bump", "one")["signs"]
            st.set_geometry(sig, inp["dual"])
            st.upload(inp["pd"], inp["vn"], inp["wn"], inp["rho"])
            if cpu is not None and "cfg3" in CPU_PD_OUT:
                # the benchmarked kernel's result on these inputs against the CPU sample's own
                st.step(DT, PIVBZ)
                cpu["gpu_parity"] = {
                    "bitwise": bool(np.array_equal(st.download(), CPU_PD_OUT["cfg3"])),
                    "checked": "pd_out of one fused step (tsg_mpdata_step, dynamic deal) on the "
                               "benchmarked inputs vs the C port's result in this sample"}
            pinned = [torch.from_numpy(np.ascontiguousarray(inp[n])).pin_memory()
                      for n in ("pd", "vn", "wn", "rho")]
            outs = [torch.empty((V, K), dtype=torch.float64).pin_memory() for _ in range(2)]
            d2h = outs[0].numel() * 8
            e2e_steps = max(4, min(args.steps, 100))  # pipeline fill / drain amortised

            def e2e_run(step_inputs, api):
                st.run_pipelined([pinned] * 3, outs + outs[:1], DT, PIVBZ)  # warm-up (all inputs)
                torch.cuda.synchronize()
                barrier()
                e0, e1 = st.run_pipelined([step_inputs] * e2e_steps,
                                          [outs[n % 2] for n in range(e2e_steps)], DT, PIVBZ)
                torch.cuda.synchronize()
                barrier()
                t_e2e = _max_over_ranks(e0.elapsed_time(e1) / 1e3 / e2e_steps, world, shared)
                h2d = sum(t.numel() * 8 for t in step_inputs if t is not None)
                if world > 1:
                    api += (f"; at N = {world} every rank feeds its own 279x256x80 periodic patch from its "
                            "host (the weak-scaling per-GPU work; the strips' halo exchange is not on "
                            "the host-fed path), value = N x V K / the slowest rank's time, bytes per rank")
                return {"value": world * V * K / t_e2e, "unit": UNIT, "h2d_bytes_per_step": h2d,
                        "d2h_bytes_per_step": d2h, "ms_per_step": t_e2e * 1e3,
                        "pcie_gbs": (h2d + d2h) / t_e2e / 1e9, "api": api}

            e2e = e2e_run([pinned[0], None, None, None],
                          "independent host-fed steps: StructuredStepper.run_pipelined, each step "
                          "H2D of a density state pd (flat canonical, pinned), on-GPU reorder, fused "
                          "step, reorder, D2H of pd_out; vn / wn / rho resident (fixed, as in the "
                          "reference's loop); steps overlapped (H2D n+1 | GPU n | D2H n-1) since they "
                          "do not depend on each other -- see e2e_time_loop for the dependent loop")
            if world == 1:
                e2e_all = e2e_run(pinned, "independent host-fed steps as e2e, with every input (pd / vn / "
                                          "wn / rho, the flat oracle call of reference.py:93-116) copied "
                                          "H2D per step")
            if world == 1:
                # the same dependent loop with the static schedule (per-step launches replayed as a
                # captured two-step graph, round 1's loop) for comparison
                n_loop = args.steps
                _lib.call("tsg_set_fused_schedule", 1)
                try:
                    st.run(n_loop, DT, PIVBZ)
                    flush_l2()
                    torch.cuda.synchronize()
                    t_loop = _timed_run(st, n_loop, stream) / n_loop
                finally:
                    _lib.call("tsg_set_fused_schedule", 0)
                loop = {"value": V * K / t_loop, "unit": UNIT, "ms_per_step": t_loop * 1e3, "steps": n_loop,
                        "roofline_frac": mpdata_algorithmic_bytes(w["rows"], cols, K) / t_loop / 1e9 / peak,
                        "api": "StructuredStepper.run with tsg_set_fused_schedule(1): static per-CTA ranges, "
                               "one launch per step replayed as a captured two-step CUDA graph"}
                del st
                torch.cuda.empty_cache()
                try:  # informational beside e2e: never lose the line over it
                    e2e_loop = e2e_time_loop(w, max(5, min(args.steps, 20)))
                except Exception as exc:  # noqa: BLE001
                    e2e_loop = {"unavailable": f"{type(exc).__name__}: {exc}"}
            else:
                del st
                torch.cuda.empty_cache()
        o1280 = None
        if args.workload == "cfg3" and not args.no_o1280:
            o1280 = o1280_strong(args, rank, world, shared, barrier, peak)

    sustained = None
    if world == 1 and args.workload == "cfg3" and args.sustained_seconds > 0:
        # last, outside the clock sampler: the headline loop kept busy for a few seconds
        # settles under the board's power cap (and would slow every record after it)
        st = StripStepper(global_rows, cols, K, rank, world, seed=0, mode=args.exchange)
        st.load_flat(inp["pd"], inp["vn"], inp["wn"], inp["rho"], inp["dual"].reshape(-1, 1))
        t_end, last, watts = time.perf_counter() + args.sustained_seconds, [], []
        while time.perf_counter() < t_end:
            last.append(_timed_run(st, 200, stream) / 200)
            watts.append(_power_w(local))
        t_sus = statistics.median(last[len(last) // 2:])
        w_tail = [x for x in watts[len(watts) // 2:] if x is not None]
        p_sus = statistics.median(w_tail) if w_tail else None
        sustained = {"ms_per_step": t_sus * 1e3, "value": GV * K / t_sus,
                     "roofline_frac": mpdata_algorithmic_bytes(my_rows, cols, K) / t_sus / 1e9 / peak,
                     "sm_mhz_after": _sm_clock_mhz(local), "power_w": p_sus,
                     "updates_per_joule": GV * K / t_sus / p_sus if p_sus else None,
                     "how": f"the headline loop as back-to-back 200-step launches for "
                            f"{args.sustained_seconds:g} s after every other record, median of the second "
                            "half (the headline is taken within the first ~0.1 s of GPU work, at boost "
                            "clock); not part of the clock sampling"}
        del st

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    bcomp = mpdata_algorithmic_bytes(my_rows, cols, K)
    achieved = bcomp / mean_step / 1e9
    traffic, traffic_src = None, None
    tfile = ROOT / "profiles" / "fused_traffic.json"
    if tfile.exists() and world == 1 and args.workload == "cfg3":
        tj = json.loads(tfile.read_text())  # the ncu capture of the 279x256x80 loop kernel
        traffic, traffic_src = tj.get("dram_bytes_per_step"), tj.get("source")
    import ctypes

    vi = [ctypes.c_int() for _ in range(6)]
    _lib.lib().tsg_fused_variant_info(variant, *[ctypes.byref(x) for x in vi])
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": mean_step * 1e3, "higher_is_better": True,
        "scaling": w["scaling"], "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (" + ("the reference's _transport_setup fields of a 279x256x80 patch per strip"
                                 if args.workload == "cfg3" else "on-device counter-hash fields") + ")",
        "config": cfg,
        "setup": {"rows_per_gpu": my_rows, "vertices": GV, "edges": 3 * GV, "dt": DT, "pivbz": PIVBZ,
                  "path": "StripStepper" + (" (periodic patch)" if world == 1 else f" ({args.exchange})"),
                  "parallelism": f"row-strips x{world}",
                  "halo_exchange": ("none" if world == 1 else
                                    "inside the persistent loop launch: boundary-row epilogue stores "
                                    "into the neighbours' halos (CUDA IPC over NVLink), per-step "
                                    "neighbour flags acquired / released in the kernel"
                                    if args.exchange == "p2p" else "NCCL grouped send/recv"),
                  **({"exchange_fallback": exchange_note} if exchange_note else {}),
                  "l2": "no flush between the timed loop's steps (each streams 320 MB per rank through "
                        "the 126 MB L2); a 256 MiB read-only L2 flush before the timed region",
                  "timed_region": f"StripStepper.run({args.steps}): {args.steps} dependent steps (the "
                                  "reference's time loop, bench.py:398-403) in "
                                  f"{loop_launches} persistent launch(es) per rank",
                  "fused_schedule": "dynamic deal (global ticket: whole tiles in "
                                    + ("band" if band else "tile-major") + " order, the tail unit by "
                                    "unit); steps chained by per-tile step counters",
                  "fused_tile": {"variant": variant, "ti": vi[0].value, "tj": vi[1].value, "kc": vi[2].value,
                                 "stages": vi[3].value, "threads": vi[4].value, "smem_bytes": vi[5].value},
                  "launch_cache": {"hits": hits.value, "misses": misses.value}},
        "step_flushed": {
            "value": GV * K / flushed_s, "unit": UNIT, "ms_per_step": flushed_s * 1e3,
            "roofline_frac": bcomp / flushed_s / 1e9 / peak, "step_ms": step_stats(step_ms),
            "l2": "256 MiB read-only L2 flush before every step (outside its CUDA events)",
            "api": "StripStepper.step: one launch per step (round 1's headline protocol)"},
        "effective_gbs": achieved,
        "paper_model_gbs": paper_model_bytes(my_rows, cols, K) / mean_step / 1e9,
        "stage_updates_per_s": GV * (6 * K + 1) / mean_step,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                     "peak_source": peak_src, "algorithmic_bytes_per_launch": bcomp,
                     "bytes_2d_per_launch": mpdata_2d_bytes(my_rows, cols),
                     "per": "per step on rank 0: the persistent launch runs all K steps, so the "
                            "kernel time per step = launch time / K (CUDA events on its stream)"},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "e2e_all_inputs": e2e_all,
        "e2e_time_loop": e2e_loop,
        "time_loop": loop,
        "o1280_strong": o1280,
        "sustained": sustained,
        "gpu_launches": loop_launches,
        "clocks": clocks.summary(),
        "timed_wall_s": t_wall,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[1])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--flushed-steps", type=int, default=50,
                    help="steps of the step_flushed record (one launch each, L2 flushed before each)")
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--variant", type=int, default=0, help="fused tile variant (0 = default)")
    ap.add_argument("--no-band", action="store_true",
                    help="disable the band schedule of large patches (tall tiles instead)")
    ap.add_argument("--exchange", choices=("p2p", "nccl"), default="p2p",
                    help="N>1 halo exchange: fused P2P epilogue stores (default) or NCCL send/recv")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="cfg3",
                    help="cfg3 (headline, weak scaling) or o1280 (strong scaling)")
    ap.add_argument("--o1280-steps", type=int, default=20,
                    help="timed steps of the o1280_strong record (cfg3 runs)")
    ap.add_argument("--no-o1280", action="store_true", help="skip the o1280_strong record")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--sustained-seconds", type=float, default=3.0,
                    help="N = 1: also run the headline loop back to back this long (0: skip)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-python-ref", action="store_true",
                    help="reference arm: skip timing the reference package itself")
    ap.add_argument("--python-ref-reps", type=int, default=3)
    args = ap.parse_args(argv)
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
