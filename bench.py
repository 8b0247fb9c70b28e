#!/usr/bin/env python
"""Benchmark of the MPDATA transport step on B200 (contract: one JSON line on rank 0).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[2], the grid of the paper's Fig. 15): one
fused MPDATA transport step on the periodic 279 x 256 x 80 patch
(71,424 vertices = the paper's node count, 214,272 edges, 80 levels), fp64,
inputs as the reference's ``_transport_setup`` (gaussian-bump density,
U[-0.5,0.5) velocities, rho = 1, uniform geometry, dt = 0.1, pivbz = 1).

* value: grid-point updates/s (V*K per step / device time), inputs resident in
  HBM; each timed step is bracketed by CUDA events on the launching stream and
  preceded (outside the events) by a 256 MiB L2 flush, so no step reads the
  previous step's data from L2.
* e2e: the same metric through the public flat-array API (StructuredStepper)
  with pinned host buffers, as the reference's time loop runs it (bench.py:398-403:
  vn / wn / rho fixed, resident like model weights): per step H2D of the density
  state pd, on-GPU reorder into the structured layout, fused step, reorder back,
  D2H of pd_out.  ``e2e_all_inputs`` is the flat oracle call pattern
  (reference.py:93-116) instead: H2D of pd/vn/wn/rho every step.
* roofline: algorithmic bytes B_comp per step / average step time, against
  the measured HBM copy bandwidth (MEASURED_PEAKS.json).
* cpu_baseline / --impl reference: the reference algorithm restated in C
  (oracle/c, bitwise equal to the reference, OpenMP over all host cores).
* N > 1: weak scaling, one 279-row strip per rank of a (279*N) x 256 x 80
  patch, row-strip decomposition with a per-step halo exchange (NCCL).
"""

from __future__ import annotations

import argparse
import json
import os
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
ROWS, COLS, LEVELS = 279, 256, 80
WORKLOAD = WORKLOADS["cfg3"]["label"]


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy, burst)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

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
# CPU baseline (the reference algorithm restated in C; test/baseline infrastructure)


def cpu_reference_steps(steps: int, warmup: int, budget_s: float | None = None, rows=ROWS,
                        cols=COLS, levels=LEVELS):
    from oracle import c_oracle
    from oracle import tsg_oracle as O

    # every host core this process may run on (torchrun exports OMP_NUM_THREADS=1 per rank)
    c_oracle.set_threads(len(os.sched_getaffinity(0)))
    inp = O.transport_inputs(rows, cols, levels, 0, "uniform", "gaussian-bump", "one")
    e2v = O.neighbor_table(rows, cols, "edges", "vertices")
    v2e = O.neighbor_table(rows, cols, "vertices", "edges")
    args = (e2v, v2e, inp["signs"], inp["dual"], inp["pd"], inp["vn"], inp["wn"], inp["rho"], DT, PIVBZ)
    out = None
    for _ in range(warmup):
        out = c_oracle.transport_step(*args, out=out)
    times = []
    t_begin = time.perf_counter()
    while True:
        t0 = time.perf_counter()
        out = c_oracle.transport_step(*args, out=out)
        times.append(time.perf_counter() - t0)
        if budget_s is None and len(times) >= steps:
            break
        if budget_s is not None and (time.perf_counter() - t_begin > budget_s and len(times) >= 3):
            break
    return times, c_oracle.threads()


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    w = WORKLOADS[args.workload]
    r, c, k = w["cpu_rows"], w["cols"], w["levels"]
    steps = args.steps if args.workload == "cfg3" else min(args.steps, 2)
    times, threads = cpu_reference_steps(steps, min(args.warmup, 1 if args.workload != "cfg3" else args.warmup),
                                         rows=r, cols=c, levels=k)
    t = sum(times) / len(times)
    value = r * c * k / t
    sample = (f"full {r}x{c}x{k} step x {len(times)}" if r == w["rows"] else
              f"{r}x{c}x{k} periodic patch (1/{w['rows'] // r} of the workload; updates/s is "
              f"size-independent) x {len(times)}")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": len(times), "warmup": args.warmup, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": w["scaling"], "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": w["label"], "rows": w["rows"], "cols": c, "levels": k},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": sample + " (reference.transport_step restated in C, oracle/c)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1908_06094_b200 import PatchSpec, StructuredStepper, _lib
    from paper_1908_06094_b200.workloads import (mpdata_2d_bytes, mpdata_algorithmic_bytes,
                                                 paper_model_bytes, transport_inputs)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
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

    w = WORKLOADS[args.workload]
    K, cols = w["levels"], w["cols"]
    global_rows = w["rows"] * world if w["scaling"] == "weak" else w["rows"]
    GV = global_rows * cols  # vertices of the whole job
    host_fed = args.workload == "cfg3" and world == 1
    exchange_note = None
    if world > 1 and not shared and args.exchange == "p2p":
        # the fused exchange stores into the neighbours' memory: it needs peer access
        # (NVLink / NVSwitch); without it the NCCL send/recv exchange runs instead
        nbrs = {(local + 1) % world, (local - 1) % world} - {local}
        if not all(torch.cuda.can_device_access_peer(local, d) for d in nbrs):
            exchange_note = f"no peer access from cuda:{local} to {sorted(nbrs)}: NCCL exchange"
            args.exchange = "nccl"
        flag = torch.tensor([args.exchange == "nccl"], dtype=torch.int32, device="cuda")
        dist.all_reduce(flag, op=dist.ReduceOp.MAX)  # every rank takes the same exchange
        if flag.item():
            args.exchange = "nccl"
            exchange_note = exchange_note or "a rank lacks peer access to its neighbours: NCCL exchange"
    if not host_fed:
        from paper_1908_06094_b200.distributed import StripStepper

        stepper = StripStepper(global_rows, cols, K, rank, world, seed=0, mode=args.exchange)
        my_rows = stepper.nrows
    else:
        my_rows = ROWS
        inp = transport_inputs(ROWS, COLS, K, 0, "uniform", "gaussian-bump", "one")
        stepper = StructuredStepper(PatchSpec(ROWS, COLS, K))
        stepper.set_geometry(inp["signs"], inp["dual"])
        stepper.upload(inp["pd"], inp["vn"], inp["wn"], inp["rho"])
    stream = torch.cuda.current_stream()
    # L2 flush by READING 256 MiB (> 126 MB L2): leaves only clean lines behind, so the
    # timed step pays no write-back of someone else's dirty data
    flush = torch.ones(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
    flush_sink = torch.empty(1, dtype=torch.float64, device="cuda")

    def flush_l2():
        flush_sink.copy_(flush.sum().reshape(1))

    for _ in range(args.warmup):
        stepper.step(DT, PIVBZ)
        stepper.swap()
    torch.cuda.synchronize()
    if not host_fed:
        stepper.check()  # a broken exchange fails here, not after every timed step has timed out
    barrier()

    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    with ClockSampler(local) as clocks:
        barrier()
        torch.cuda.synchronize()
        t_wall0 = time.perf_counter()
        for s in range(args.steps):
            flush_l2()  # evict the previous step's data from L2 (outside the events)
            evs[s][0].record(stream)
            stepper.step(DT, PIVBZ)
            evs[s][1].record(stream)
            stepper.swap()
        torch.cuda.synchronize()
        barrier()
        t_wall = time.perf_counter() - t_wall0
    if not host_fed:
        stepper.finish()
        stepper.check()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    total_s = sum(step_ms) / 1e3
    if world > 1:
        t = torch.tensor([total_s], dtype=torch.float64, device="cpu" if shared else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_s = float(t.item())
    mean_step = total_s / args.steps
    value = GV * K / mean_step
    V = my_rows * cols

    # e2e through the public flat API from pinned host buffers (N=1): every step copies its
    # inputs H2D, reorders them into the structured layout, steps, reorders back and copies
    # pd_out D2H; StructuredStepper.run_pipelined overlaps step n+1's H2D with step n's GPU
    # work and step n-1's D2H (PCIe is full duplex).  Primary: the reference's time loop
    # (only the density state crosses PCIe, vn / wn / rho stay resident); secondary: the
    # flat oracle call pattern (every input every step).
    e2e = e2e_all = None
    if host_fed:
        pinned = [torch.from_numpy(np.ascontiguousarray(inp[n])).pin_memory()
                  for n in ("pd", "vn", "wn", "rho")]
        outs = [torch.empty((V, K), dtype=torch.float64).pin_memory() for _ in range(2)]
        d2h = outs[0].numel() * 8
        e2e_steps = max(4, min(args.steps, 40))

        def e2e_run(step_inputs, api):
            stepper.run_pipelined([pinned] * 3, outs + outs[:1], DT, PIVBZ)  # warm-up (all inputs)
            torch.cuda.synchronize()
            e0, e1 = stepper.run_pipelined([step_inputs] * e2e_steps,
                                           [outs[n % 2] for n in range(e2e_steps)], DT, PIVBZ)
            torch.cuda.synchronize()
            t_e2e = e0.elapsed_time(e1) / 1e3 / e2e_steps
            h2d = sum(t.numel() * 8 for t in step_inputs if t is not None)
            return {"value": V * K / t_e2e, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": t_e2e * 1e3,
                    "pcie_gbs": (h2d + d2h) / t_e2e / 1e9, "api": api}

        e2e = e2e_run([pinned[0], None, None, None],
                      "StructuredStepper.run_pipelined, the reference's time loop (bench.py:398-403): "
                      "per step H2D of the density state pd (flat canonical, pinned), on-GPU reorder, "
                      "fused step, reorder, D2H of pd_out; vn / wn / rho fixed and resident")
        e2e_all = e2e_run(pinned, "StructuredStepper.run_pipelined, the flat oracle call pattern "
                                  "(reference.py:93-116): H2D of pd / vn / wn / rho every step")

    # back-to-back time loop (tsg_mpdata_run ping-pong, no L2 flush: the 320 MB of inputs
    # exceed the 126 MB L2), the reference's bench loop (bench.py:398-403) -- informational
    loop = None
    if host_fed:
        n_loop = 100
        stepper.run(n_loop, DT, PIVBZ)
        torch.cuda.synchronize()
        l0, l1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        l0.record(stream)
        stepper.run(n_loop, DT, PIVBZ)
        l1.record(stream)
        torch.cuda.synchronize()
        t_loop = l0.elapsed_time(l1) / 1e3 / n_loop
        loop = {"value": V * K / t_loop, "unit": UNIT, "ms_per_step": t_loop * 1e3, "steps": n_loop,
                "l2": "no flush: inputs (320 MB) larger than L2",
                "api": "StructuredStepper.run (tsg_mpdata_run, one fused launch per step)"}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    peak, peak_src = _peaks()
    bcomp = mpdata_algorithmic_bytes(my_rows, cols, K)
    achieved = bcomp / mean_step / 1e9
    traffic = None
    tfile = ROOT / "profiles" / "fused_traffic.json"
    if tfile.exists() and host_fed:  # the ncu capture is of the 279x256x80 launch
        traffic = json.loads(tfile.read_text()).get("dram_bytes_per_launch")
    from paper_1908_06094_b200._lib import lib as _l
    import ctypes

    vi = [ctypes.c_int() for _ in range(6)]
    variant = _l().tsg_fused_variant_of(stepper.grid.handle, 0, my_rows)
    band = world == 1 and _l().tsg_fused_band_of(stepper.grid.handle, 0, my_rows) == 1
    _l().tsg_fused_variant_info(variant, *[ctypes.byref(x) for x in vi])
    cpu = None
    if not args.no_cpu and world == 1:  # the host baseline is measured at N = 1 only
        cr = w["cpu_rows"]
        times, threads = cpu_reference_steps(0, 1 if cr == w["rows"] else 0, budget_s=args.cpu_seconds,
                                             rows=cr, cols=cols, levels=K)
        tc = statistics.median(times)
        cpu = {"value": cr * cols * K / tc, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": (f"{cr}x{cols}x{K} periodic patch" + ("" if cr == w["rows"] else
                          f" (1/{w['rows'] // cr} of the per-job patch; updates/s is size-independent)"))
                         + f", step x {len(times)} (median), reference.transport_step restated in C "
                           "(oracle/c), OpenMP"}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": mean_step * 1e3, "higher_is_better": True,
        "scaling": w["scaling"], "vs_baseline": None, "dtype": "f64",
        "data": "synthetic" + ("" if host_fed else " (on-device counter-hash fields)"),
        "config": {"workload": w["label"], "rows": global_rows, "cols": cols, "levels": K,
                   "rows_per_gpu": my_rows, "vertices": GV, "edges": 3 * GV,
                   "dt": DT, "pivbz": PIVBZ, "parallelism": f"row-strips x{world}",
                   "halo_exchange": ("none" if world == 1 else
                                     "one launch per step: boundary-row epilogue stores into the "
                                     "neighbours' halos (CUDA IPC over NVLink), in-kernel step fence"
                                     if args.exchange == "p2p" else "NCCL grouped send/recv"),
                   **({"exchange_fallback": exchange_note} if exchange_note else {}),
                   "l2": "256 MiB read-only L2 flush before every timed step (outside the events)",
                   "fused_schedule": ("band round robin" if band else "contiguous ranges"),
                   "fused_tile": {"variant": variant, "ti": vi[0].value, "tj": vi[1].value, "kc": vi[2].value,
                                  "stages": vi[3].value, "threads": vi[4].value,
                                  "smem_bytes": vi[5].value}},
        "ms_per_step_median": statistics.median(step_ms) if step_ms else None,
        "effective_gbs": achieved,
        "paper_model_gbs": paper_model_bytes(my_rows, cols, K) / mean_step / 1e9,
        "stage_updates_per_s": GV * (6 * K + 1) / mean_step,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": bcomp,
                     "bytes_2d_per_launch": mpdata_2d_bytes(my_rows, cols),
                     "per": "rank 0's fused launch(es) per step"},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "e2e_all_inputs": e2e_all,
        "time_loop": loop,
        "gpu_launches": args.steps * (1 if world == 1 or args.exchange == "p2p" else 3),
        "clocks": clocks.summary(),
        "timed_wall_s": t_wall,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[1])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--variant", type=int, default=0, help="fused tile variant (0 = default)")
    ap.add_argument("--no-band", action="store_true",
                    help="disable the band schedule of large patches (tall tiles instead)")
    ap.add_argument("--exchange", choices=("p2p", "nccl"), default="p2p",
                    help="N>1 halo exchange: fused P2P epilogue stores (default) or NCCL send/recv")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="cfg3",
                    help="cfg3 (headline, weak scaling) or o1280 (strong scaling)")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
