"""Where the reference's dependent loop (bench.py:398-403) spends its time through the
drop-in API at 279x256x80: the host core copy + halo refresh of the reference's own
_copy_core, and run_fused (pd_in upload + device reorder, the fused step, reorder +
pd_out download).  python tools/e2e_loop_breakdown.py [steps]"""
import statistics
import sys
import time

sys.path.insert(0, "/root/repo")
import torch  # noqa: E402

from paper_1908_06094_b200 import (MpdataParams, PatchSpec, TileSpec, build_geometry, build_mpdata,  # noqa: E402
                                   build_state, flat_to_field, halo_update, run_fused, sync)
from paper_1908_06094_b200.workloads import transport_inputs  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
R, C, K = 279, 256, 80
spec = PatchSpec(R, C, K)
inp = transport_inputs(R, C, K, 0, "uniform", "gaussian-bump", "one", signs=False)
state = build_state(spec)
geo = build_geometry(spec, "uniform", seed=0)
for name in ("pd_in", "vn", "wn", "rho"):
    f = getattr(state, name)
    flat_to_field(inp[{"pd_in": "pd"}.get(name, name)], f)
    halo_update(f)
comp = build_mpdata(spec, state, geo, MpdataParams(0.1, 1.0))
tiles = TileSpec(R, C, 1)
h = spec.halo
T = {"copy": [], "halo": [], "run_fused": [], "upload": [], "download": []}
for step in range(steps + 2):
    t0 = time.perf_counter()
    if step:
        values = state.pd_out.array("primary", "r")[h:h + R, :, h:h + C, :, :]
        state.pd_in.array("primary", "rw")[h:h + R, :, h:h + C, :, :] = values
    t1 = time.perf_counter()
    if step:
        halo_update(state.pd_in)
    t2 = time.perf_counter()
    run_fused(comp, tiles)
    t3 = time.perf_counter()
    if step >= 2:
        T["copy"].append(t1 - t0)
        T["halo"].append(t2 - t1)
        T["run_fused"].append(t3 - t2)
# the transfers alone
for _ in range(steps):
    state.pd_in.array("primary", "rw")
    t0 = time.perf_counter()
    sync(state.pd_in, "mirror")
    t1 = time.perf_counter()
    state.pd_out.mark_device_written()
    sync(state.pd_out, "primary")
    t2 = time.perf_counter()
    T["upload"].append(t1 - t0)
    T["download"].append(t2 - t1)
for k, v in T.items():
    print(f"{k:10s} median {statistics.median(v) * 1e3:7.3f} ms  min {min(v) * 1e3:7.3f}")
print(f"threads: torch {torch.get_num_threads()}")
