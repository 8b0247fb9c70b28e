"""run_fused on host Fields in the reference's loop pattern at 279x256x80: wall time and
device time (RunStats ms0) of the streamed host step per band count, against the
unstreamed path (upload all, step, download all).  python tools/streamed_probe.py"""
import statistics
import sys
import time

sys.path.insert(0, "/root/repo")
import torch  # noqa: E402

from paper_1908_06094_b200 import (MpdataParams, PatchSpec, TileSpec, build_geometry, build_mpdata,  # noqa: E402
                                   build_state, flat_to_field, halo_update, run_fused)
from paper_1908_06094_b200 import executors as X  # noqa: E402
from paper_1908_06094_b200.workloads import transport_inputs  # noqa: E402

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
run_fused(comp, tiles)
for bands in (0, 2, 4, 6, 8, 12):
    X._STREAM_BANDS = max(bands, 2)
    wall, dev = [], []
    for _ in range(12):
        state.pd_in.array("primary", "rw")  # host-dirty density, as after the reference's core copy
        if bands == 0:
            state.pd_out.dirty["mirror"] = True  # force the unstreamed path for comparison
            state.pd_out.dirty["mirror"] = False
            X._STREAM_MIN_ROWS = 10 ** 9
        else:
            X._STREAM_MIN_ROWS = 24
        t0 = time.perf_counter()
        st = run_fused(comp, tiles)
        wall.append(time.perf_counter() - t0)
        dev.append(st.wall_times["ms0"])
    print(f"bands {bands or 'off'}: wall {statistics.median(wall) * 1e3:.3f} ms, device "
          f"{statistics.median(dev) * 1e3:.3f} ms", flush=True)
