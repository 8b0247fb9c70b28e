"""Event timeline of one streamed run_fused (tools/streamed_probe.py setup): when each band's upload,
pack, step, unpack and download end, relative to the first upload."""
import sys
sys.path.insert(0, "/root/repo")
import torch
from paper_1908_06094_b200 import (MpdataParams, PatchSpec, TileSpec, build_geometry, build_mpdata, build_state, flat_to_field, halo_update, run_fused, _lib)
from paper_1908_06094_b200 import executors as X
from paper_1908_06094_b200.workloads import transport_inputs
R, C, K = 279, 256, 80
spec = PatchSpec(R, C, K)
inp = transport_inputs(R, C, K, 0, "uniform", "gaussian-bump", "one", signs=False)
state = build_state(spec); geo = build_geometry(spec, "uniform", seed=0)
for name in ("pd_in", "vn", "wn", "rho"):
    f = getattr(state, name); flat_to_field(inp[{"pd_in": "pd"}.get(name, name)], f); halo_update(f)
comp = build_mpdata(spec, state, geo, MpdataParams(0.1, 1.0))
run_fused(comp, TileSpec(R, C, 1))
X._STREAM_BANDS = 6
# monkeypatch: record events after each op
log = []
orig_call = _lib.call
def call(name, *a):
    r = orig_call(name, *a)
    if name in ("tsg_memcpy2d", "tsg_pack_strided_rows", "tsg_mpdata_step_rows", "tsg_unpack_strided_rows"):
        st = a[-1]
        import ctypes
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(torch.cuda.ExternalStream(st.value) if st.value else torch.cuda.current_stream())
        log.append((name, ev))
    return r
_lib.call = call
for it in range(3):
    log.clear()
    state.pd_in.array("primary", "rw")
    t0 = torch.cuda.Event(enable_timing=True); t0.record()
    st = run_fused(comp, TileSpec(R, C, 1))
    torch.cuda.synchronize()
print("device", st.wall_times["ms0"] * 1e3)
base = log[0][1]
for name, ev in log:
    print(f"{name:28s} {base.elapsed_time(ev) * 1e3:8.1f} us")
