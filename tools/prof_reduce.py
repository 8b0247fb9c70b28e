"""Run the V->V structured reduce a few times at 256x256x80 (ncu target)."""
import sys
sys.path.insert(0, "/root/repo")
import torch
from paper_1908_06094_b200 import _lib
from paper_1908_06094_b200.device import DeviceGrid
g = DeviceGrid(256, 256, 80)
s = _lib.stream_handle()
src, dst = g.empty(0, 80), g.empty(0, 80)
_lib.call("tsg_fill_hash", g.handle, 0, 80, 3, 0.0, 1.0, _lib.ptr(src), s)
for _ in range(4):
    _lib.call("tsg_neighbor_reduce", g.handle, 0, 0, 80, _lib.ptr(src), None, _lib.ptr(dst), s)
torch.cuda.synchronize()
