"""Host<->device 2-D copies of row bands of a level-outer host layout (279x256x80) vs one
1-D copy: does a band-strided DMA run at the link rate?"""
import sys, time
sys.path.insert(0, "/root/repo")
import torch, ctypes
from paper_1908_06094_b200 import _lib
R, C, K = 279, 256, 80
rs = 264  # row stride (elements) of the default host layout at this size
plane = (R + 2) * rs
n = plane * K
h = torch.rand(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")
h2 = torch.empty(n, dtype=torch.float64).pin_memory()
def t(fn, reps=20):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
s = _lib.stream_handle()
one = lambda: d.copy_(h, non_blocking=True)
def bands(B, kind=1):
    cuts = [1 + (R * i) // B for i in range(B + 1)]
    for i in range(B):
        lo, hi = cuts[i], cuts[i + 1]
        off = 8 * lo * rs
        w = 8 * (hi - lo) * rs
        if kind == 1:
            _lib.call("tsg_memcpy2d", ctypes.c_void_p(d.data_ptr() + off), 8 * plane, ctypes.c_void_p(h.data_ptr() + off), 8 * plane, w, K, 1, s)
        else:
            _lib.call("tsg_memcpy2d", ctypes.c_void_p(h2.data_ptr() + off), 8 * plane, ctypes.c_void_p(d.data_ptr() + off), 8 * plane, w, K, 2, s)
print("1D H2D full", round(t(one), 3), "ms")
for B in (1, 2, 6, 12):
    print(f"2D H2D {B} bands", round(t(lambda: bands(B)), 3), "ms", " D2H", round(t(lambda: bands(B, 2)), 3), "ms")

# concurrency: H2D bands on one stream while D2H bands run on another
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def both(B, two_d=True):
    cuts = [1 + (R * i) // B for i in range(B + 1)]
    for i in range(B):
        lo, hi = cuts[i], cuts[i + 1]
        off, w = 8 * lo * rs, 8 * (hi - lo) * rs
        if two_d:
            _lib.call("tsg_memcpy2d", ctypes.c_void_p(d.data_ptr() + off), 8 * plane,
                      ctypes.c_void_p(h.data_ptr() + off), 8 * plane, w, K, 1, _lib.stream_handle(s1))
            _lib.call("tsg_memcpy2d", ctypes.c_void_p(h2.data_ptr() + off), 8 * plane,
                      ctypes.c_void_p(d2.data_ptr() + off), 8 * plane, w, K, 2, _lib.stream_handle(s2))
        else:
            a, b = n * i // B, n * (i + 1) // B
            with torch.cuda.stream(s1):
                d[a:b].copy_(h[a:b], non_blocking=True)
            with torch.cuda.stream(s2):
                h2[a:b].copy_(d2[a:b], non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


d2 = torch.rand(n, dtype=torch.float64, device="cuda")
for B in (1, 6, 12):
    print(f"concurrent H2D + D2H, {B} bands: 2-D {t(lambda: both(B)):.3f} ms, 1-D {t(lambda: both(B, False)):.3f} ms")
