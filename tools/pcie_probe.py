"""PCIe probe: H2D and D2H of a 45.7 MB density state (pinned host memory), alone and
concurrently, as one copy or split over several streams (copy engines).
python tools/pcie_probe.py"""
import torch

N = 71424 * 80
h_in = torch.rand(N, dtype=torch.float64).pin_memory()
h_out = torch.empty(N, dtype=torch.float64).pin_memory()
d_in = torch.empty(N, dtype=torch.float64, device="cuda")
d_out = torch.rand(N, dtype=torch.float64, device="cuda")
streams = [torch.cuda.Stream() for _ in range(16)]


def run(split, h2d=True, d2h=True, reps=20):
    cur = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for it in range(reps + 2):
        if it == 2:
            torch.cuda.synchronize()
            a.record(cur)
        evs = []
        for q in range(split):
            lo, hi = N * q // split, N * (q + 1) // split
            if h2d:
                s = streams[q]
                s.wait_stream(cur)
                with torch.cuda.stream(s):
                    d_in[lo:hi].copy_(h_in[lo:hi], non_blocking=True)
                evs.append(s)
            if d2h:
                s = streams[8 + q]
                s.wait_stream(cur)
                with torch.cuda.stream(s):
                    h_out[lo:hi].copy_(d_out[lo:hi], non_blocking=True)
                evs.append(s)
        for s in evs:
            cur.wait_stream(s)
    b.record(cur)
    torch.cuda.synchronize()
    t = a.elapsed_time(b) / reps / 1e3
    nb = N * 8 * (int(h2d) + int(d2h))
    print(f"split {split} h2d {h2d} d2h {d2h}: {t * 1e3:.3f} ms  {nb / t / 1e9:.1f} GB/s total", flush=True)


for split in (1, 2, 4, 8):
    run(split, True, False)
    run(split, False, True)
    run(split, True, True)
