"""cfg5 parity at full size: the O1280-class patch (2560x2576x137) stepped as
two (or more) row strips in as many processes sharing one GPU (the persistent strip loop:
fused P2P exchange, per-step neighbour flags inside one launch) against the single-patch
persistent loop and the static per-step schedule, compared bitwise through a device-side
hash of every interior row.  Needs ~110 GB of device memory; not part of the test suite.

    python tools/o1280_strips_check.py [steps] [strips]
"""
import os
import socket
import sys

sys.path.insert(0, "/root/repo")
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROWS, COLS, K = 2560, 2576, 137


def row_hashes(t: torch.Tensor) -> torch.Tensor:
    """One 64-bit mixing hash per storage row of a [rows, colors, cols, inner] fp64 tensor."""
    x = t.contiguous().view(torch.int64)
    mix = x * 0x9E3779B97F4A7C15 + (x >> 29)
    return mix.reshape(t.shape[0], -1).sum(dim=1)


def worker(rank, world, port, steps, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1908_06094_b200.distributed import StripStepper

    st = StripStepper(ROWS, COLS, K, rank, world, seed=11, mode="p2p", timeout_ms=600000)
    st.run(steps, 0.05, 0.9)
    torch.cuda.synchronize()
    st.check()
    dist.barrier()
    mine = (st.row0, row_hashes(st.interior("pd")[..., :K]).cpu())
    del st
    torch.cuda.empty_cache()
    parts = [None] * world
    dist.all_gather_object(parts, mine)
    if rank == 0:
        from paper_1908_06094_b200 import _lib

        got = torch.cat([h for _, h in sorted(parts, key=lambda p: p[0])])
        res = {}
        for sched in (0, 1):  # the persistent loop, and the static per-step schedule
            _lib.call("tsg_set_fused_schedule", sched)
            single = StripStepper(ROWS, COLS, K, 0, 1, seed=11)
            single.run(steps, 0.05, 0.9)
            torch.cuda.synchronize()
            res[sched] = row_hashes(single.interior("pd")[..., :K]).cpu()
            del single
            torch.cuda.empty_cache()
        _lib.call("tsg_set_fused_schedule", 0)
        q.put((bool(torch.equal(got, res[0])), bool(torch.equal(res[0], res[1])), int(got.numel())))
    dist.destroy_process_group()


if __name__ == "__main__":
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    world = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=worker, args=(r, world, port, steps, q)) for r in range(world)]
    for p in ps:
        p.start()
    ok, ok_static, nrows = q.get(timeout=3000)
    for p in ps:
        p.join()
    print(f"O1280 {ROWS}x{COLS}x{K}, {world} strips (persistent strip loops, fused P2P exchange) vs "
          f"the single patch (persistent loop), {steps} steps, {nrows} row hashes: "
          f"bitwise {'EQUAL' if ok else 'DIFFERENT'}; single patch persistent loop vs static "
          f"per-step schedule: {'EQUAL' if ok_static else 'DIFFERENT'}", flush=True)
