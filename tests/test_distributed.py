"""Multi-GPU decomposition logic.

CPU (gloo, world size 2 and 3, spawned processes): the row-strip decomposition and the
per-step halo exchange move exactly the right rows, and strip-local steps with exchanged
halos reproduce the single-patch step bitwise (the oracle stands in for the device
step -- test infrastructure only).  GPU: several StripSteppers on one device with an
in-process exchanger reproduce the single-patch fused kernel bitwise, which exercises the
row-range kernel and the strip halo bookkeeping of the product path.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1908_06094_b200.distributed import RowStrips, exchange_halo_rows


def test_row_strips_balanced():
    s = RowStrips(10, 3)
    assert [s.strip(r) for r in range(3)] == [(0, 4), (4, 3), (7, 3)]
    assert s.up(0) == 2 and s.down(2) == 0
    with pytest.raises(ValueError):
        RowStrips(5, 3)


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _worker(rank, world, port, rows, cols, levels, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import tsg_oracle as O

        strips = RowStrips(rows, world)
        row0, nr = strips.strip(rank)
        # 1. exchange moves the right rows: fill interior with global row ids
        f = torch.full((nr + 2, 1, cols + 2, 4), -1.0)
        for r in range(nr):
            f[r + 1] = float(row0 + r)
        for w in exchange_halo_rows(f, nr, rank, world):
            w.wait()
        ok1 = (f[0].eq(float((row0 - 1) % rows)).all().item()
               and f[nr + 1].eq(float((row0 + nr) % rows)).all().item())
        # 2. strip-local oracle steps with exchanged pd halos == the global step, 3 steps
        inp = O.transport_inputs(rows, cols, levels, 3, "random", "random", "random")
        pd = inp["pd"].reshape(rows, cols, levels)
        ext = np.arange(row0 - 1, row0 + nr + 1) % rows  # strip + halo rows (global ids)
        loc = {k: inp[k].reshape(rows, -1, cols, inp[k].shape[-1] if inp[k].ndim > 1 else 1)[ext]
               for k in ("vn", "wn", "rho", "signs")}
        dual = inp["dual"].reshape(rows, cols)[ext]
        mine = torch.from_numpy(np.ascontiguousarray(pd[ext]))  # [nr+2, cols, K]
        gpd = inp["pd"]
        lr = nr + 2
        e2v = O.neighbor_table(lr, cols, "edges", "vertices")
        v2e = O.neighbor_table(lr, cols, "vertices", "edges")
        for _ in range(3):
            out = O.transport_step(e2v, v2e, loc["signs"].reshape(-1, 6), dual.reshape(-1),
                                   mine.numpy().reshape(-1, levels), loc["vn"].reshape(-1, levels),
                                   loc["wn"].reshape(-1, levels + 1), loc["rho"].reshape(-1, levels),
                                   0.2, 0.8)["pd_out"].reshape(lr, cols, levels)
            mine = torch.from_numpy(np.ascontiguousarray(out))
            for w in exchange_halo_rows(mine, nr, rank, world):
                w.wait()
            gpd = O.step_inputs(rows, cols, dict(inp, pd=gpd), 0.2, 0.8)["pd_out"]
        want = gpd.reshape(rows, cols, levels)[row0:row0 + nr]
        ok2 = np.array_equal(mine.numpy()[1:nr + 1], want)
        q.put((rank, bool(ok1), bool(ok2)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_strip_exchange_and_decomposition_invariance(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, 9, 5, 4, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs)
    assert all(ok1 and ok2 for _, ok1, ok2 in res), res


@pytest.mark.gpu
def test_strip_steppers_on_one_gpu_match_single_patch(cuda_ok):
    """Row-range fused kernel + strip halos == periodic single-patch step, bitwise."""
    from paper_1908_06094_b200.distributed import StripStepper

    rows, cols, K, world = 23, 37, 21, 3
    reg = {}

    def exchange(field, nrows, rank, world_, group):
        reg.setdefault(id(field), (rank, field))
        return []

    single = StripStepper(rows, cols, K, 0, 1, seed=5)
    steppers = [StripStepper(rows, cols, K, r, world, seed=5, exchange=exchange) for r in range(world)]

    def halo(name):
        for r, s in enumerate(steppers):
            up, down = steppers[(r - 1) % world], steppers[(r + 1) % world]
            getattr(s, name)[0] = getattr(up, name)[up.nrows]
            getattr(s, name)[s.nrows + 1] = getattr(down, name)[1]

    for name in ("pd", "vn", "wn", "rho", "dual"):
        halo(name)
    for _ in range(4):
        single.step(0.2, 0.8)
        single.swap()
        for s in steppers:
            s._launch(1, s.nrows - 1, 0.2, 0.8, torch.cuda.current_stream())
            s._launch(0, 1, 0.2, 0.8, torch.cuda.current_stream())
            s._launch(s.nrows - 1, s.nrows, 0.2, 0.8, torch.cuda.current_stream())
        for s in steppers:
            s.swap()
        halo("pd")
    torch.cuda.synchronize()
    got = torch.cat([s.interior("pd") for s in steppers], 0)
    assert torch.equal(got, single.interior("pd"))


@pytest.mark.gpu
@pytest.mark.parametrize("world,shape", [(2, (16, 29, 18)), (3, (23, 37, 21)), (4, (64, 40, 33))])
def test_nccl_mode_step_with_in_process_exchanger(cuda_ok, world, shape):
    """StripStepper.step() in mode="nccl" end to end: interior rows overlapped with the
    previous exchange, wait on the pending requests, boundary rows, then the exchange of
    pd_out issued on the comm stream after a recorded event -- with LocalRing standing in
    for batch_isend_irecv (device copies on the comm stream, waitable requests covering
    sends and receives).  Bitwise equal to the single-patch step after 5 steps."""
    from paper_1908_06094_b200.distributed import LocalRing, StripStepper

    rows, cols, K = shape
    ring = LocalRing()
    steppers = [StripStepper(rows, cols, K, r, world, seed=11, exchange=ring, mode="nccl")
                for r in range(world)]
    for st in steppers:
        ring.add(st)
    ring.static()
    single = StripStepper(rows, cols, K, 0, 1, seed=11)
    for _ in range(5):
        single.step(0.2, 0.8)
        single.swap()
        for st in steppers:
            st.step(0.2, 0.8)
        for st in steppers:
            st.swap()
    for st in steppers:
        st.finish()
    torch.cuda.synchronize()
    assert all(st.comm is not torch.cuda.current_stream() for st in steppers)
    got = torch.cat([st.interior("pd") for st in steppers], 0)
    assert torch.equal(got, single.interior("pd"))
    # the pd_out halo rows received by the last exchange hold the neighbours' rows
    for r, st in enumerate(steppers):
        up, down = steppers[(r - 1) % world], steppers[(r + 1) % world]
        assert torch.equal(st.pd[0], up.pd[up.nrows]) and torch.equal(st.pd[st.nrows + 1], down.pd[1])


@pytest.mark.gpu
def test_strip_load_flat_matches_the_oracle(cuda_ok):
    """load_flat: the reference's flat inputs (row slices per strip) -> strips; one patch
    (world 1) and 3 in-process strips both equal the oracle's step bitwise."""
    from oracle import tsg_oracle as O
    from paper_1908_06094_b200.distributed import LocalRing, StripStepper

    rows, cols, K, dt, pivbz = 21, 26, 12, 0.2, 0.8
    inp = O.transport_inputs(rows, cols, K, 4, "uniform", "random", "random")
    want = O.step_inputs(rows, cols, inp, dt, pivbz)["pd_out"].reshape(rows, cols, K)

    def rows_of(name, r0, n):
        a = inp[name]
        per = a.shape[0] // rows
        return a[r0 * per:(r0 + n) * per]

    single = StripStepper(rows, cols, K, 0, 1)
    single.load_flat(inp["pd"], inp["vn"], inp["wn"], inp["rho"], inp["dual"].reshape(-1, 1))
    single.step(dt, pivbz)
    torch.cuda.synchronize()
    assert np.array_equal(single.interior("pd_out")[:, 0, :, :K].cpu().numpy(), want)
    ring = LocalRing()
    steppers = [StripStepper(rows, cols, K, r, 3, exchange=ring) for r in range(3)]
    for st in steppers:
        ring.add(st)
    for st in steppers:
        st.load_flat(*(rows_of(n, st.row0, st.nrows) for n in ("pd", "vn", "wn", "rho")),
                     rows_of("dual", st.row0, st.nrows).reshape(-1, 1))
    torch.cuda.synchronize()
    for st in steppers:
        st.step(dt, pivbz)
    torch.cuda.synchronize()
    got = torch.cat([st.interior("pd_out") for st in steppers], 0)[:, 0, :, :K].cpu().numpy()
    assert np.array_equal(got, want)
    with pytest.raises(ValueError, match="values for this strip"):
        single.load_flat(inp["pd"][:-1], inp["vn"], inp["wn"], inp["rho"])


def _p2p_worker(rank, world, port, q, single_launch=True, graph=False, shape=(17, 29, 18)):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1908_06094_b200.distributed import StripStepper

        rows, cols, K = shape
        st = StripStepper(rows, cols, K, rank, world, seed=7, mode="p2p", timeout_ms=60000,
                          single_launch=single_launch)
        if graph == "mixed":  # persistent loops and single-launch steps share the step counter
            st.run(2, 0.2, 0.8)
            st.step(0.2, 0.8)
            st.swap()
            st.run(3, 0.2, 0.8)
        elif graph:  # 1 + 5 steps: persistent loop launches (or the captured graph), odd tail
            st.run(1, 0.2, 0.8)
            st.run(5, 0.2, 0.8)
        else:
            for _ in range(6):
                st.step(0.2, 0.8)
                st.swap()
        torch.cuda.synchronize()
        st.check()
        dist.barrier()  # every rank's last step has landed in its neighbours' halos
        mine = st.interior("pd").cpu()
        parts = [None] * world
        dist.all_gather_object(parts, (st.row0, mine))
        ok = None
        if rank == 0:
            single = StripStepper(rows, cols, K, 0, 1, seed=7)
            for _ in range(6):
                single.step(0.2, 0.8)
                single.swap()
            want = single.interior("pd").cpu()
            got = torch.cat([p for _, p in sorted(parts, key=lambda x: x[0])], 0)
            ok = bool(torch.equal(got, want))
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world,single_launch,graph,shape", [
    (2, True, False, (17, 29, 18)), (2, False, False, (17, 29, 18)), (3, True, False, (17, 29, 18)),
    (2, True, True, (17, 29, 18)), (3, True, True, (17, 29, 18)), (2, True, "mixed", (17, 29, 18)),
    (2, True, True, (9, 40, 80)),
    # four ranks, uneven strips (6 / 6 / 6 / 5 rows: tile rows cut by strip edges)
    (4, True, True, (23, 29, 18)),
    # strips large enough for the band schedule (interior rows banded, boundary rows last)
    (2, True, True, (512, 608, 32))])
def test_p2p_fused_exchange_processes_share_one_gpu(cuda_ok, world, single_launch, graph, shape):
    """Ranks (processes) on one GPU: IPC-mapped density buffers, boundary rows stored
    straight into the neighbour's halo by the step kernel, device-side step fence -- the
    multi-GPU fused-exchange path end to end, as one launch per step (in-kernel fence and
    release) or as the five-launch sequence; result == single-patch step bitwise."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_p2p_worker, args=(r, world, port, q, single_launch, graph, shape))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs)
    r0 = [r for r in res if r[0] == 0][0]
    assert r0[1] is True, res
