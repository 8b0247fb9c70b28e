"""GPU tests of the fused kernel's work deal (csrc/mpdata_dyn.cu): the dynamically dealt
single step and the persistent multi-step loop (tsg_mpdata_run) against the static
schedule and the oracle, bitwise.  The arithmetic contract is SURVEY Appendix A
(reference.py:93-116); the loop is the reference's time loop (bench.py:398-403) with the
pd_in / pd_out ping-pong in place of its core copy."""

import numpy as np
import pytest

from oracle import tsg_oracle as O

pytestmark = pytest.mark.gpu

T = pytest.importorskip("paper_1908_06094_b200")


def _stepper(shape, seed):
    r, c, k = shape
    inp = O.transport_inputs(r, c, k, seed, "random", "random", "random")
    st = T.StructuredStepper(T.PatchSpec(r, c, k))
    st.set_geometry(inp["signs"], inp["dual"])
    st.upload(inp["pd"], inp["vn"], inp["wn"], inp["rho"])
    return inp, st


def _schedule(sched):
    from paper_1908_06094_b200 import _lib

    _lib.call("tsg_set_fused_schedule", sched)


def _wait_error(st):
    import ctypes

    from paper_1908_06094_b200 import _lib

    err = ctypes.c_int(-1)
    _lib.call("tsg_fused_wait_error", st.grid.handle, ctypes.byref(err))
    return err.value


@pytest.mark.parametrize("shape", [(279, 256, 80), (37, 45, 50), (2, 2, 2), (6, 70, 137), (9, 300, 17)])
def test_dynamic_step_matches_oracle_and_static(cuda_ok, shape):
    import torch

    inp, st = _stepper(shape, 3)
    want = O.step_inputs(shape[0], shape[1], inp, 0.2, 0.8)["pd_out"] if shape[0] * shape[1] < 20000 else None
    got = {}
    try:
        for sched in (1, 0):
            _schedule(sched)
            st.step(0.2, 0.8)
            got[sched] = st.download()
    finally:
        _schedule(0)
    torch.cuda.synchronize()
    assert np.array_equal(got[0], got[1])
    if want is not None:
        assert np.array_equal(got[0], want)


@pytest.mark.parametrize("shape", [(279, 256, 80), (13, 21, 20), (2, 2, 3), (5, 33, 2)])
@pytest.mark.parametrize("steps", [2, 3, 7])
def test_persistent_loop_matches_repeated_steps(cuda_ok, shape, steps):
    """One multi-step launch == the static schedule's captured loop == single steps."""
    inp, st = _stepper(shape, 5)
    res = {}
    try:
        for sched in (1, 0):
            _schedule(sched)
            st.upload(inp["pd"], inp["vn"], inp["wn"], inp["rho"])
            st.run(steps, 0.1, 1.0)
            res[sched] = st.download()
    finally:
        _schedule(0)
    assert _wait_error(st) == 0
    # reference loop on the host oracle for small cases
    if shape[0] * shape[1] * shape[2] <= 20000:
        pd = inp["pd"].copy()
        for _ in range(steps):
            pd = O.step_inputs(shape[0], shape[1], dict(inp, pd=pd), 0.1, 1.0)["pd_out"]
        assert np.array_equal(res[0], pd)
    assert np.array_equal(res[0], res[1])


def test_persistent_loop_parity_across_calls(cuda_ok):
    """An odd loop leaves the state in the other buffer; the next loop starts from it."""
    shape = (20, 40, 24)
    inp, st = _stepper(shape, 8)
    st.run(3, 0.1, 1.0)
    st.swap()  # the newest density becomes the input (as after step())
    st.run(4, 0.1, 1.0)
    a = st.download()
    inp2, st2 = _stepper(shape, 8)
    for _ in range(7):
        st2.step(0.1, 1.0)
        st2.swap()
    b = st2.fetch("pd")
    assert np.array_equal(a, b)
    assert _wait_error(st) == 0


def test_dynamic_deal_balances_the_ctas(cuda_ok):
    """Every CTA of a dynamically dealt step takes work and the units add up."""
    import ctypes

    import torch

    from paper_1908_06094_b200 import _lib

    inp, st = _stepper((279, 256, 80), 0)
    tr = torch.zeros(4 * 148 * 4, dtype=torch.int64, device="cuda")
    _lib.call("tsg_debug_trace", ctypes.c_void_p(tr.data_ptr()))
    try:
        st.step(0.1, 1.0)
        torch.cuda.synchronize()
    finally:
        _lib.call("tsg_debug_trace", None)
    t = tr.view(-1, 4).cpu().numpy()
    t = t[t[:, 0] > 0]
    units = t[:, 3]
    assert units.sum() == 70 * 16 * 5  # tiles x chunks of the 4x16x16 unit
    assert units.min() >= 1


def test_strip_stepper_run_on_one_gpu_is_the_persistent_loop(cuda_ok):
    """StripStepper(world=1).run(n) (tsg_mpdata_run) == n x (step; swap), both parities."""
    from paper_1908_06094_b200.distributed import StripStepper

    for n in (4, 5):
        a = StripStepper(31, 48, 33, 0, 1, seed=2)
        b = StripStepper(31, 48, 33, 0, 1, seed=2)
        a.run(n, 0.2, 0.8)
        for _ in range(n):
            b.step(0.2, 0.8)
            b.swap()
        assert np.array_equal(a.interior("pd").cpu().numpy(), b.interior("pd").cpu().numpy())
        assert a.steps_done == b.steps_done == n


def test_long_persistent_loops_match_single_steps(cuda_ok):
    """A 501-step launch, then a second one of 250 steps on the same handle (the tile
    counters' base carried across launches), equals 751 single launches bitwise."""
    shape = (37, 45, 50)
    inp, st = _stepper(shape, 9)
    st.run(501, 0.1, 1.0)
    st.swap()
    st.run(250, 0.1, 1.0)
    a = st.download()
    assert _wait_error(st) == 0
    inp2, st2 = _stepper(shape, 9)
    for _ in range(751):
        st2.step(0.1, 1.0)
        st2.swap()
    assert np.array_equal(a, st2.fetch("pd"))
