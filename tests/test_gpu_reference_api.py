"""GPU tests of ``paper_1908_06094_b200.reference``, the drop-in for the reference's flat
stage API (reference.py:1-160): every stage function against the oracle, bitwise, under
the canonical and a relabelled (UN) numbering, at even, odd and single-level counts and on
1-D arrays; numpy in -> numpy out, CUDA in -> CUDA out; the reference's errors."""

import numpy as np
import pytest

from oracle import tsg_oracle as O

pytestmark = pytest.mark.gpu

T = pytest.importorskip("paper_1908_06094_b200")
R = T.reference


def _relabel(table, fwd_rows, fwd_ids):
    """A table under new numberings: row r' = fwd_rows[r], entries mapped by fwd_ids."""
    out = np.empty_like(table)
    out[fwd_rows] = fwd_ids[table]
    return out


def _perm(n, seed):
    return np.random.default_rng(seed).permutation(n)


@pytest.mark.parametrize("shape", [(13, 21, 20), (7, 9, 7), (5, 6, 2)])
@pytest.mark.parametrize("relabel", [False, True])
def test_flat_stages_match_oracle(cuda_ok, shape, relabel):
    r, c, k = shape
    inp = O.transport_inputs(r, c, k, 2, "random", "random", "random")
    e2v = O.neighbor_table(r, c, "edges", "vertices")
    v2e = O.neighbor_table(r, c, "vertices", "edges")
    pd, vn, wn, rho = inp["pd"], inp["vn"], inp["wn"], inp["rho"]
    signs, dual = inp["signs"], inp["dual"].reshape(-1)
    if relabel:  # any numbering: permute vertices and edges consistently
        pv, pe = _perm(len(pd), 1), _perm(len(vn), 2)
        e2v, v2e = _relabel(e2v, pe, pv), _relabel(v2e, pv, pe)
        pd2, vn2, wn2, rho2 = (np.empty_like(x) for x in (pd, vn, wn, rho))
        pd2[pv], vn2[pe], wn2[pv], rho2[pv] = pd, vn, wn, rho
        sg2, du2 = np.empty_like(signs), np.empty_like(dual)
        sg2[pv], du2[pv] = signs, dual
        pd, vn, wn, rho, signs, dual = pd2, vn2, wn2, rho2, sg2, du2
    flux = R.upwind_flux(e2v, vn, pd)
    assert isinstance(flux, np.ndarray)
    assert np.array_equal(flux, O.upwind_flux(e2v, vn, pd))
    assert np.array_equal(R.centred_flux(e2v, vn, pd), O.centred_flux(e2v, vn, pd))
    fluz = R.upwind_fluz(wn, pd, 0.75)
    assert np.array_equal(fluz, O.upwind_fluz(wn, pd, 0.75))
    div = R.flux_divergence(v2e, signs, dual, flux, fluz)
    assert np.array_equal(div, O.flux_divergence(v2e, signs, dual, flux, fluz))
    out = R.advance_density(pd, div, rho, 0.1)
    assert np.array_equal(out, O.advance_density(pd, div, rho, 0.1))
    step = R.transport_step(e2v, v2e, signs, dual, pd, vn, wn, rho, 0.1, 0.75)
    assert np.array_equal(step["pd_out"], out)
    c2e = O.neighbor_table(r, c, "cells", "edges")
    length = 0.5 + np.random.default_rng(3).random(len(vn))
    area = 0.2 + np.random.default_rng(4).random(len(c2e))
    assert np.array_equal(R.cell_divergence(c2e, vn, length, area), O.cell_divergence(c2e, vn, length, area))
    c2c = O.neighbor_table(r, c, "cells", "cells")
    a = np.random.default_rng(5).random((len(c2c), k))
    fac = 0.5 + np.random.default_rng(6).random((len(c2c), 1))
    assert np.array_equal(R.neighbor_sum(c2c, a), O.neighbor_sum(c2c, a))
    assert np.array_equal(R.neighbor_sum_scaled(c2c, a, fac), O.neighbor_sum_scaled(c2c, a, fac))


@pytest.mark.parametrize("k", [40, 41])
def test_flat_stages_long_sweeps(cuda_ok, k):
    """A patch whose item sweeps are long enough for one-pass grids (tsg_common.cuh
    item_grid): the level-pair forms and pipelined gathers (even level count) and the point
    forms (odd: rows not 16-byte aligned), each stage and the whole step, bitwise."""
    import torch

    r, c = 1024, 1024
    inp = O.transport_inputs(r, c, k, 2, "random", "random", "random")
    e2v = O.neighbor_table(r, c, "edges", "vertices")
    v2e = O.neighbor_table(r, c, "vertices", "edges")
    c2e = O.neighbor_table(r, c, "cells", "edges")
    dev = {n: torch.from_numpy(np.ascontiguousarray(x)).cuda()
           for n, x in (("e2v", e2v), ("v2e", v2e), ("c2e", c2e), ("pd", inp["pd"]), ("vn", inp["vn"]),
                        ("wn", inp["wn"]), ("rho", inp["rho"]), ("signs", inp["signs"]),
                        ("dual", inp["dual"].reshape(-1)))}
    flux = O.upwind_flux(e2v, inp["vn"], inp["pd"])
    fluz = O.upwind_fluz(inp["wn"], inp["pd"], 0.5)
    got = R.upwind_fluz(dev["wn"], dev["pd"], 0.5)
    assert np.array_equal(got.cpu().numpy(), fluz)
    div = O.flux_divergence(v2e, inp["signs"], inp["dual"].reshape(-1), flux, fluz)
    got = R.flux_divergence(dev["v2e"], dev["signs"], dev["dual"], torch.from_numpy(flux).cuda(),
                            torch.from_numpy(fluz).cuda())
    assert np.array_equal(got.cpu().numpy(), div)
    out = R.advance_density(dev["pd"], torch.from_numpy(div).cuda(), dev["rho"], 0.1)
    assert np.array_equal(out.cpu().numpy(), O.advance_density(inp["pd"], div, inp["rho"], 0.1))
    length = 0.5 + np.random.default_rng(3).random(len(e2v))
    area = 0.2 + np.random.default_rng(4).random(len(c2e))
    got = R.cell_divergence(dev["c2e"], dev["vn"], torch.from_numpy(length).cuda(), torch.from_numpy(area).cuda())
    assert np.array_equal(got.cpu().numpy(), O.cell_divergence(c2e, inp["vn"], length, area))
    got = R.upwind_flux(dev["e2v"], dev["vn"], dev["pd"])
    assert np.array_equal(got.cpu().numpy(), flux)
    step = R.transport_step(dev["e2v"], dev["v2e"], dev["signs"], dev["dual"], dev["pd"], dev["vn"], dev["wn"],
                            dev["rho"], 0.1, 0.5)
    got = step["pd_out"]
    got = got.cpu().numpy() if hasattr(got, "cpu") else got
    assert np.array_equal(got, O.advance_density(inp["pd"], div, inp["rho"], 0.1))


def test_one_dimensional_arrays_and_device_tensors(cuda_ok):
    import torch

    r, c = 6, 8
    c2c = O.neighbor_table(r, c, "cells", "cells")
    a = np.random.default_rng(0).random(len(c2c))
    got = R.neighbor_sum(c2c, a)
    assert got.shape == a.shape and np.array_equal(got, O.neighbor_sum(c2c, a))
    e2v = O.neighbor_table(r, c, "edges", "vertices")
    vn = np.random.default_rng(1).random(len(e2v)) - 0.5
    pd = np.random.default_rng(2).random(r * c)
    assert np.array_equal(R.upwind_flux(e2v, vn, pd), O.upwind_flux(e2v, vn, pd))
    # CUDA tensors stay on the device
    a2 = torch.as_tensor(np.random.default_rng(3).random((len(c2c), 6)), device="cuda")
    t = torch.as_tensor(c2c, device="cuda")
    got = R.neighbor_sum(t, a2)
    assert got.is_cuda and np.array_equal(got.cpu().numpy(), O.neighbor_sum(c2c, a2.cpu().numpy()))


def test_reference_errors(cuda_ok):
    n = 10
    with pytest.raises(ValueError, match="need at least 2 levels"):
        R.upwind_fluz(np.zeros((n, 2)), np.zeros((n, 1)), 1.0)
    with pytest.raises(ValueError, match="wn must be staggered"):
        R.upwind_fluz(np.zeros((n, 4)), np.zeros((n, 2)), 1.0)
    e2v = np.array([[0, 1], [1, n]])  # id n is out of range
    with pytest.raises(IndexError):
        R.upwind_flux(e2v, np.zeros((2, 3)), np.zeros((n, 3)))
    with pytest.raises(ValueError):
        R.advance_density(np.zeros((n, 3)), np.zeros((n, 2)), np.ones((n, 3)), 0.1)
    # an empty neighbourhood sums to 0.0
    got = R.neighbor_sum(np.zeros((4, 0), dtype=np.int64), np.ones((3, 2)))
    assert np.array_equal(got, np.zeros((4, 2)))
