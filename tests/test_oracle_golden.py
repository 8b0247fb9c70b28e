"""Pin the CPU oracle against golden vectors produced by the real reference.

The golden fixtures come from tests/golden/make_golden.py, which runs
``tristencil`` unmodified.  Everything here is bitwise (np.array_equal) --
stricter than the north-star tolerance of 1e-12 relative.
"""

import numpy as np
import pytest

from oracle import tsg_oracle as O
from tests.hashing import sha

RELS = list(O.OFFSETS)


@pytest.mark.parametrize("shape", [(2, 2), (3, 3), (2, 5), (4, 3), (5, 6), (7, 4), (8, 8)])
def test_tables_and_signs(golden, shape):
    r, c = shape
    for (f, t) in RELS:
        assert np.array_equal(O.neighbor_table(r, c, f, t), golden[f"tbl_{r}x{c}_{f}_{t}"]), (f, t)
    assert np.array_equal(O.edge_signs(r, c), golden[f"signs_{r}x{c}"])


@pytest.mark.parametrize("shape", [(5, 7), (16, 8), (3, 9), (4, 4), (4, 2), (6, 5)])
def test_numberings(golden, shape):
    r, c = shape
    for loc in ("vertices", "cells", "edges"):
        assert np.array_equal(O.un_forward(r, c, loc), golden[f"perm_un_{r}x{c}_{loc}"])
    for loc in ("vertices", "cells"):
        assert np.array_equal(O.hn_forward(r, c, loc), golden[f"perm_hn_{r}x{c}_{loc}"])


def test_permuted_tables(golden):
    for r, c in ((16, 8), (5, 7)):
        for num, fn in (("un", O.un_forward), ("hn", O.hn_forward)):
            p = fn(r, c, "cells")
            got = O.neighbor_table(r, c, "cells", "cells", p, p)
            assert np.array_equal(got, golden[f"tblp_{num}_{r}x{c}_cells_cells"])
    pv, pe = O.hn_forward(4, 4, "vertices"), O.un_forward(4, 4, "edges")
    assert np.array_equal(O.neighbor_table(4, 4, "edges", "vertices", pe, pv),
                          golden["tblp_relabel_4x4_edges_vertices"])
    assert np.array_equal(O.neighbor_table(4, 4, "vertices", "edges", pv, pe),
                          golden["tblp_relabel_4x4_vertices_edges"])


def test_hilbert(golden):
    for n in (2, 4):
        rows = golden[f"hilbert_file_n{n}"]
        x, y = O.hilbert_xy(n, rows[:, 0])
        assert np.array_equal(np.stack([x, y], 1), rows[:, 1:])
        for d, xx, yy in rows:
            assert O.hilbert_rank(n, int(xx), int(yy)) == d
    for n in (8, 32):
        x, y = O.hilbert_xy(n, np.arange(n * n))
        assert np.array_equal(np.stack([x, y], 1), golden[f"hilbert_xy_n{n}"])


def _small_cases(golden_hashes):
    return golden_hashes["small_transport"]


def test_transport_small_cases_bitwise(golden, golden_hashes):
    for meta in _small_cases(golden_hashes):
        k = meta["key"]
        r, c, _ = meta["shape"]
        out = O.transport_step(
            O.neighbor_table(r, c, "edges", "vertices"), O.neighbor_table(r, c, "vertices", "edges"),
            golden[f"{k}_signs"], golden[f"{k}_dual"], golden[f"{k}_pd"], golden[f"{k}_vn"],
            golden[f"{k}_wn"], golden[f"{k}_rho"], meta["dt"], meta["pivbz"], meta["flux_op"])
        for name in ("flux", "fluz", "div", "pd_out"):
            assert np.array_equal(out[name], golden[f"{k}_{name}"]), (k, name)


def test_input_generation_reproduces_reference(golden, golden_hashes):
    """transport_inputs == the reference's _transport_case / _transport_setup draws."""
    for meta in _small_cases(golden_hashes):
        k = meta["key"]
        r, c, lev = meta["shape"]
        inp = O.transport_inputs(r, c, lev, meta["seed"], meta["geometry"], "random", "random")
        for name in ("pd", "vn", "wn", "rho", "dual", "signs"):
            assert np.array_equal(inp[name], golden[f"{k}_{name}"]), (k, name)


@pytest.mark.parametrize("key", ["cfg1_s0", "cfg1_s1", "cfg1_default", "cfg2_rand"])
def test_transport_hashed_cases(golden_hashes, key):
    e = golden_hashes["transport"][key]
    cfg = e["config"]
    inp = O.transport_inputs(e["rows"], e["cols"], e["levels"], cfg.get("seed", 0),
                             cfg.get("geometry", "uniform"), cfg.get("preset", "gaussian-bump"), "one")
    ih = {n: sha(inp[n]) for n in e["inputs"]}
    if e["exp_dependent"] and ih["pd"] != e["inputs"]["pd"]:
        pytest.skip("np.exp differs from the golden host in the last ulp")
    assert ih == e["inputs"]
    out = O.step_inputs(e["rows"], e["cols"], inp, e["dt"], e["pivbz"])
    assert {n: sha(out[n]) for n in e["outputs"]} == e["outputs"]


def test_transport_multistep_hash(golden_hashes):
    e = golden_hashes["transport"]["cfg1_s2_10steps"]
    inp = O.transport_inputs(44, 72, 10, 2, "random", "random", "one")
    for _ in range(e["steps"]):
        inp["pd"] = O.step_inputs(44, 72, inp, e["dt"], e["pivbz"])["pd_out"]
    assert sha(inp["pd"]) == e["outputs"]["pd_out"]


def test_neighbor_sums(golden):
    for r, c, lev in ((16, 8, 2), (5, 7, 3)):
        key = f"k_{r}x{c}x{lev}"
        a, fac = golden[f"{key}_a"], golden[f"{key}_fac"]
        for num in ("sn", "un", "hn"):
            p = {"sn": np.arange(2 * r * c), "un": O.un_forward(r, c, "cells"),
                 "hn": O.hn_forward(r, c, "cells")}[num]
            inv = np.empty_like(p)
            inv[p] = np.arange(p.size)
            t = O.neighbor_table(r, c, "cells", "cells", p, p)
            k1 = O.neighbor_sum(t, a[inv])[p]
            k2 = O.neighbor_sum_scaled(t, a[inv], fac[inv])[p]
            assert np.array_equal(k1, golden[f"{key}_k1"]), num
            assert np.array_equal(k2, golden[f"{key}_k2"]), num


def test_nine_relation_reduce(golden):
    for (f, t) in RELS:
        got = O.neighbor_sum(O.neighbor_table(6, 5, f, t), golden[f"red_{f}_{t}_a"])
        assert np.array_equal(got, golden[f"red_{f}_{t}_b"]), (f, t)


def test_cell_divergence(golden):
    c2e = O.neighbor_table(5, 5, "cells", "edges")
    got = O.cell_divergence(c2e, golden["cdiv_vn"], golden["cdiv_length"], golden["cdiv_area"])
    assert np.array_equal(got, golden["cdiv_0"])
    geo = O.geometry(5, 5, "random", 7)
    assert np.array_equal(geo["weights"], golden["cdiv_weights"])
    w = O.weighted_divergence(c2e, golden["cdiv_vn"], golden["cdiv_weights"])
    assert np.array_equal(w, golden["cdiv_1"])


def test_c_oracle_matches_golden(golden, golden_hashes):
    """The C restatement (CPU baseline) is bitwise equal to the reference."""
    from oracle import c_oracle

    for meta in _small_cases(golden_hashes):
        k = meta["key"]
        r, c, _ = meta["shape"]
        out = c_oracle.transport_step(
            O.neighbor_table(r, c, "edges", "vertices"), O.neighbor_table(r, c, "vertices", "edges"),
            golden[f"{k}_signs"], golden[f"{k}_dual"], golden[f"{k}_pd"], golden[f"{k}_vn"],
            golden[f"{k}_wn"], golden[f"{k}_rho"], meta["dt"], meta["pivbz"], meta["flux_op"])
        for name in ("flux", "fluz", "div", "pd_out"):
            assert np.array_equal(out[name], golden[f"{k}_{name}"]), (k, name)
    e = golden_hashes["transport"]["cfg2_rand"]
    inp = O.transport_inputs(128, 128, 80, 0, "random", "random", "one")
    out = c_oracle.transport_step(
        O.neighbor_table(128, 128, "edges", "vertices"), O.neighbor_table(128, 128, "vertices", "edges"),
        inp["signs"], inp["dual"], inp["pd"], inp["vn"], inp["wn"], inp["rho"], e["dt"], e["pivbz"])
    assert {n: sha(out[n]) for n in e["outputs"]} == e["outputs"]
    for r, c, lev in ((16, 8, 2), (5, 7, 3)):
        key = f"k_{r}x{c}x{lev}"
        t = O.neighbor_table(r, c, "cells", "cells")
        assert np.array_equal(c_oracle.neighbor_sum(t, golden[f"{key}_a"]), golden[f"{key}_k1"])
        assert np.array_equal(c_oracle.neighbor_sum(t, golden[f"{key}_a"], golden[f"{key}_fac"]),
                              golden[f"{key}_k2"])
