"""CPU-side tests: the C ABI library's exports and argument checks, and the host logic
(patch/layout/numbering/storage bookkeeping) pinned to the reference's golden answers.
No compute call here needs a GPU."""

import ctypes
import json
import re
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from oracle import tsg_oracle as O
from paper_1908_06094_b200 import _lib
from paper_1908_06094_b200.topology import LocationType as L

ROOT = Path(__file__).resolve().parents[1]


# -- the C ABI -------------------------------------------------------------------------


def header_functions():
    text = (ROOT / "include" / "tsg.h").read_text()
    return sorted(set(re.findall(r"\b(tsg_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _lib.lib()
    names = header_functions()
    assert len(names) >= 25
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # and the Python binding declares exactly the header's entry points
    assert sorted(_lib.SIGNATURES) == names


def test_nm_lists_the_symbols():
    out = subprocess.run(["nm", "-D", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (tsg_[a-z0-9_]+)", out))
    assert set(header_functions()) <= exported


def test_abi_version_and_pitch():
    lib = _lib.lib()
    assert lib.tsg_abi_version() == 1
    assert [lib.tsg_inner_pitch(n) for n in (1, 2, 3, 6, 63, 64, 80, 81, 137, 138)] == [1, 2, 4, 6, 64, 64, 80, 96, 144, 144]
    from paper_1908_06094_b200.device import inner_pitch

    assert [inner_pitch(n) for n in (1, 2, 3, 6, 63, 64, 80, 81, 137, 138)] == [1, 2, 4, 6, 64, 64, 80, 96, 144, 144]


def test_argument_errors_map_to_reference_exceptions():
    lib = _lib.lib()
    with pytest.raises(ValueError, match=">= 2"):
        _lib.check(lib.tsg_build_neighbor_table(1, 4, 0, 2, None, None, None, None))
    with pytest.raises(ValueError, match="relation"):
        _lib.check(lib.tsg_build_neighbor_table(4, 4, 7, 2, None, None, ctypes.c_void_p(8), None))
    with pytest.raises(ValueError, match="grid is NULL"):
        _lib.check(lib.tsg_mpdata_step(None, *([None] * 7), 0.1, 1.0, 0, None))
    p = ctypes.c_void_p(16)
    with pytest.raises(ValueError, match="at least 2 levels"):
        _lib.check(lib.tsg_transport_indirect(*([p] * 8), 4, 12, 1, 0.1, 1.0, 0, *([p] * 4), None))
    with pytest.raises(ValueError, match="operator"):
        _lib.check(lib.tsg_transport_indirect(*([p] * 8), 4, 12, 3, 0.1, 1.0, 7, *([p] * 4), None))
    with pytest.raises(ValueError, match="hn numbering is not defined for edges"):
        _lib.check(lib.tsg_make_permutation(4, 4, 2, 2, p, p, None))
    with pytest.raises(ValueError, match="variant"):
        _lib.check(lib.tsg_set_fused_variant(99))
    assert "variant" in lib.tsg_last_error().decode()
    # round-2 entry points validate before any device work
    with pytest.raises(ValueError, match="reduce variant"):
        _lib.check(lib.tsg_set_reduce_variant(20))
    with pytest.raises(ValueError, match="point limit"):
        _lib.check(lib.tsg_set_point_limit(-1))
    _lib.check(lib.tsg_set_point_limit(0))
    with pytest.raises(ValueError, match="NULL"):
        _lib.check(lib.tsg_flat_flux(None, p, p, 4, 2, 0, p, None))
    with pytest.raises(ValueError, match="operator"):
        _lib.check(lib.tsg_flat_flux(p, p, p, 4, 2, 5, p, None))
    with pytest.raises(ValueError, match="at least 2 levels"):
        _lib.check(lib.tsg_flat_fluz(p, p, 4, 1, 1.0, p, None))
    with pytest.raises(ValueError, match="bad shape"):
        _lib.check(lib.tsg_flat_divergence(p, -1, p, p, p, p, 4, 2, p, None))
    with pytest.raises(ValueError, match="NULL"):
        _lib.check(lib.tsg_flat_advance(p, None, p, 4, 0.1, p, None))
    with pytest.raises(ValueError, match="bad shape"):
        _lib.check(lib.tsg_flat_cell_divergence(p, 3, p, p, p, 4, 0, p, None))
    with pytest.raises(ValueError, match="kind"):
        _lib.check(lib.tsg_memcpy2d(p, 64, p, 64, 64, 2, 3, None))
    with pytest.raises(ValueError, match="extents"):
        _lib.check(lib.tsg_memcpy2d(p, 32, p, 64, 64, 2, 1, None))
    with pytest.raises(ValueError, match="grid is NULL"):
        _lib.check(lib.tsg_pack_strided_rows(None, 0, 4, p, None, 1, 0, 1, p, None))


def test_grid_create_validates_before_touching_the_device():
    lib = _lib.lib()
    h = ctypes.c_void_p()
    with pytest.raises(ValueError, match="rows and cols"):
        _lib.check(lib.tsg_grid_create(1, 5, 3, 3, ctypes.byref(h)))
    with pytest.raises(ValueError, match="levels"):
        _lib.check(lib.tsg_grid_create(4, 5, 0, 3, ctypes.byref(h)))


def test_fused_variant_smem_fits_an_sm():
    lib = _lib.lib()
    v = 1
    while lib.tsg_fused_variant_info(v, *[None] * 6) == 0:
        vals = [ctypes.c_int() for _ in range(6)]
        _lib.check(lib.tsg_fused_variant_info(v, *[ctypes.byref(x) for x in vals]))
        ti, tj, kc, stages, threads, smem = (x.value for x in vals)
        # LV lanes per vertex: 16 / 32 (a thread per level) or kc / 2 (a thread per level pair),
        # plus one producer warp in the warp-specialised variants
        assert threads in (ti * tj * 16, ti * tj * 32, ti * tj * kc // 2, ti * tj * kc // 2 + 32)
        assert threads <= 1024 and kc % 16 == 0
        stage = sum(-(-b // 128) * 128 for b in ((ti + 2) * (tj + 2) * (kc + 4) * 8,
                                                 (ti + 1) * 3 * (tj + 1) * kc * 8,
                                                 ti * tj * (kc + 2) * 8, ti * tj * kc * 8))
        assert smem == stages * stage + 128 <= 232448
        v += 1
    assert v > 8


def test_device_offset_constant_matches_canonical_tables():
    """csrc/tsg_offsets.cuh must encode connectivity.OFFSET_TABLES (= the reference's)."""
    from paper_1908_06094_b200.connectivity import OFFSET_TABLES, offset_array

    src = (ROOT / "paper_1908_06094_b200" / "csrc" / "tsg_offsets.cuh").read_text()
    body = src[src.index("c_offsets[9][3][6][3] = {"):]
    body = body[:body.index("};")]
    groups = [g for g in body.split("// ")[1:]]
    arr = offset_array()
    names = {"V": L.VERTICES, "C": L.CELLS, "E": L.EDGES}
    for g in groups:
        head, rest = g.split("\n", 1)
        f, t = (names[x.strip()] for x in head.split("->"))
        triples = [tuple(map(int, m)) for m in re.findall(r"\{(-?\d+), (-?\d+), (-?\d+)\}", rest)]
        want = [e for per in OFFSET_TABLES[(f, t)] for e in per]
        assert triples == want, (f, t)
        rel = f.code * 3 + t.code
        flat = [tuple(arr[rel, c, s]) for c in range(f.colors) for s in range(len(OFFSET_TABLES[(f, t)][0]))]
        assert flat == want
    # ... and the canonical tables are the oracle's (pinned to the reference's golden tables)
    for (f, t), per in OFFSET_TABLES.items():
        assert per == O.OFFSETS[(f.value, t.value)]


# -- host logic ---------------------------------------------------------------------------


def test_patch_spec_validation():
    from paper_1908_06094_b200 import PatchSpec

    PatchSpec(2, 2, 1)
    for args, msg in (((1, 4, 2), "rows and cols"), ((4, 4, 0), "levels"), ((4, 4, 2, 0), "halo"),
                      ((3, 4, 2, 4), "alias"), ((4.0, 4, 2), "integer")):
        with pytest.raises(ValueError, match=msg):
            PatchSpec(*args)


def test_element_ids_roundtrip():
    from paper_1908_06094_b200 import PatchSpec, element_coord, element_count, element_id

    spec = PatchSpec(5, 7, 1)
    for loc in L:
        assert element_count(spec, loc) == 35 * loc.colors
        for eid in range(element_count(spec, loc)):
            i, c, j = element_coord(spec, loc, eid)
            assert element_id(spec, loc, i, c, j) == eid == (i * loc.colors + c) * 7 + j
        assert element_id(spec, loc, -1, 0, 7) == element_id(spec, loc, 4, 0, 0)


def test_layouts_known_answers(golden_hashes):
    from paper_1908_06094_b200 import LayoutSpec, LinearLayout, PatchSpec, sn_offset

    orders = {"default": ("extra", "level", "row", "color", "column"),
              "level-inner": ("extra", "row", "color", "column", "level")}
    for e in golden_hashes["layouts"]:
        lin = LinearLayout(LayoutSpec(orders[e["order"]], e["alignment"]), e["sizes"], e["halo"])
        assert lin.padded == e["padded"] and lin.strides == e["strides"]
        assert lin.front_pad == e["front_pad"] and lin.total == e["total"]
    spec = PatchSpec(5, 4, 3)
    for loc, i, c, j, k, want in golden_hashes["sn_offset_5x4x3"]:
        assert sn_offset(LayoutSpec(), spec, L(loc), i, c, j, k) == want
    with pytest.raises(IndexError, match="row"):
        LinearLayout(LayoutSpec(), {"row": 3, "color": 1, "column": 3, "level": 1, "extra": 1}, 1).offset(5, 0, 0)
    with pytest.raises(ValueError):
        LayoutSpec(("row", "row", "color", "column", "level"))


def test_hilbert_scalar_functions(golden):
    from paper_1908_06094_b200 import hilbert_rank, hilbert_xy

    for n in (2, 4):
        for d, x, y in golden[f"hilbert_file_n{n}"]:
            assert hilbert_xy(n, int(d)) == (x, y) and hilbert_rank(n, int(x), int(y)) == d
    xy = golden["hilbert_xy_n32"]
    for d in range(0, 1024, 7):
        assert hilbert_xy(32, d) == tuple(xy[d]) and hilbert_rank(32, *map(int, xy[d])) == d
    with pytest.raises(ValueError):
        hilbert_xy(6, 0)


def test_permutation_contract():
    from paper_1908_06094_b200 import Permutation

    p = Permutation.from_forward([2, 0, 1])
    assert list(p.inverse) == [1, 2, 0]
    with pytest.raises(ValueError, match="bijection"):
        Permutation(forward=np.array([0, 0, 1]), inverse=np.array([0, 1, 2]))


def test_plane_access_model_exact():
    """Acceptance C1: the paper's Table 2 integers."""
    import paper_1908_06094_b200 as T

    counts = {"nodes": 71424, "edges": 213199}
    assert T.plane_access_total(counts, T.UNFUSED_PLANE_WEIGHTS) == 1140638
    assert T.plane_access_total(counts, T.FUSED_PLANE_WEIGHTS) == 357120
    with pytest.raises(ValueError):
        T.plane_access_total({"nodes": 1}, T.UNFUSED_PLANE_WEIGHTS)


def test_params_and_tiles_validation():
    from paper_1908_06094_b200 import MpdataParams, TileSpec
    from paper_1908_06094_b200.mpdata import flux_stage

    assert MpdataParams().dt == 0.1 and MpdataParams().pivbz == 1.0
    for kw, msg in ((dict(dt=-0.1), "dt"), (dict(dt=float("nan")), "dt"), (dict(pivbz=float("inf")), "pivbz")):
        with pytest.raises(ValueError, match=msg):
            MpdataParams(**kw)
    with pytest.raises(ValueError, match="operator"):
        flux_stage("sideways")
    with pytest.raises(ValueError):
        TileSpec(0, 4)


def test_storage_shapes_and_contracts():
    from paper_1908_06094_b200 import (DivergenceError, PatchSpec, Selector, StalenessError,
                                       make_storage, sync)

    spec = PatchSpec(4, 5, 3)
    f = make_storage(spec, L.EDGES, "f")
    assert f.shape == (6, 3, 7, 3, 1) and f.inner == 3
    w = make_storage(spec, L.VERTICES, "w", levels=4)
    assert w.shape[3] == 4
    s = make_storage(spec, L.VERTICES, "s", Selector(level=False, extra=True), extra_len=6)
    assert s.shape == (6, 1, 7, 1, 6) and s.inner == 6
    with pytest.raises(ValueError, match="color"):
        make_storage(spec, L.CELLS, "c", Selector(color=False))
    with pytest.raises(ValueError, match="extra"):
        make_storage(spec, L.CELLS, "c", Selector(extra=True))
    f.dirty["mirror"] = True
    with pytest.raises(StalenessError):
        f.array("primary")
    f.dirty["primary"] = True
    with pytest.raises(DivergenceError):
        sync(f, "primary")


def test_host_preset_and_halo_match_the_oracle():
    from paper_1908_06094_b200 import PatchSpec, init_preset, make_storage
    from paper_1908_06094_b200.kernels import field_to_flat

    spec = PatchSpec(6, 5, 3)
    f = make_storage(spec, L.VERTICES, "pd_in")
    for preset in ("uniform", "gaussian-bump", "random"):
        init_preset(f, preset, seed=3)
        assert np.array_equal(field_to_flat(f), O.preset(6, 5, 1, 3, "pd_in", preset, 3))
    arr = f.array()
    assert np.array_equal(arr[0], arr[6]) and np.array_equal(arr[7], arr[1])
    assert np.array_equal(arr[:, :, 0], arr[:, :, 5]) and np.array_equal(arr[:, :, 6], arr[:, :, 1])


def test_host_writes_do_not_drop_newer_device_data():
    """init_preset / flat_to_field on a field whose device copy is newer raise the
    reference's StalenessError (storage.py:130-145) instead of discarding that copy."""
    from paper_1908_06094_b200 import PatchSpec, StalenessError, flat_to_field, init_preset, make_storage

    spec = PatchSpec(4, 5, 3)
    f = make_storage(spec, L.VERTICES, "pd_in")
    f.dirty["mirror"] = True  # as after a kernel wrote the device copy
    with pytest.raises(StalenessError):
        init_preset(f, "uniform")
    with pytest.raises(StalenessError):
        flat_to_field(np.zeros((20, 3)), f)
    assert f.dirty["mirror"]


def test_workload_inputs_reproduce_reference_draws(golden, golden_hashes):
    from paper_1908_06094_b200.workloads import mpdata_algorithmic_bytes, transport_inputs

    for meta in golden_hashes["small_transport"][:8]:
        k = meta["key"]
        r, c, lev = meta["shape"]
        inp = transport_inputs(r, c, lev, meta["seed"], meta["geometry"], "random", "random", signs=False)
        for name in ("pd", "vn", "wn", "rho", "dual"):
            assert np.array_equal(inp[name], golden[f"{k}_{name}"]), (k, name)
    assert mpdata_algorithmic_bytes(279, 256, 80) == 319408128


def test_bench_reference_arm_contract():
    """--impl reference runs the C restatement on the host and prints the contract line."""
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "2",
                          "--warmup", "3"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "cpu_baseline", "e2e", "impl", "config"):
        assert key in line
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
