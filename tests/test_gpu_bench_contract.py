"""bench.py's own arm on the GPU prints the contract line (a short run): every required key,
the roofline and cpu_baseline objects, e2e with its copy bytes, a positive launch count,
clocks, identical config dicts in both arms, and the in-run parity check of the
benchmarked kernel against the CPU sample."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _line(*args):
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True, text=True,
                         timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


def test_bench_line_contract(cuda_ok):
    line = _line("--steps", "8", "--warmup", "3", "--no-o1280", "--cpu-seconds", "2", "--flushed-steps", "4",
                 "--sustained-seconds", "0.2")
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e",
                "gpu_launches", "clocks"):
        assert key in line, key
    assert line["value"] > 0 and line["n_gpus"] == 1 and line["steps"] == 8 and line["dtype"] == "f64"
    r = line["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1.2
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9 and r["traffic"] > 0
    cb = line["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] > 0 and cb["gpu_parity"]["bitwise"]
    e = line["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert line["gpu_launches"] >= 1 and "sm_mhz" in line["clocks"]
    assert "l2" in line["config"]
    ref = _line("--impl", "reference", "--steps", "3", "--warmup", "3", "--no-python-ref")
    assert ref["config"] == line["config"] and ref["metric"] == line["metric"] and ref["unit"] == line["unit"]
