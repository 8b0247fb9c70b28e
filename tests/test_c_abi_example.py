"""examples/c_abi_transport.c: a caller of the C ABI with no Python in the process.

The CPU test compiles and links it against include/tsg.h and the in-tree libtsg.so (the
header and the library stay in step with a plain-C caller); the GPU test runs it: flat
table-driven step == structured fused step, and a 5-step persistent loop == five chained
flat steps, bitwise, on two shapes."""

import shutil
import subprocess
from pathlib import Path

import pytest

from paper_1908_06094_b200 import _lib

ROOT = Path(__file__).resolve().parents[1]
SRC = ROOT / "examples" / "c_abi_transport.c"
CUDA = Path("/usr/local/cuda")


def _build(tmp_path):
    if shutil.which("gcc") is None or not (CUDA / "include" / "cuda_runtime.h").exists():
        pytest.skip("gcc or the CUDA headers are not available")
    if not _lib.LIB_PATH.exists():
        pytest.skip("libtsg.so is not built")
    exe = tmp_path / "c_abi_transport"
    libdir = _lib.LIB_PATH.parent
    cmd = ["gcc", "-O2", "-std=c99", "-Wall", "-Wextra", "-Werror", f"-I{ROOT / 'include'}",
           f"-I{CUDA / 'include'}", str(SRC), f"-L{libdir}", f"-l:{_lib.LIB_PATH.name}",
           f"-L{CUDA / 'lib64'}", "-lcudart", f"-Wl,-rpath,{libdir}", "-o", str(exe)]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_c_example_compiles_and_links(tmp_path):
    assert _build(tmp_path).exists()


@pytest.mark.gpu
@pytest.mark.parametrize("shape", [(37, 45, 24), (64, 96, 80)])
def test_c_example_runs_bitwise(tmp_path, cuda_ok, shape):
    exe = _build(tmp_path)
    out = subprocess.run([str(exe), *map(str, shape)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.startswith("OK"), out.stdout
