"""The C ABI from a plain C program (no Python in the call path): compile
tests/c/abi_solve.c against include/bhcp_b200.h and libbhcp_b200.so and run it
on the GPU (a 2D solve checked against the closed form, status read-back and
the invalid-argument contract)."""

import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
PKG = ROOT / "paper_2107_06381_b200"
CUDA = Path("/usr/local/cuda")


def build(tmp_path):
    cc = shutil.which("gcc")
    if cc is None:
        pytest.skip("gcc not available")
    exe = tmp_path / "abi_solve"
    cmd = [cc, "-O2", "-std=gnu11", str(ROOT / "tests/c/abi_solve.c"), "-I", str(ROOT / "include"),
           "-I", str(CUDA / "include"), "-L", str(PKG), "-lbhcp_b200", "-L", str(CUDA / "lib64"), "-lcudart",
           "-lm", f"-Wl,-rpath,{PKG}", f"-Wl,-rpath,{CUDA / 'lib64'}", "-o", str(exe)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_program_compiles(tmp_path):
    if not (PKG / "libbhcp_b200.so").exists():
        pytest.skip("library not built")
    build(tmp_path)


@pytest.mark.gpu
def test_c_program_solves_on_gpu(tmp_path):
    exe = build(tmp_path)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "C_ABI_OK" in r.stdout
