"""The C++ drop-in header (include/kronglm_b200.hpp) compiles against the C
ABI (CPU) and runs a reference-style fit_path on the GPU."""
import os
import subprocess

import pytest

from paper_1510_03298_b200 import build as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "shim_path.cpp")


def _compile(out):
    B.build()
    cmd = ["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"), SRC, "-o", out,
           "-L", os.path.dirname(B.LIB), "-lkronglm_b200", "-Wl,-rpath," + os.path.dirname(B.LIB)]
    subprocess.run(cmd, check=True)


def test_shim_compiles_and_links(tmp_path):
    _compile(str(tmp_path / "shim_path"))


@pytest.mark.gpu
def test_shim_fit_path_runs(tmp_path):
    exe = str(tmp_path / "shim_path")
    _compile(exe)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
