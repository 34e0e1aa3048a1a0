"""CPU-side checks of the drop-in boundary: the C-ABI library builds/loads and
exports every symbol include/kronglm_b200.h declares; host-only entry points
(input builders, index map) agree with the oracle.  No device compute."""
import ctypes
import os
import re

import numpy as np
import pytest

from oracle import oracle as O
from paper_1510_03298_b200 import _lib, build as B
from paper_1510_03298_b200 import kronglm as K

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "kronglm_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(kg_[a-z0-9_]+)\s*\(", src)))


def test_library_builds_and_exports_every_declared_symbol():
    B.build()
    lib = ctypes.CDLL(B.LIB)
    syms = declared_symbols()
    assert len(syms) >= 40
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # the ctypes binding covers the whole header
    assert sorted(_lib.EXPORTED) == syms


def test_product_does_not_reference_the_oracle():
    pkg = os.path.join(ROOT, "paper_1510_03298_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in txt.replace("oracles", ""), f


def test_host_builders_match_oracle():
    for n, p in ((40, 10), (100, 30), (365, 60), (4096, 256), (23, 7)):
        pts = np.linspace(0, 1, n)
        assert np.array_equal(K.bspline_design(pts, 4, p), O.bspline_design(pts, 4, p))
    pts = np.linspace(0.0, 7.0, 23)
    for order in (1, 2, 3, 4):
        assert np.array_equal(K.bspline_design(pts, order, 7), O.bspline_design(pts, order, 7))
    for a in ((25, 5), (977, 5), (33, 4), (81, 4), (168, 4)):
        assert K.default_basis_count(*a) == O.default_basis_count(*a)
    assert K.linear_index([2, 1, 2], [2, 3, 2]) == 8
    with pytest.raises(ValueError):
        K.linear_index([0, 1], [2, 3])
    with pytest.raises(ValueError):
        K.bspline_design([0.0, 0.0, 1.0], 4, 5)


def test_import_kronglm_exposes_the_reference_module_surface():
    """`import kronglm` works like the pybind11 module (kronglm_py.cpp:115-249):
    every in-scope function of the reference module is there (dense_materialize
    and simulate are the test oracle and the data generator, out of scope)."""
    import kronglm
    for name in ("linear_index", "rho", "h_map", "g_map", "lambda_max", "fit_path", "predict", "bspline_design",
                 "default_basis_count", "outer_solve", "mse_heldout"):
        assert callable(getattr(kronglm, name)), name
    assert kronglm.fit_path is K.fit_path
    assert issubclass(kronglm.EvalError, RuntimeError)


def test_result_accessors_reject_out_of_range_models():
    """kg_result_* accessors on a NULL result / bad index return NaN or -1
    instead of indexing past the vectors (no device work)."""
    L = _lib.load()
    assert np.isnan(L.kg_result_lambda(None, 0))
    assert np.isnan(L.kg_result_objective(None, 3))
    assert L.kg_result_inner_iters(None, 0) == -1
    assert L.kg_result_outer_iters(None, -1) == -1
    assert L.kg_result_status(None, 0) == -1
    assert L.kg_result_nonzero(None, 0) == -1
    assert L.kg_result_n_outer(None, 0) == -1
    assert L.kg_result_trace(None, 0, None) == _lib.KG_EINVAL


def test_bench_refuses_missing_gpus_with_one_json_line():
    """bench.py prints exactly one JSON line on stdout, whatever native libraries
    write there (file descriptor 1 is pointed at stderr for the run), and a
    --gpus N request on a box with fewer GPUs is refused, not run at N = 1."""
    import json
    import subprocess
    import sys
    import torch
    if torch.cuda.device_count() >= 2:
        pytest.skip("needs a box with fewer than 2 GPUs")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--steps", "1", "--warmup", "1"],
                       capture_output=True, text=True, timeout=300)
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    assert "refusing" in json.loads(lines[0])["error"]
    assert r.returncode != 0
