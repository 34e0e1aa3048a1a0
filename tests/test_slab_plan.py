"""Host logic of the slab pass's scatter/gather Y step (kg_slab_gather_plan,
include/kronglm_b200.h): the plan must reproduce X1^T w from the row quads'
window partials for every mode-1 factor the BASELINE configs use.  CPU only."""
import ctypes as C

import numpy as np
import pytest

from paper_1510_03298_b200 import _lib
from paper_1510_03298_b200 import kronglm as K


def plan(X):
    X = np.asfortranarray(X, dtype=np.float64)
    n, p = X.shape
    groups = (p + 7) // 8
    slots = np.zeros(groups * 64, dtype=np.int32)
    gmax, plane = C.c_int32(), C.c_int32()
    st = _lib.load().kg_slab_gather_plan(n, p, X.ctypes.data_as(C.POINTER(C.c_double)),
                                         slots.ctypes.data_as(C.POINTER(C.c_int32)), C.byref(gmax), C.byref(plane))
    return st, slots.reshape(groups * 8, 8), gmax.value, plane.value


@pytest.mark.parametrize("n,p", [(256, 64), (64, 20), (100, 30), (40, 10), (60, 14), (32, 10), (128, 32)])
def test_gather_plan_reproduces_the_transposed_product(n, p):
    X = K.bspline_design(np.linspace(0, 1, n), 4, p)
    st, slots, gmax, plane = plan(X)
    assert st == 0
    assert plane % 8 == 2 and plane >= 5 * (n // 4) + 1
    assert 1 <= gmax <= 8
    # the row quads' window partials of X^T w, as the row threads of k_slab4 form them
    rng = np.random.default_rng(n + p)
    w = rng.standard_normal(n)
    part = np.zeros(plane)
    first = [int(np.nonzero(X[r])[0][0]) for r in range(n)]
    for q in range(n // 4):
        wlo = min(first[4 * q], p - 5)
        for t in range(5):
            part[5 * q + t] = sum(X[r, wlo + t] * w[r] for r in range(4 * q, 4 * q + 4))
    want = X.T @ w
    for k in range(slots.shape[0]):
        used = slots[k][slots[k] != plane - 1]
        assert list(used) == sorted(used), "ascending quads: a fixed summation order"
        assert len(used) <= gmax
        got = part[used].sum()
        assert abs(got - (want[k] if k < p else 0.0)) <= 1e-13 * max(1.0, np.abs(want).max())
        assert np.all(slots[k][len(used):] == plane - 1), "padded with the zero slot"


def test_baseline_factors_need_five_slots():
    """Every mode-1 factor of the BASELINE configs (cubic B-splines on a ~4x finer
    grid) needs five gather slots per basis function: k_slab4<5>."""
    for n, p in ((256, 64), (64, 20), (100, 30)):
        st, _, gmax, _ = plan(K.bspline_design(np.linspace(0, 1, n), 4, p))
        assert st == 0 and gmax == 5


def test_gather_plan_rejects_what_the_pass_cannot_take():
    X = K.bspline_design(np.linspace(0, 1, 42), 4, 10)
    assert plan(X)[0] != 0                      # rows not a multiple of 4
    assert plan(np.ones((32, 10)))[0] != 0      # dense rows leave the 5-wide window
    Y = K.bspline_design(np.linspace(0, 1, 512), 4, 8)
    assert plan(Y)[0] != 0                      # 512 / 8: more than 8 quads per basis function
