"""Armijo backtracking (outer.cpp:106-144) beyond the full step.

Port of the reference case "a poisson step on stale unit weights backtracks
and still descends" (proj/tests/test_outer.cpp:140-177): Poisson counts in
[300, 500] on a small random design, lambda = 1e-4, unit weights -- the
subproblem solution overshoots and the search must reject t = 1.  A second
case with counts near 1e4 needs j > 8, which on the device runs past the
first batch of kMaxTrials = 8 trial log-likelihoods (kg_solver.cu's batched
trial passes).  The oracle cases run on CPU; the GPU cases compare the
CUDA outer_solve record by record with the oracle's (OuterTrace)."""
import numpy as np
import pytest

from oracle import oracle as O
from tests import helpers as H

MAXIT = 12  # outer iterations per comparison (unit weights converge slowly; status max_iterations is fine)


def case(seed, lo, hi):
    rng = np.random.default_rng(seed)
    design = H.make_design(rng, (4, 3), [(2, 2)])
    y = np.asfortranarray(np.floor(rng.uniform(lo, hi, (4, 3))))
    return design, y


def check_descent(res):
    prev = res["initial_objective"]
    for rec in res["iterations"]:
        if rec["armijo_j"] >= 0:
            assert rec["objective"] <= prev + 1e-12 * max(1.0, abs(prev))
            prev = rec["objective"]


def test_oracle_stale_unit_weights_backtrack_and_descend():  # test_outer.cpp:140-177
    design, y = case(64, 300.0, 500.0)
    r = O.outer_solve(design, "poisson", y, 1e-4, iwls="unit", maxit=MAXIT)
    js = [int(rec["armijo_j"]) for rec in r["iterations"]]
    assert js[0] >= 1, js
    assert r["iterations"][0]["objective"] < r["initial_objective"]
    check_descent(r)


def test_oracle_large_counts_need_more_than_eight_backtracks():
    design, y = case(65, 8000.0, 12000.0)
    r = O.outer_solve(design, "poisson", y, 1e-4, iwls="unit", maxit=MAXIT)
    js = [int(rec["armijo_j"]) for rec in r["iterations"]]
    assert max(js) > 8, js
    check_descent(r)


@pytest.mark.gpu
@pytest.mark.parametrize("seed,lo,hi", [(64, 300.0, 500.0), (65, 8000.0, 12000.0), (66, 300.0, 500.0)])
@pytest.mark.parametrize("iwls", ["unit", "exact"])
def test_device_armijo_trace_matches_oracle(seed, lo, hi, iwls):
    from paper_1510_03298_b200 import kronglm as K
    design, y = case(seed, lo, hi)
    want = O.outer_solve(design, "poisson", y, 1e-4, iwls=iwls, maxit=MAXIT)
    got = K.outer_solve(design, "poisson", y, 1e-4, iwls=iwls, maxit=MAXIT)
    assert got["status"] == want["status"]
    assert abs(got["initial_objective"] - want["initial_objective"]) <= 1e-12 * abs(want["initial_objective"])
    assert len(got["iterations"]) == len(want["iterations"])
    for g, w in zip(got["iterations"], want["iterations"]):
        assert g["armijo_j"] == int(w["armijo_j"])
        assert g["alpha"] == w["alpha"]
        assert g["inner_iterations"] == int(w["inner_iterations"])
        assert abs(g["objective"] - w["objective"]) <= 1e-8 * max(1.0, abs(w["objective"]))
        assert abs(g["delta_k"] - w["delta_k"]) <= 1e-8 * max(1.0, abs(w["objective"]))
    scale = max(np.max(np.abs(want["coef_flat"])), 1e-300)
    assert np.max(np.abs(got["coef_flat"] - want["coef_flat"])) / scale <= 1e-8
    if iwls == "unit":
        js = [r["armijo_j"] for r in got["iterations"]]
        assert max(js) >= 1
        if lo > 1000:
            assert max(js) > 8  # exercised the second trial batch on the device
