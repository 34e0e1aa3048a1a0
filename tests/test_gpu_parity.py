"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle and the
dense Kronecker product, on the reference's own test designs and on B-spline
designs shaped like the BASELINE configs.

Tolerances: operator maps 1e-12 (test_array.cpp:142-193); path parity per
lambda: identical truncation/status, identical support, coefficients within
1e-8 relative to max|theta|, objectives within 1e-8 relative (north_star)."""
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_1510_03298_b200 import configs
from paper_1510_03298_b200 import kronglm as K
from tests import helpers as H

pytestmark = pytest.mark.gpu

COEF_RTOL = 1e-8
OBJ_RTOL = 1e-8


def bspline_design(n, p):
    return [[K.bspline_design(np.linspace(0, 1, nj), 4, pj) for nj, pj in zip(n, p)]]


# --------------------------------------------------------------- operators
def test_h_g_rho_match_dense_and_oracle_on_random_corpus():  # acceptance.cpp:53-80
    rng = np.random.default_rng(1001)
    for _ in range(60):
        design = H.random_design(rng)
        xd = H.dense(design)
        th = H.random_coef(rng, design)
        u = rng.uniform(-1, 1, H.row_dims(design))
        h = K.h_map(design, th)
        g = H.flat(K.g_map(design, u))
        assert np.max(np.abs(h.ravel(order="F") - xd @ H.flat(th))) <= 1e-12
        assert np.max(np.abs(g - xd.T @ u.ravel(order="F"))) <= 1e-12
        assert np.max(np.abs(h - O.h_map(design, th))) <= 1e-12
        lhs, rhs = float(np.vdot(h, u)), float(H.flat(th) @ g)
        assert abs(lhs - rhs) <= 1e-12 * max(1.0, abs(rhs))
        v = rng.uniform(0, 2, H.row_dims(design))
        want = xd.T @ (v.ravel(order="F") * (xd @ H.flat(th)))
        assert np.max(np.abs(H.flat(K.xtwx_apply(design, v, th)) - want)) <= 1e-12


def test_row_blocked_chain_contractions_match_oracle():
    """Shapes large enough for the row-blocked H/G chain kernels (k_contract_gb:
    mode-3 steps with alpha = p1 p2 = 2048 and 64 row groups): h_map, g_map
    and the adjoint identity against the oracle's banded maps."""
    rng = np.random.default_rng(77)
    design = bspline_design((40, 80, 1024), (32, 64, 256))
    th = [rng.uniform(-1, 1, (32, 64, 256))]
    u = rng.uniform(-1, 1, (40, 80, 1024))
    h = K.h_map(design, th)
    hw = O.h_map(design, th)
    assert np.max(np.abs(h - hw)) <= 1e-12 * max(1.0, np.max(np.abs(hw)))
    g = H.flat(K.g_map(design, u))
    gw = H.flat(O.g_map(design, u))
    assert np.max(np.abs(g - gw)) <= 1e-12 * max(1.0, np.max(np.abs(gw)))
    lhs, rhs = float(np.vdot(h, u)), float(H.flat(th) @ g)
    assert abs(lhs - rhs) <= 1e-12 * max(1.0, abs(rhs))


def test_rho_matches_oracle_and_rotates():
    rng = np.random.default_rng(13)
    a = rng.uniform(-1, 1, (3, 4, 2))
    r = K.rho(np.eye(3), a)
    assert r.shape == (4, 2, 3)
    for i in range(3):
        assert np.array_equal(r[:, :, i], a[i])
    for xs, ashape in (((2, 3), (3, 4)), ((4, 2), (2, 3, 5)), ((4, 3), (3,))):
        x = rng.standard_normal(xs)
        a = rng.uniform(-1, 1, ashape)
        assert np.max(np.abs(K.rho(x, a) - O.rho(x, a))) <= 1e-13
    with pytest.raises(ValueError):
        K.rho(rng.standard_normal((2, 4)), rng.uniform(-1, 1, (3, 4)))


@pytest.mark.parametrize("n,p", [((40, 40, 40), (10, 10, 10)), ((64, 64, 365), (20, 20, 60)),
                                 ((100, 100, 50), (30, 30, 12)), ((700, 300), (64, 40)), ((97,), (13,))])
def test_bspline_maps_match_oracle(n, p):
    rng = np.random.default_rng(7)
    design = bspline_design(n, p)
    th = [rng.standard_normal(p)]
    u = rng.standard_normal(n)
    h, ho = K.h_map(design, th), O.h_map(design, th)
    assert np.max(np.abs(h - ho)) <= 1e-12 * max(1.0, np.max(np.abs(ho)))
    g, go = H.flat(K.g_map(design, u)), H.flat(O.g_map(design, u))
    assert np.max(np.abs(g - go)) <= 1e-12 * max(1.0, np.max(np.abs(go)))


def test_spectral_radii_match_oracle():
    rng = np.random.default_rng(50)
    for n, p in ((40, 10), (64, 20), (365, 60), (256, 64)):
        x = K.bspline_design(np.linspace(0, 1, n), 4, p)
        D = K.Design([[x]])
        assert D.spectral(0, 0) == pytest.approx(O.spectral_radius(x.T @ x), rel=1e-12)
    x = rng.standard_normal((7, 5))
    assert K.Design([[x]]).spectral(0, 0) == pytest.approx(np.linalg.eigvalsh(x.T @ x).max(), rel=1e-10)


def test_lambda_max_matches_oracle_and_closed_form():  # test_penalty.cpp:107-137
    rng = np.random.default_rng(44)
    design = H.make_design(rng, (4, 3, 2), [(2, 2, 2)])
    y = rng.standard_normal((4, 3, 2))
    want = np.max(np.abs(H.dense(design).T @ y.ravel(order="F"))) / 24.0
    assert K.lambda_max(design, "gaussian", y) == pytest.approx(want, rel=1e-13)
    for fam in ("gaussian", "binomial", "poisson", "gamma"):
        d = bspline_design((30, 20), (8, 6))
        yy = H.random_data(rng, fam, (30, 20))
        assert K.lambda_max(d, fam, yy) == pytest.approx(O.lambda_max(d, fam, yy), rel=1e-12)
    d2 = H.make_design(rng, (3, 2), [(2, 2)])
    assert K.lambda_max(d2, "gaussian", np.zeros((3, 2))) == 0.0
    with pytest.raises(ValueError):
        K.lambda_max(d2, "poisson", -np.ones((3, 2)))


# -------------------------------------------------------------------- path
def compare_paths(got, want, coef_rtol=COEF_RTOL, obj_rtol=OBJ_RTOL, check_iters=True):
    assert got["truncated"] == want["truncated"]
    assert len(got["lambdas"]) == len(want["lambdas"])
    np.testing.assert_allclose(got["lambdas"], want["lambdas"], rtol=1e-13)
    worst = 0.0
    for t in range(len(want["lambdas"])):
        cg, cw = H.flat(got["coefficients"][t]), H.flat(want["coefficients"][t])
        assert np.array_equal(cg != 0, cw != 0), f"support differs at lambda {t}"
        scale = max(np.max(np.abs(cw)), 1e-300)
        err = np.max(np.abs(cg - cw)) / scale if cw.size else 0.0
        worst = max(worst, err)
        assert err <= coef_rtol, f"lambda {t}: coef rel err {err:.3e}"
        fo, fg = want["objectives"][t], got["objectives"][t]
        assert abs(fg - fo) <= obj_rtol * max(abs(fo), 1e-300), f"lambda {t}: objective"
        if check_iters:
            assert got["outer_iters"][t] == want["outer_iters"][t], f"lambda {t}: outer iterations"
            assert got["inner_iters"][t] == want["inner_iters"][t], f"lambda {t}: inner iterations"
    return worst


def test_gaussian_path_matches_oracle_c1_shape():
    d = configs.make("C1")
    kw = dict(n_lambda=100, lambda_min_ratio=1e-4)
    got = K.fit_path(d["design"], "gaussian", d["y"], **kw)
    want = O.fit_path(d["design"], "gaussian", d["y"], **kw)
    assert got["lambda_max"] == pytest.approx(want["lambda_max"], rel=1e-12)
    compare_paths(got, want)


def test_nonzero_counts_and_pinned_result_arrays():
    """fit_path's "nonzero" key (counted on the device) equals the counts of the
    returned coefficient arrays, which are views of a recycled page-locked
    block; a second fit must not overwrite the first fit's arrays."""
    d = configs.make("C1")
    kw = dict(n_lambda=20, lambda_min_ratio=1e-2)
    a = K.fit_path(d["design"], "gaussian", d["y"], **kw)
    first = [c.copy() for c in a["coefficients"][-1]]  # one array per component
    b = K.fit_path(d["design"], "gaussian", 2.0 * d["y"], **kw)
    for got in (a, b):
        for coef, nz in zip(got["coefficients"], got["nonzero"]):
            assert nz == int(sum(np.count_nonzero(c) for c in coef))
    for x, y in zip(first, a["coefficients"][-1]):
        assert np.array_equal(x, y)
    assert max(b["nonzero"]) > 0


def test_poisson_path_matches_oracle_small():
    rng = np.random.default_rng(5)
    design = bspline_design((24, 20, 30), (8, 6, 9))
    B = np.zeros((8, 6, 9))
    m = rng.random(B.shape) < 0.15
    B[m] = rng.standard_normal(m.sum())
    eta = configs.tensor_h(design[0], B)
    y = rng.poisson(np.exp(np.log(20.0) / eta.max() * eta)).astype(float)
    kw = dict(n_lambda=15, lambda_min_ratio=1e-3)
    got = K.fit_path(design, "poisson", y, **kw)
    want = O.fit_path(design, "poisson", y, **kw)
    compare_paths(got, want)


@pytest.mark.parametrize("fam", ["binomial", "gamma"])
def test_other_families_match_oracle(fam):
    rng = np.random.default_rng(11)
    design = bspline_design((20, 18), (7, 6))
    y = H.random_data(rng, fam, (20, 18))
    kw = dict(n_lambda=8, lambda_min_ratio=1e-2)
    compare_paths(K.fit_path(design, fam, y, **kw), O.fit_path(design, fam, y, **kw))


def test_two_component_design_generic_route():  # c = 2: unfused route
    rng = np.random.default_rng(72)
    design = H.make_design(rng, (5, 4, 3), [(3, 2, 2), (2, 2, 1)])
    eta = O.h_map(design, H.random_coef(rng, design, -0.7, 0.7))
    y = eta + rng.normal(0, 0.3, eta.shape)
    kw = dict(n_lambda=20, lambda_min_ratio=1e-3, inner_tol=1e-11)
    compare_paths(K.fit_path(design, "gaussian", y, **kw), O.fit_path(design, "gaussian", y, **kw))
    yp = rng.poisson(np.exp(0.3 * eta)).astype(float)
    kw = dict(n_lambda=8, lambda_min_ratio=1e-2)
    compare_paths(K.fit_path(design, "poisson", yp, **kw), O.fit_path(design, "poisson", yp, **kw))


def _masked_weights(shape):
    a = np.ones(int(np.prod(shape)))
    a[::4] = 0.0
    return np.asfortranarray(a.reshape(shape, order="F"))


GAUSS_CASES = {
    "ridge": dict(penalty="ridge", lambdas=[0.05, 0.02, 0.01, 0.005]),
    "elasticnet": dict(penalty="elasticnet", alpha=0.5, n_lambda=6),
    "masked_weights": dict(weights="masked", n_lambda=6),
    "nu_half": dict(nu=0.5, n_lambda=6),
    "inner_maxit": dict(n_lambda=6, inner_maxit=7),
    "nu_zero": dict(nu=0.0, n_lambda=6),  # backtracking every iteration (inner.cpp:169-183)
}


@pytest.mark.parametrize("case", sorted(GAUSS_CASES))
def test_gaussian_options_match_oracle(case):
    rng = np.random.default_rng(73)
    design = bspline_design((16, 14, 6), (6, 5, 4))
    y = rng.standard_normal((16, 14, 6))
    kw = dict(GAUSS_CASES[case])
    if kw.get("weights") == "masked":
        kw["weights"] = _masked_weights(y.shape)
    compare_paths(K.fit_path(design, "gaussian", y, **kw), O.fit_path(design, "gaussian", y, **kw))


@pytest.mark.parametrize("case", ["unit", "masked_weights", "nu_zero"])
def test_poisson_options_match_oracle(case):
    rng = np.random.default_rng(73)
    design = bspline_design((16, 14, 6), (6, 5, 4))
    yp = rng.poisson(1.5, size=(16, 14, 6)).astype(float)
    kw = dict(n_lambda=5, lambda_min_ratio=1e-2)
    if case == "unit":
        kw["iwls"] = "unit"
    elif case == "nu_zero":
        kw["nu"] = 0.0
    else:
        kw["weights"] = _masked_weights(yp.shape)
    compare_paths(K.fit_path(design, "poisson", yp, **kw), O.fit_path(design, "poisson", yp, **kw))


def test_constant_weight_gram_route_matches_oracle():
    """Constant prior weights take the Gram route (X^T W X = w (x)_j X_j^T X_j); a
    weight array with one differing cell takes the n-space route.  Both must
    match the oracle's n-space restatement."""
    rng = np.random.default_rng(81)
    design = bspline_design((18, 15, 8), (7, 6, 4))
    B = np.zeros((7, 6, 4))
    m = rng.random(B.shape) < 0.2
    B[m] = rng.standard_normal(m.sum())
    y = np.asfortranarray(configs.tensor_h(design[0], B) + 0.5 * rng.standard_normal((18, 15, 8)))
    a = np.full(y.shape, 2.5, order="F")
    kw = dict(n_lambda=12, lambda_min_ratio=1e-3)
    compare_paths(K.fit_path(design, "gaussian", y, weights=a, **kw),
                  O.fit_path(design, "gaussian", y, weights=a, **kw))
    a2 = a.copy()
    a2[3, 4, 5] = 2.0
    compare_paths(K.fit_path(design, "gaussian", y, weights=a2, **kw),
                  O.fit_path(design, "gaussian", y, weights=a2, **kw))


def test_masked_cells_insulated_on_gpu():  # test_path.cpp:115-138
    rng = np.random.default_rng(74)
    design = bspline_design((12, 10, 6), (5, 4, 4))
    for fam in ("gaussian", "poisson"):
        y = H.random_data(rng, fam, (12, 10, 6))
        a = np.ones(y.size)
        a[::4] = 0.0
        a = a.reshape(y.shape, order="F")
        base = K.fit_path(design, fam, y, weights=a, n_lambda=8, lambda_min_ratio=1e-2)
        y2 = y.ravel(order="F").copy()
        y2[::4] = 0.75
        other = K.fit_path(design, fam, y2.reshape(y.shape, order="F"), weights=a, n_lambda=8,
                           lambda_min_ratio=1e-2)
        for c1, c2 in zip(base["coefficients"], other["coefficients"]):
            assert np.max(np.abs(H.flat(c1) - H.flat(c2))) <= 1e-10


def test_truncation_first_model_failure_and_errors():  # test_path.cpp:241-283
    rng = np.random.default_rng(79)
    design = H.make_design(rng, (5, 4, 3), [(2, 2, 2)])
    y = H.random_data(rng, "poisson", (5, 4, 3))
    lmax = K.lambda_max(design, "poisson", y)
    p = K.fit_path(design, "poisson", y, n_lambda=6, lambda_min_ratio=1e-3, maxit=1, tol=1e-14)
    q = O.fit_path(design, "poisson", y, n_lambda=6, lambda_min_ratio=1e-3, maxit=1, tol=1e-14)
    assert p["truncated"] and len(p["lambdas"]) == len(q["lambdas"])
    with pytest.raises(RuntimeError):
        K.fit_path(design, "poisson", y, lambdas=[0.5 * lmax, 0.25 * lmax], maxit=1, tol=1e-14)
    with pytest.raises(ValueError):
        K.fit_path(design, "gaussian", y, penalty="ridge")
    with pytest.raises(ValueError):
        K.fit_path(design, "gaussian", y, lambdas=[0.1, 0.1])
    with pytest.raises(ValueError):
        K.fit_path(design, "poisson", -y - 1.0)


def test_single_lambda_and_boundary():  # test_path.cpp:49-60, acceptance criterion 8
    rng = np.random.default_rng(71)
    design = H.make_design(rng, (4, 3), [(2, 3)])
    y = rng.standard_normal((4, 3))
    p = K.fit_path(design, "gaussian", y, n_lambda=1)
    assert len(p["lambdas"]) == 1 and p["lambdas"][0] == p["lambda_max"]
    assert np.max(np.abs(H.flat(p["coefficients"][0]))) == 0.0


def test_predict_matches_dense():  # test_path.cpp:140-158
    rng = np.random.default_rng(74)
    design = H.make_design(rng, (4, 3), [(2, 3)])
    th = H.random_coef(rng, design)
    eta, mu = K.predict(design, "poisson", th)
    e = H.dense(design) @ H.flat(th)
    assert np.max(np.abs(eta.ravel(order="F") - e)) <= 1e-12
    assert np.max(np.abs(mu.ravel(order="F") - np.exp(e))) <= 1e-12
    eta0, mu0 = K.predict(design, "poisson", [np.zeros((2, 3))])
    assert np.all(eta0 == 0.0) and np.all(mu0 == 1.0)


def test_runs_are_bitwise_deterministic():  # test_outer.cpp:363-395 analogue
    d = configs.make("C1")
    a = K.fit_path(d["design"], "gaussian", d["y"], n_lambda=20)
    b = K.fit_path(d["design"], "gaussian", d["y"], n_lambda=20)
    for ca, cb in zip(a["coefficients"], b["coefficients"]):
        assert np.array_equal(H.flat(ca), H.flat(cb))
    assert a["objectives"] == b["objectives"]


def test_full_size_adjoint_property_c2():
    """Size-independent property at a BASELINE size: <H theta, u> = <theta, G u>."""
    rng = np.random.default_rng(2)
    d = configs.make("C2")
    D = K.Design(d["design"])
    th = [rng.standard_normal(d["p"])]
    u = rng.standard_normal(d["n"])
    lhs = float(np.vdot(K.h_map(D, th), u))
    rhs = float(H.flat(th) @ H.flat(K.g_map(D, u)))
    assert abs(lhs - rhs) <= 1e-11 * max(1.0, abs(rhs))


def test_c2_full_size_path_prefix_matches_oracle():
    """BASELINE config C2 at full size through the resident whole-path kernel:
    the bulk coefficient copy equals the per-model reads, and the first models
    of the path match the oracle's warm-started outer_solve (same support,
    coefficients and objective within 1e-8, same inner iteration counts)."""
    d = configs.make("C2")
    ctx = K.Context(0)
    D = K.Design(d["design"], ctx)
    obs = K.Observation(D, d["y"])
    lmax = O.lambda_max(d["design"], "gaussian", d["y"])
    assert abs(K.lambda_max(D, "gaussian", d["y"]) - lmax) <= 1e-13 * lmax
    nl, ratio = d["n_lambda"], d["lambda_min_ratio"]
    lams = [lmax * np.exp(np.log(ratio) / (nl - 1) * t) if t else lmax for t in range(nl)]
    res = K.fit_path_resident(D, obs, "gaussian", lambdas=lams)  # the same inputs on both sides
    assert res.n_models == d["n_lambda"] and not res.truncated
    allc = res.coefs()
    for t in (0, 1, res.n_models // 2, res.n_models - 1):
        assert np.array_equal(allc[t], res.coef(t))
    O.set_threads(os.cpu_count() or 1)
    init = None
    for t in range(3):
        r = O.outer_solve(d["design"], "gaussian", d["y"], res.lambdas[t], init=init)
        init = r["coef"]
        w, g = r["coef_flat"], allc[t]
        assert np.array_equal(g != 0, w != 0), f"support differs at lambda {t}"
        assert np.max(np.abs(g - w)) <= COEF_RTOL * max(np.max(np.abs(w)), 1e-300)
        assert abs(res.objectives[t] - r["final_objective"]) <= OBJ_RTOL * abs(r["final_objective"])
        assert res.inner_iters[t] == sum(int(x["inner_iterations"]) for x in r["iterations"])


def _fused_pass_bytes(D, obs):
    import ctypes as C
    from paper_1510_03298_b200 import _lib
    ms, b = C.c_double(), C.c_double()
    D.ctx.check(_lib.load().kg_time_kernel(D.ctx.h, D.h, obs.h, 0, 2, C.byref(ms), C.byref(b)))
    return b.value


def test_sharded_context_world1_nccl_matches_unsharded():
    """kg_ctx_create_sharded with a real one-rank NCCL communicator: every
    cross-slab all-reduce runs (identity on one rank) and the sharded n-space
    loop is host driven; paths equal the unsharded ones."""
    uid = K.nccl_unique_id()
    assert len(uid) == 128
    ctx = K.Context.sharded(0, 0, 1, uid)
    rng = np.random.default_rng(17)
    design = bspline_design((20, 16, 12), (7, 6, 5))
    B = np.zeros((7, 6, 5))
    m = rng.random(B.shape) < 0.2
    B[m] = rng.standard_normal(m.sum())
    eta = configs.tensor_h(design[0], B)
    y = rng.poisson(np.exp(np.log(15.0) / eta.max() * eta)).astype(float)
    for fam, yy in (("poisson", y), ("gaussian", eta + rng.normal(0, 0.2, eta.shape))):
        kw = dict(n_lambda=6, lambda_min_ratio=1e-2)
        D = K.Design(design, ctx)
        got = K.fit_path_resident(D, K.Observation(D, yy), fam, **kw)
        want = K.fit_path(design, fam, yy, **kw)
        res = {"lambdas": got.lambdas, "objectives": got.objectives, "truncated": got.truncated,
               "coefficients": [D.blocks(c) for c in got.coefs()], "outer_iters": got.outer_iters,
               "inner_iters": got.inner_iters}
        compare_paths(res, want)
    ctx.close()


def test_local_slab_contexts_partition_the_operator_maps():
    """World-2 sharded contexts without a communicator (local partials): each
    rank's design keeps its rows of X_d, h_map gives that slab of eta and the
    g_map partials sum to the full X^T u (G = sum_g G_g)."""
    rng = np.random.default_rng(23)
    n, p = (12, 10, 9), (5, 4, 4)
    design = bspline_design(n, p)
    th = [rng.standard_normal(p)]
    u = rng.standard_normal(n)
    eta_full = K.h_map(design, th)
    g_full = H.flat(K.g_map(design, u))
    total = np.zeros_like(g_full)
    for r in range(2):
        ctx = K.Context.sharded(0, r, 2, None)
        D = K.Design(design, ctx)
        lo, hi = K.shard_rows(n[-1], r, 2)
        assert D.local_row_dims == (n[0], n[1], hi - lo)
        np.testing.assert_allclose(K.h_map(D, th), eta_full[:, :, lo:hi], rtol=0, atol=1e-13)
        total += H.flat(K.g_map(D, np.asfortranarray(u[:, :, lo:hi])))
        D.close()
        ctx.close()
    np.testing.assert_allclose(total, g_full, rtol=1e-13, atol=1e-13)


def test_mse_heldout_matches_oracle_and_is_u_shaped():
    """kg_mse_heldout (path.cpp:91-126) on the device against the oracle, on the
    reference's held-out workflow (test_path.cpp:195-237): held-out cells get
    zero observation weight in the fit and the held-out SSE curve is U-shaped."""
    rng = np.random.default_rng(76)
    n1, n2 = 16, 14
    X1 = K.bspline_design(np.arange(1.0, n1 + 1), 4, 10)
    X2 = K.bspline_design(np.arange(1.0, n2 + 1), 4, 9)
    design = [[X1, X2]]
    i, j = np.meshgrid(np.arange(1, n1 + 1), np.arange(1, n2 + 1), indexing="ij")
    truth = 3.0 * np.sin(2 * np.pi * i / 16.0) * np.cos(2 * np.pi * j / 14.0)
    y = np.asfortranarray(truth + rng.standard_normal((n1, n2)))
    mask = np.zeros(n1 * n2)
    a = np.ones(n1 * n2)
    mask[3::7] = 1.0
    a[3::7] = 0.0
    mask = np.asfortranarray(mask.reshape((n1, n2), order="F"))
    a = np.asfortranarray(a.reshape((n1, n2), order="F"))
    D = K.Design(design)
    res = K.fit_path_resident(D, K.Observation(D, y, a), "gaussian", n_lambda=20, lambda_min_ratio=1e-5)
    assert not res.truncated
    got = K.mse_heldout(res, "gaussian", y, mask)
    want = O.mse_heldout(design, "gaussian", [D.blocks(c) for c in res.coefs()], y, mask)
    np.testing.assert_allclose(got["mse"], want["mse"], rtol=1e-12)
    assert got["argmin"] == want["argmin"]
    assert 0 < got["argmin"] < res.n_models - 1
    with pytest.raises(ValueError):
        K.mse_heldout(res, "gaussian", y, np.zeros_like(mask))
    bad = mask.copy()
    bad[0, 0] = 2.0
    with pytest.raises(ValueError):
        K.mse_heldout(res, "gaussian", y, bad)


@pytest.mark.parametrize("case", ["poisson_c1", "binomial_2d", "two_component"])
def test_tensor_weights_match_oracle(case):
    """iwls = "tensor" (compute_weights' geometric-mean factors, GramBlocks,
    xtwx_apply_tensor, lipschitz_tensor_exact; outer.cpp:53-103,
    design.cpp:126-177, inner.cpp:73-91) against the oracle."""
    rng = np.random.default_rng(31)
    if case == "poisson_c1":
        design = bspline_design((18, 14, 10), (6, 5, 4))
        B = np.zeros((6, 5, 4))
        m = rng.random(B.shape) < 0.3
        B[m] = rng.standard_normal(m.sum())
        eta = configs.tensor_h(design[0], B)
        y = rng.poisson(np.exp(np.log(12.0) / eta.max() * eta)).astype(float)
        fam = "poisson"
    elif case == "binomial_2d":
        design = bspline_design((20, 18), (7, 6))
        y = H.random_data(rng, "binomial", (20, 18))
        fam = "binomial"
    else:
        design = H.make_design(rng, (6, 5, 4), [(3, 2, 2), (2, 2, 2)])
        eta = O.h_map(design, H.random_coef(rng, design, -0.5, 0.5))
        y = rng.poisson(np.exp(0.4 * eta)).astype(float)
        fam = "poisson"
    kw = dict(n_lambda=6, lambda_min_ratio=1e-2, iwls="tensor")
    compare_paths(K.fit_path(design, fam, y, **kw), O.fit_path(design, fam, y, **kw))


def _slab_route_taken(design, y):
    """kg_time_kernel(which=6) runs only on a design whose fits take the slab route."""
    import ctypes as C
    from paper_1510_03298_b200 import _lib
    ctx = K.Context(0)
    D = K.Design(design, ctx)
    obs = K.Observation(D, y)
    ms, b = C.c_double(), C.c_double()
    st = _lib.load().kg_time_kernel(ctx.h, D.h, obs.h, 6, 1, C.byref(ms), C.byref(b))
    ctx.close()
    return st == 0


SLAB_SHAPES = [((60, 52, 30), (14, 12, 8)),    # tail chunk (52 = 6 x 8 + 4), p1 not a multiple of 8: k_slab2
               ((32, 72, 24), (10, 20, 7)),    # odd chunk count (9), several column groups (n1 = 32): k_slab2
               ((128, 40, 17), (32, 10, 6)),   # odd chunk count, odd last mode: k_slab2
               ((64, 48, 20), (16, 12, 6)),    # whole chunk pairs: k_slab4 (bulk-copy v ring)
               ((60, 48, 30), (14, 12, 8)),    # k_slab4 with a partly active row warp (15 quads), padded row groups
               ((256, 32, 6), (64, 10, 4))]    # k_slab4 at the largest mode-1 extents (all 256 row threads)


@pytest.mark.parametrize("n,p", SLAB_SHAPES)
def test_slab_route_poisson_paths_match_oracle(n, p):
    """The slab pass (modes 1 and 2 of X^T W X fused per last-mode slice:
    k_slab4 on whole chunk pairs, k_slab2 otherwise) on irregular shapes -- a
    partial last chunk of mode-2 rows, odd chunk counts, p1 with padded row
    groups, several row-thread column groups, partly active row warps --
    against the oracle's Poisson path (same supports, coefficients, objectives
    and iteration counts)."""
    rng = np.random.default_rng(sum(n) + sum(p))
    design = bspline_design(n, p)
    B = np.zeros(p)
    m = rng.random(p) < 0.15
    B[m] = rng.standard_normal(m.sum())
    eta = configs.tensor_h(design[0], B)
    y = rng.poisson(np.exp(np.log(20.0) / max(eta.max(), 1e-3) * eta)).astype(float)
    assert _slab_route_taken(design, y), "this shape should run the slab route"
    kw = dict(n_lambda=8, lambda_min_ratio=1e-2)
    got = K.fit_path(design, "poisson", y, **kw)
    want = O.fit_path(design, "poisson", y, **kw)
    compare_paths(got, want)


@pytest.mark.gpu
@pytest.mark.parametrize("switch", ["KG_SLAB_K2", "KG_SLAB_DMMA"])
def test_slab_fallback_kernels_match_oracle(switch):
    """The slab-pass kernels behind the default one -- k_slab2 (register-staged
    v, taken on odd chunk counts) and k_slab (Y by DMMA, taken without a gather
    table) -- forced by their developer switches onto the k_slab4 shapes, in a
    fresh process (the switches are read once)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, KG_DEV="1", **{switch: "1"})
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.join(root, "tests", "test_gpu_parity.py"), "-m", "gpu",
                        "-q", "-x", "-k", "test_slab_route_poisson_paths_match_oracle"],
                       env=env, cwd=root, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "6 passed" in r.stdout, r.stdout[-500:]


_FIT_DUMP = """
import sys, numpy as np
sys.path.insert(0, {root!r})
from paper_1510_03298_b200 import configs
from paper_1510_03298_b200 import kronglm as K
n, p = (64, 48, 20), (16, 12, 6)
design = [[K.bspline_design(np.linspace(0, 1, a), 4, b) for a, b in zip(n, p)]]
rng = np.random.default_rng(7)
B = np.zeros(p); m = rng.random(p) < 0.15; B[m] = rng.standard_normal(m.sum())
eta = configs.tensor_h(design[0], B)
y = rng.poisson(np.exp(np.log(20.0) / max(eta.max(), 1e-3) * eta)).astype(float)
out = K.fit_path(design, "poisson", y, n_lambda=8, lambda_min_ratio=1e-2)
np.savez({dst!r}, coef=np.stack([c[0].ravel(order="F") for c in out["coefficients"]]),
         obj=np.array(out["objectives"]), inner=np.array(out["inner_iters"]))
"""


@pytest.mark.gpu
def test_forked_control_and_dependent_launches_change_nothing(tmp_path):
    """The slab route's FISTA body runs the control kernel beside the mode-3 G
    step and chains its n-space kernels by programmatic dependent launch.  With
    both switched off (KG_NO_FORK, KG_NO_PDL: the serial body) the fit must be
    bitwise identical: the overlap may not reorder anything that is read."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for tag, extra in (("overlap", {}), ("serial", {"KG_DEV": "1", "KG_NO_FORK": "1", "KG_NO_PDL": "1"})):
        dst = str(tmp_path / f"{tag}.npz")
        r = subprocess.run([sys.executable, "-c", _FIT_DUMP.format(root=root, dst=dst)], env=dict(os.environ, **extra),
                           cwd=root, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(np.load(dst))
    a, b = outs
    assert np.array_equal(a["inner"], b["inner"])
    assert np.array_equal(a["obj"], b["obj"])
    assert np.array_equal(a["coef"], b["coef"])
    assert a["inner"].sum() > 100
