"""Pins the CPU oracle (oracle/kronglm_oracle.cpp) against the reference's own
known-answer and property tests.  Each test cites the reference test it ports.
These run without a GPU (the oracle is the parity checker for the CUDA path)."""
import numpy as np
import pytest

from oracle import oracle as O
from tests import helpers as H

FAMS = ["gaussian", "binomial", "poisson", "gamma"]


# ---------------------------------------------------------------- array core
def test_linear_index_known_answers():  # test_array.cpp:50-57, test_smoke.py:19-22
    assert O.linear_index([1, 1], [2, 3]) == 1
    assert O.linear_index([2, 3], [2, 3]) == 6
    assert O.linear_index([2, 1, 2], [2, 3, 2]) == 8
    for bad in ([0, 1], [1, 4]):
        with pytest.raises(ValueError):
            O.linear_index(bad, [2, 3])
    with pytest.raises(ValueError):
        O.linear_index([1], [2, 3])


def test_linear_index_bijection():  # test_array.cpp:59-77
    for ext in ([2, 3, 2], [7], [17, 3, 5, 4], [1, 9, 1]):
        seen = set()
        for idx in np.ndindex(*ext[::-1]):
            pos = O.linear_index([i + 1 for i in idx[::-1]], ext)
            assert 1 <= pos <= int(np.prod(ext))
            seen.add(pos)
        assert len(seen) == int(np.prod(ext))


def _rho_naive(x, a):
    """Entrywise definition of the rotated contraction (test_array.cpp:16-40)."""
    a2 = a.reshape(a.shape[0], -1, order="F")
    out = (x @ a2).T  # rest x r
    return out.reshape(tuple(a.shape[1:]) + (x.shape[0],), order="F")


def test_rho_identity_rotates():  # test_array.cpp:79-91
    rng = np.random.default_rng(11)
    a = rng.uniform(-1, 1, (3, 4, 2))
    r = O.rho(np.eye(3), a)
    assert r.shape == (4, 2, 3)
    for i1 in range(3):
        assert np.array_equal(r[:, :, i1], a[i1])


def test_rho_matches_naive():  # test_array.cpp:93-125
    rng = np.random.default_rng(13)
    x = rng.standard_normal((4, 3))
    a = rng.uniform(-1, 1, 3)
    assert np.max(np.abs(O.rho(x, a) - x @ a)) <= 1e-14
    for xs, ashape in (((2, 3), (3, 4)), ((4, 2), (2, 3, 5))):
        x = rng.standard_normal(xs)
        a = rng.uniform(-1, 1, ashape)
        assert np.max(np.abs(O.rho(x, a) - _rho_naive(x, a))) <= 1e-13
    with pytest.raises(ValueError):
        O.rho(rng.standard_normal((2, 4)), rng.uniform(-1, 1, (3, 4)))


def test_h_g_match_dense_kron():  # test_array.cpp:142-151, test_smoke.py:25-49
    rng = np.random.default_rng(1)
    design = H.make_design(rng, (4, 3, 2), [(2, 3, 2), (3, 2, 1)])
    theta = H.random_coef(rng, design)
    xd = H.dense(design)
    eta = O.h_map(design, theta)
    assert eta.shape == (4, 3, 2)
    assert np.max(np.abs(eta.ravel(order="F") - xd @ H.flat(theta))) <= 1e-12
    u = rng.standard_normal((4, 3, 2))
    g = H.flat(O.g_map(design, u))
    assert np.max(np.abs(g - xd.T @ u.ravel(order="F"))) <= 1e-12
    lhs, rhs = float(np.vdot(eta, u)), float(np.dot(H.flat(theta), g))
    assert abs(lhs - rhs) <= 1e-12 * max(1.0, abs(rhs))


def test_kronecker_corpus_adjoint_linearity():  # test_array.cpp:167-193, acceptance.cpp:53-80
    rng = np.random.default_rng(18)
    for _ in range(50):
        design = H.random_design(rng)
        xd = H.dense(design)
        th, th2 = H.random_coef(rng, design), H.random_coef(rng, design)
        u = rng.uniform(-1, 1, H.row_dims(design))
        h = O.h_map(design, th).ravel(order="F")
        g = H.flat(O.g_map(design, u))
        assert np.max(np.abs(h - xd @ H.flat(th))) <= 1e-12
        assert np.max(np.abs(g - xd.T @ u.ravel(order="F"))) <= 1e-12
        assert abs(h @ u.ravel(order="F") - H.flat(th) @ g) <= 1e-12 * max(1, abs(H.flat(th) @ g))
        mix = [0.3 * a - 1.7 * b for a, b in zip(th, th2)]
        want = 0.3 * h - 1.7 * O.h_map(design, th2).ravel(order="F")
        assert np.max(np.abs(O.h_map(design, mix).ravel(order="F") - want)) <= 1e-12


def test_identity_designs():  # test_array.cpp:127-165
    rng = np.random.default_rng(14)
    design = [[np.eye(3), np.eye(2), np.eye(4)]]
    th = H.random_coef(rng, design)
    assert np.max(np.abs(O.h_map(design, th) - th[0])) <= 1e-14
    design2 = [[np.eye(3), np.eye(2)], [np.eye(3), np.eye(2)]]
    u = rng.uniform(-1, 1, (3, 2))
    for blk in O.g_map(design2, u):
        assert np.array_equal(blk, u)


def test_xtwx_dense():  # test_array.cpp:195-219
    rng = np.random.default_rng(19)
    for _ in range(20):
        design = H.random_design(rng)
        xd = H.dense(design)
        th = H.random_coef(rng, design)
        v = rng.uniform(0, 2, H.row_dims(design))
        want = xd.T @ (v.ravel(order="F") * (xd @ H.flat(th)))
        assert np.max(np.abs(H.flat(O.xtwx_apply(design, v, th)) - want)) <= 1e-12


def test_dimension_mismatch():  # test_array.cpp:288-297
    rng = np.random.default_rng(21)
    design = H.make_design(rng, (3, 4), [(2, 2)])
    with pytest.raises(ValueError):
        O.g_map(design, rng.uniform(-1, 1, (4, 3)))
    with pytest.raises(ValueError):
        O.h_map(design, [rng.uniform(size=(3, 2))])


# -------------------------------------------------------------------- family
def test_family_closed_forms():  # test_family.cpp:35-186
    assert O.mean("gaussian", [0.7])[0] == pytest.approx(0.7, rel=1e-15)
    assert O.mean("binomial", [0.0])[0] == pytest.approx(0.5, rel=1e-15)
    assert O.mean("poisson", [1.0])[0] == pytest.approx(2.718281828459045, rel=1e-15)
    assert np.isfinite(O.mean("poisson", [1e4])[0])
    assert O.score("poisson", [3.0], [0.0])[0] == pytest.approx(2.0, rel=1e-15)
    assert O.glm_weights("gaussian", [0.0])[0] == 1.0
    assert O.glm_weights("binomial", [0.0])[0] == pytest.approx(0.25, rel=1e-15)
    assert O.glm_weights("poisson", [np.log(2.0)])[0] == pytest.approx(2.0, rel=1e-14)
    assert O.glm_weights("gamma", [-1.3])[0] == 1.0
    assert O.working_response("poisson", [3.0], [0.0])[0] == pytest.approx(2.0, rel=1e-15)
    rng = np.random.default_rng(34)
    for fam in FAMS:
        w = O.glm_weights(fam, rng.uniform(-200, 200, 40))
        assert np.all(w >= 1e-10) and np.all(w <= np.exp(30.0))


def test_loglik_values_and_evalerror():  # test_family.cpp:59-108
    rng = np.random.default_rng(31)
    y = rng.uniform(-2, 2, 12)
    assert O.loglik("gaussian", y, y) == pytest.approx(0.5 * y @ y, rel=1e-14)
    assert O.loglik("poisson", np.zeros(6), np.zeros(6)) == pytest.approx(-6.0, rel=1e-15)
    y = np.zeros(4)
    y[2] = 1e308
    with pytest.raises(O.EvalError) as ei:
        O.loglik("gaussian", y, np.full(4, 1e4))
    assert ei.value.cell == 2


def test_score_finite_differences():  # test_family.cpp:121-145, acceptance criterion 3
    rng = np.random.default_rng(33)
    for fam in FAMS:
        for _ in range(10):
            n = int(rng.integers(1, 17))
            y = H.random_data(rng, fam, n)
            a = np.ones(n)
            a[3::5] = 0.0
            eta = rng.uniform(-2, 2, n)
            u = O.score(fam, y, eta, a)
            for i in range(n):
                h = 1e-6 * max(1.0, abs(eta[i]))
                lo, hi = eta.copy(), eta.copy()
                lo[i] -= h
                hi[i] += h
                fd = (O.loglik(fam, y, hi, a) - O.loglik(fam, y, lo, a)) / (2 * h)
                assert abs(fd - u[i]) <= 1e-6 * max(1.0, abs(u[i]))


def test_working_response_identity():  # test_family.cpp:188-206
    rng = np.random.default_rng(36)
    for fam in FAMS:
        for _ in range(5):
            n = int(rng.integers(1, 30))
            y = H.random_data(rng, fam, n)
            eta = rng.uniform(-2, 2, n)
            z = O.working_response(fam, y, eta)
            gen = O.score(fam, y, eta) / O.glm_weights(fam, eta) + eta
            assert np.all(np.abs(z - gen) <= 1e-12 * np.maximum(1.0, np.abs(gen)))


def test_zero_weight_insulation_family():  # test_family.cpp:208-228
    rng = np.random.default_rng(37)
    for fam in FAMS:
        y = H.random_data(rng, fam, 12)
        a = np.ones(12)
        a[[5, 7]] = 0
        eta = rng.uniform(-2, 2, 12)
        y2 = y.copy()
        y2[5], y2[7] = 123.0, 0.25
        assert O.loglik(fam, y, eta, a) == O.loglik(fam, y2, eta, a)
        assert np.array_equal(O.score(fam, y, eta, a), O.score(fam, y2, eta, a))


def test_validate():  # test_family.cpp:249-268
    y = np.array([-0.5, 0.0])
    for fam in ("poisson", "gamma"):
        with pytest.raises(ValueError):
            O.validate(fam, y)
    y = np.array([1.5, 0.0])
    with pytest.raises(ValueError):
        O.validate("binomial", y)
    O.validate("gaussian", y)
    O.validate("binomial", y, np.array([0.0, 1.0]))


# ------------------------------------------------------------------- penalty
def test_penalty_values_and_prox():  # test_penalty.cpp:22-54
    th = np.array([1.0, -2.0, 0.0])
    assert O.penalty_value(th, "lasso") == pytest.approx(3.0, rel=1e-15)
    assert O.penalty_value(th, "ridge") == pytest.approx(5.0, rel=1e-15)
    assert O.penalty_value([2.0, 0.0], "elasticnet", 0.5) == pytest.approx(4.0, rel=1e-15)
    out = O.prox([3.0, -0.5], 1.0)
    assert out[0] == pytest.approx(2.0, rel=1e-15) and out[1] == 0.0
    assert O.prox([4.0], 0.5, "ridge")[0] == pytest.approx(2.0, rel=1e-15)
    z = np.random.default_rng(41).standard_normal(5)
    assert np.max(np.abs(O.prox(z, 1e-300) - z)) <= 1e-12
    with pytest.raises(ValueError):
        O.prox(z, 0.0)


def test_prox_grid_optimality():  # test_penalty.cpp:56-82
    rng = np.random.default_rng(42)
    for pen, al in (("lasso", 0.0), ("ridge", 0.0), ("elasticnet", 0.7)):
        for _ in range(3):
            z = rng.uniform(-3, 3, 2)
            g = rng.uniform(0.1, 2.0)
            best = O.prox(z, g, pen, al)

            def f(x):
                return 0.5 * np.sum((x - z) ** 2) + g * O.penalty_value(x, pen, al)

            fb = f(best)
            span = np.max(np.abs(z)) + 1.0
            for xi in np.linspace(-span, span, 41):
                for xj in np.linspace(-span, span, 41):
                    assert fb <= f(np.array([xi, xj])) + 1e-12


def test_lambda_max_closed_form():  # test_penalty.cpp:107-116, test_smoke.py:72-79
    rng = np.random.default_rng(44)
    design = H.make_design(rng, (4, 3, 2), [(2, 2, 2)])
    y = rng.standard_normal((4, 3, 2))
    want = np.max(np.abs(H.dense(design).T @ y.ravel(order="F"))) / 24.0
    assert O.lambda_max(design, "gaussian", y) == pytest.approx(want, rel=1e-13)
    d2 = H.make_design(rng, (3, 2), [(2, 2)])
    assert O.lambda_max(d2, "gaussian", np.zeros((3, 2))) == 0.0
    assert O.lambda_max(d2, "poisson", np.ones((3, 2))) == pytest.approx(0.0, abs=1e-15)
    with pytest.raises(ValueError):
        O.lambda_max(d2, "gaussian", rng.standard_normal((3, 2)), penalty="ridge")


def test_zero_at_lambda_max():  # test_penalty.cpp:139-158, acceptance criterion 8
    rng = np.random.default_rng(46)
    for fam in ("gaussian", "poisson"):
        design = H.make_design(rng, (4, 3, 2), [(2, 2, 2)])
        y = H.random_data(rng, fam, (4, 3, 2))
        lmax = O.lambda_max(design, fam, y)
        assert lmax > 0
        above = O.outer_solve(design, fam, y, lmax * (1 + 1e-6), inner_tol=1e-10)
        assert np.max(np.abs(above["coef_flat"])) == 0.0
        below = O.outer_solve(design, fam, y, lmax * 0.99, inner_tol=1e-10)
        assert np.max(np.abs(below["coef_flat"])) > 0.0


# ------------------------------------------------------------ spectral/inner
def test_spectral_radius_vs_eigh():
    rng = np.random.default_rng(50)
    for _ in range(10):
        x = rng.standard_normal((6, 4))
        g = x.T @ x
        assert O.spectral_radius(g) == pytest.approx(np.linalg.eigvalsh(g).max(), rel=1e-10)


def test_lipschitz_upper():  # test_inner.cpp:41-69, acceptance criterion 4
    design = [[np.eye(2), np.eye(3)]]
    assert O.lipschitz_upper(design, np.ones((2, 3))) == pytest.approx(1.0 / 6.0, rel=1e-12)
    rng = np.random.default_rng(52)
    for _ in range(20):
        design = H.random_design(rng)
        v = rng.uniform(0.3, 2.0, H.row_dims(design))
        xd = H.dense(design)
        exact = np.linalg.eigvalsh(xd.T @ (v.ravel(order="F")[:, None] * xd)).max() / xd.shape[0]
        up = O.lipschitz_upper(design, v)
        assert up >= exact * (1 - 1e-12)
        assert O.lipschitz_upper(design, 3.5 * v) == pytest.approx(3.5 * up, rel=1e-12)


def test_fista_known_answers():  # test_inner.cpp:155-198
    rng = np.random.default_rng(55)
    design = H.make_design(rng, (3, 4), [(2, 3)])
    v = rng.uniform(0.3, 2.0, (3, 4))
    z = rng.uniform(-1, 1, (3, 4))
    xtwz = H.dense(design).T @ (v * z).ravel(order="F")
    lam = 2.0 * np.max(np.abs(xtwz)) / 12.0
    res = O.fista_solve(design, v, z, lam)
    assert np.max(np.abs(res["coef_flat"])) == 0.0 and res["converged"]

    design = [[np.eye(3), np.eye(2), np.eye(2)]]
    z = rng.uniform(-1, 1, (3, 2, 2))
    res = O.fista_solve(design, np.ones((3, 2, 2)), z, 0.0, inner_tol=1e-14, inner_maxit=10000)
    assert np.max(np.abs(res["coef_flat"] - z.ravel(order="F"))) <= 1e-12

    design = H.make_design(rng, (4, 6), [(2, 6)])
    v = rng.uniform(0.3, 2.0, (4, 6))
    z = rng.uniform(-2, 2, (4, 6))
    res = O.fista_solve(design, v, z, 0.05, inner_tol=1e-13, inner_maxit=50000)
    xd = H.dense(design)
    star = H.dense_gaussian_minimizer(xd, v.ravel(order="F"), z.ravel(order="F"), 0.05)
    r = xd @ star - z.ravel(order="F")
    g_star = 0.5 * np.sum(v.ravel(order="F") * r * r) / 24 + 0.05 * np.abs(star).sum()
    assert abs(res["objective"] - g_star) <= 1e-8


def test_fista_rate_certificate():  # test_inner.cpp:201-231, acceptance criterion 5
    rng = np.random.default_rng(56)
    for _ in range(5):
        design = H.make_design(rng, (4, 3, 3), [(3, 2, 2)])
        v = rng.uniform(0.5, 2.0, (4, 3, 3))
        z = rng.uniform(-2, 2, (4, 3, 3))
        init = H.random_coef(rng, design)
        res = O.fista_solve(design, v, z, 0.02, init=init, inner_tol=0.0, inner_maxit=150, record_history=True)
        xd = H.dense(design)
        star = H.dense_gaussian_minimizer(xd, v.ravel(order="F"), z.ravel(order="F"), 0.02, iters=30000)
        r = xd @ star - z.ravel(order="F")
        g_star = 0.5 * np.sum(v.ravel(order="F") * r * r) / 36 + 0.02 * np.abs(star).sum()
        d0 = np.sum((H.flat(init) - star) ** 2)
        for k, g in res["history"]:
            if k == 0:
                continue
            assert g - g_star <= 2 * res["lipschitz"] * d0 / (k + 1) ** 2 + 1e-12 * max(1, abs(g_star))


def test_fista_nu_modes_and_monitoring():  # test_inner.cpp:233-316
    rng = np.random.default_rng(59)
    design = H.make_design(rng, (5, 3), [(3, 2)])
    v = rng.uniform(0.3, 2.0, (5, 3))
    z = rng.uniform(-1, 1, (5, 3))
    fast = O.fista_solve(design, v, z, 0.02, nu=0.0, inner_tol=1e-12, inner_maxit=20000)
    safe = O.fista_solve(design, v, z, 0.02, nu=1.0, inner_tol=1e-12, inner_maxit=20000)
    half = O.fista_solve(design, v, z, 0.02, nu=0.5, inner_tol=1e-12, inner_maxit=20000)
    sparse = O.fista_solve(design, v, z, 0.02, inner_tol=1e-12, inner_maxit=20000, monitor_every=10)
    assert fast["converged"] and safe["converged"] and sparse["converged"]
    for other in (fast, half, sparse):
        assert abs(other["objective"] - safe["objective"]) <= 1e-9 * max(1, abs(safe["objective"]))
    res = O.fista_solve(design, v, z, 0.05, extrapolation="none", inner_tol=0.0, inner_maxit=200,
                        init=H.random_coef(rng, design), record_history=True)
    gs = [g for _, g in res["history"]]
    assert all(b <= a + 1e-12 for a, b in zip(gs, gs[1:]))


def test_fista_rejects_bad_problems():  # test_inner.cpp:318-336
    rng = np.random.default_rng(62)
    design = H.make_design(rng, (4, 3), [(2, 2)])
    v = rng.uniform(0.3, 2.0, (4, 3))
    v[0, 0] = -0.1
    with pytest.raises(ValueError):
        O.fista_solve(design, v, rng.uniform(size=(4, 3)), 0.0)


# --------------------------------------------------------------------- outer
def test_gaussian_shortcut_matches_fista():  # test_outer.cpp:179-202
    rng = np.random.default_rng(65)
    design = H.make_design(rng, (4, 3, 2), [(2, 2, 2)])
    y = rng.standard_normal((4, 3, 2))
    res = O.outer_solve(design, "gaussian", y, 0.05, inner_tol=1e-12, inner_maxit=50000)
    assert res["weight_evaluations"] == 1 and res["status"] == "converged" and len(res["iterations"]) == 1
    direct = O.fista_solve(design, np.ones((4, 3, 2)), y, 0.05, inner_tol=1e-12, inner_maxit=50000)
    assert np.max(np.abs(res["coef_flat"] - direct["coef_flat"])) <= 1e-10


def test_poisson_outer_vs_dense():  # test_outer.cpp:219-246
    rng = np.random.default_rng(67)
    design = H.make_design(rng, (6, 5, 4), [(3, 3, 3)])
    eta_true = rng.uniform(-1, 1.5, (6, 5, 4))
    y = rng.poisson(np.exp(eta_true)).astype(float)
    res = O.outer_solve(design, "poisson", y, 0.02, tol=1e-10, inner_tol=1e-12, inner_maxit=20000)
    assert res["status"] == "converged"
    objs = [res["initial_objective"]] + [r["objective"] for r in res["iterations"]]
    assert all(b <= a + 1e-12 * max(1, abs(a)) for a, b in zip(objs, objs[1:]))
    xd = H.dense(design)
    yf = y.ravel(order="F")
    star = H.dense_poisson_minimizer(xd, yf, 0.02, iters=20000)
    f_star = H.poisson_objective(xd, yf, star, 0.02)
    assert abs((res["final_objective"] - f_star) / abs(f_star)) <= 1e-4


def test_descent_every_family():  # test_outer.cpp:248-261
    rng = np.random.default_rng(68)
    for fam in FAMS:
        design = H.make_design(rng, (5, 4, 2), [(3, 2, 2)])
        y = H.random_data(rng, fam, (5, 4, 2))
        res = O.outer_solve(design, fam, y, 0.01)
        objs = [res["initial_objective"]] + [r["objective"] for r in res["iterations"]]
        assert all(b <= a + 1e-12 * max(1, abs(a)) for a, b in zip(objs, objs[1:]))
        assert res["status"] == "converged"


def test_weight_modes_agree():  # test_outer.cpp:262-291
    rng = np.random.default_rng(69)
    design = H.make_design(rng, (5, 4, 3), [(2, 2, 2)])
    y = rng.poisson(np.exp(rng.uniform(-0.8, 0.8, (5, 4, 3)))).astype(float)
    objs = []
    for mode in ("exact", "unit", "tensor"):
        res = O.outer_solve(design, "poisson", y, 0.01, iwls=mode, tol=1e-10, maxit=400, inner_tol=1e-12,
                            inner_maxit=20000)
        assert res["status"] == "converged"
        objs.append(res["final_objective"])
    assert abs(objs[1] - objs[0]) <= 1e-6 * max(1, abs(objs[0]))
    assert abs(objs[2] - objs[0]) <= 1e-6 * max(1, abs(objs[0]))


def test_malformed_outer_configs():  # test_outer.cpp:293-313
    rng = np.random.default_rng(80)
    design = H.make_design(rng, (3, 2), [(2, 2)])
    y = rng.standard_normal((3, 2))
    with pytest.raises(ValueError):
        O.outer_solve(design, "gaussian", y, 0.1, armijo_b=1.0)
    with pytest.raises(ValueError):
        O.outer_solve(design, "gaussian", y, 0.1, armijo_v=0.0)
    with pytest.raises(ValueError):
        O.outer_solve(design, "gaussian", y, -0.1)


# ---------------------------------------------------------------------- path
def test_lambda_sequence_and_single():  # test_path.cpp:27-60
    rng = np.random.default_rng(71)
    design = H.make_design(rng, (4, 3), [(2, 3)])
    y = rng.standard_normal((4, 3))
    p = O.fit_path(design, "gaussian", y, n_lambda=1)
    assert len(p["lambdas"]) == 1 and p["lambdas"][0] == p["lambda_max"]
    assert np.max(np.abs(H.flat(p["coefficients"][0]))) == 0.0 and not p["truncated"]
    p = O.fit_path(design, "gaussian", y, n_lambda=3, lambda_min_ratio=0.01)
    lm = p["lambda_max"]
    assert p["lambdas"][1] == pytest.approx(0.1 * lm, rel=1e-12)
    assert p["lambdas"][2] == pytest.approx(0.01 * lm, rel=1e-12)


def test_gaussian_desk_path_invariants():  # test_path.cpp:62-113
    rng = np.random.default_rng(72)
    design = H.make_design(rng, (5, 4, 3), [(3, 2, 2)])
    eta = O.h_map(design, H.random_coef(rng, design, -0.7, 0.7))
    y = eta + rng.normal(0, 0.3, eta.shape)
    p = O.fit_path(design, "gaussian", y, n_lambda=30, lambda_min_ratio=1e-3, inner_tol=1e-11)
    assert len(p["lambdas"]) == 30 and not p["truncated"]
    assert np.max(np.abs(H.flat(p["coefficients"][0]))) == 0.0
    xd = H.dense(design)
    yf = y.ravel(order="F")
    n = yf.size
    for t in range(1, 30):
        prev = H.flat(p["coefficients"][t - 1])
        e = xd @ prev
        f_prev = -np.sum(yf * e - 0.5 * e * e) / n + p["lambdas"][t] * np.abs(prev).sum()
        assert p["objectives"][t] <= f_prev + 1e-12 * max(1, abs(f_prev))


def test_masked_cells_insulated():  # test_path.cpp:115-138, acceptance criterion 10
    rng = np.random.default_rng(73)
    for fam in ("gaussian", "poisson"):
        design = H.make_design(rng, (4, 3, 2), [(2, 2, 2)])
        y = H.random_data(rng, fam, (4, 3, 2))
        a = np.ones((4, 3, 2))
        a.ravel(order="F")[::4] = 0.0
        af = np.asfortranarray(a)
        af_flat = af.ravel(order="F")
        af_flat[::4] = 0.0
        af = af_flat.reshape(a.shape, order="F")
        base = O.fit_path(design, fam, y, weights=af, n_lambda=8, lambda_min_ratio=1e-2)
        y2 = np.asfortranarray(y).ravel(order="F").copy()
        y2[::4] = 0.75
        other = O.fit_path(design, fam, y2.reshape(y.shape, order="F"), weights=af, n_lambda=8,
                           lambda_min_ratio=1e-2)
        assert len(base["lambdas"]) == len(other["lambdas"])
        for c1, c2 in zip(base["coefficients"], other["coefficients"]):
            assert np.max(np.abs(H.flat(c1) - H.flat(c2))) <= 1e-10


def test_truncation_and_first_model_failure():  # test_path.cpp:241-264
    rng = np.random.default_rng(79)
    design = H.make_design(rng, (5, 4, 3), [(2, 2, 2)])
    y = H.random_data(rng, "poisson", (5, 4, 3))
    lmax = O.lambda_max(design, "poisson", y)
    p = O.fit_path(design, "poisson", y, n_lambda=6, lambda_min_ratio=1e-3, maxit=1, tol=1e-14)
    assert p["truncated"] and 1 <= len(p["lambdas"]) < 6
    with pytest.raises(RuntimeError):
        O.fit_path(design, "poisson", y, lambdas=[0.5 * lmax, 0.25 * lmax], maxit=1, tol=1e-14)


def test_explicit_grids():  # test_path.cpp:266-283
    rng = np.random.default_rng(77)
    design = H.make_design(rng, (4, 3), [(2, 2)])
    y = rng.standard_normal((4, 3))
    with pytest.raises(ValueError):
        O.fit_path(design, "gaussian", y, penalty="ridge")
    assert len(O.fit_path(design, "gaussian", y, penalty="ridge", lambdas=[1.0, 0.1, 0.01])["lambdas"]) == 3
    with pytest.raises(ValueError):
        O.fit_path(design, "gaussian", y, lambdas=[0.1, 0.1])


# ------------------------------------------------------------------- bspline
def test_bspline_rows_and_counts():  # test_bspline.cpp, test_smoke.py:82-89, acceptance criterion 9
    pts = np.linspace(0.0, 7.0, 23)
    assert O.default_basis_count(len(pts), 5) == 5
    b = O.bspline_design(pts, 4, 7)
    assert b.shape == (23, 7)
    assert np.max(np.abs(b.sum(axis=1) - 1)) <= 1e-12 and b.min() >= 0
    assert [O.default_basis_count(*a) for a in ((25, 5), (977, 5), (33, 4), (81, 4), (168, 4))] == [5, 196, 9, 21, 42]
    for n, p in ((40, 10), (100, 30), (500, 120), (64, 20), (365, 60), (256, 64), (1024, 256)):
        x = O.bspline_design(np.linspace(0, 1, n), 4, p)
        assert np.max((x != 0).sum(axis=1)) <= 4
        assert np.max(np.abs(x.sum(axis=1) - 1)) <= 1e-12


def test_mse_heldout_known_answers():  # test_path.cpp:160-192
    rng = np.random.default_rng(75)
    design = H.make_design(rng, (4, 3), [(2, 2)])
    y = rng.standard_normal((4, 3))
    path = O.fit_path(design, "gaussian", y, n_lambda=5, lambda_min_ratio=0.05)
    coefs = path["coefficients"]
    with pytest.raises(ValueError):
        O.mse_heldout(design, "gaussian", coefs, y, np.zeros((4, 3)))
    mask = np.zeros(12)
    mask[[3, 7]] = 1.0
    mask = mask.reshape((4, 3), order="F")
    truth = O.h_map(design, coefs[2])  # gaussian mean = eta
    res = O.mse_heldout(design, "gaussian", coefs, truth, mask)
    assert res["mse"][2] == 0.0 and res["argmin"] == 2
    mask = np.zeros(12)
    mask[5] = 1.0
    mask = mask.reshape((4, 3), order="F")
    res = O.mse_heldout(design, "gaussian", coefs, y, mask)
    for t, c in enumerate(coefs):
        mu = O.h_map(design, c).ravel(order="F")[5]
        assert res["mse"][t] == pytest.approx((mu - y.ravel(order="F")[5]) ** 2, rel=1e-12)
    bad = mask.copy()
    bad[0, 0] = 0.5
    with pytest.raises(ValueError):
        O.mse_heldout(design, "gaussian", coefs, y, bad)
