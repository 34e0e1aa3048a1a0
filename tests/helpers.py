"""Shared test helpers: seeded random designs and an independent dense (numpy)
restatement used to check the matrix-free code (the role the reference's dense
oracle plays, proj/src/oracle.cpp:12-42 and :122-164)."""
import numpy as np


def random_design(rng, max_c=2, max_d=3, max_n=5, max_p=4):
    c = int(rng.integers(1, max_c + 1))
    d = int(rng.integers(1, max_d + 1))
    rows = [int(rng.integers(1, max_n + 1)) for _ in range(d)]
    return [[np.asfortranarray(rng.standard_normal((rows[j], int(rng.integers(1, max_p + 1)))))
             for j in range(d)] for _ in range(c)]


def make_design(rng, rows, cols):
    return [[np.asfortranarray(rng.standard_normal((n, p))) for n, p in zip(rows, comp)] for comp in cols]


def dense(design):
    mats = []
    for comp in design:
        m = comp[0]
        for x in comp[1:]:
            m = np.kron(x, m)
        mats.append(m)
    return np.hstack(mats)


def random_coef(rng, design, lo=-1.0, hi=1.0):
    return [np.asfortranarray(rng.uniform(lo, hi, size=tuple(x.shape[1] for x in comp))) for comp in design]


def flat(blocks):
    return np.concatenate([np.asarray(b).ravel(order="F") for b in blocks])


def row_dims(design):
    return tuple(x.shape[0] for x in design[0])


def soft(z, g):
    return np.sign(z) * np.maximum(np.abs(z) - g, 0.0)


def prox(z, g, penalty="lasso", alpha=0.0):
    if penalty == "lasso":
        return soft(z, g)
    if penalty == "ridge":
        return z / (1.0 + 2.0 * g)
    return soft(z, g) / (1.0 + 2.0 * alpha * g)


def dense_gaussian_minimizer(xd, v, z, lam, penalty="lasso", alpha=0.0, iters=100000):
    """Plain proximal gradient on 1/(2n)|sqrt(v)(X th - z)|^2 + lam J (independent of the solver)."""
    n = xd.shape[0]
    gram = xd.T @ (v[:, None] * xd)
    lip = np.linalg.eigvalsh(gram).max() / n
    b = xd.T @ (v * z)
    th = np.zeros(xd.shape[1])
    step = 1.0 / lip
    for _ in range(iters):
        nxt = th - step * (gram @ th - b) / n
        if lam > 0:
            nxt = prox(nxt, step * lam, penalty, alpha)
        if np.array_equal(nxt, th):
            break
        th = nxt
    return th


def dense_poisson_minimizer(xd, y, lam, a=None, iters=60000):
    """Plain PG on -l/n + lam |th|_1 with a global Lipschitz bound refreshed per iteration."""
    n = xd.shape[0]
    a = np.ones(n) if a is None else a
    th = np.zeros(xd.shape[1])
    for _ in range(iters):
        eta = xd @ th
        mu = np.exp(np.clip(eta, -30, 30))
        grad = -(xd.T @ (a * (y - mu))) / n
        lip = np.linalg.eigvalsh(xd.T @ ((a * mu)[:, None] * xd)).max() / n
        nxt = soft(th - grad / lip, lam / lip)
        if np.array_equal(nxt, th):
            break
        th = nxt
    return th


def poisson_objective(xd, y, th, lam, a=None):
    n = xd.shape[0]
    a = np.ones(n) if a is None else a
    eta = xd @ th
    ll = np.sum(a * (y * eta - np.exp(np.clip(eta, -30, 30))))
    return -ll / n + lam * np.abs(th).sum()


def random_data(rng, family, dims):
    if family == "gaussian":
        return rng.standard_normal(dims)
    if family == "binomial":
        return rng.uniform(0, 1, dims)
    if family == "poisson":
        return np.floor(rng.uniform(0, 1, dims) * 6.0)
    return 0.1 + 3.0 * rng.uniform(0, 1, dims)
