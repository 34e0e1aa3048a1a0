"""Seeded synthetic stand-ins for the BASELINE.json configs.

The paper's neuron / taxi datasets are not available; these generators draw
inputs with the configs' shapes, factor types and value distributions.  The
same arrays feed the CUDA path and the CPU checker used by the tests.  Factors are clamped
uniform cubic B-spline bases on equispaced points of [0, 1]."""
from __future__ import annotations

import numpy as np

SEED0 = 1510032980


def _factors(n, p, bspline=None):
    if bspline is None:
        from . import kronglm as K
        bspline = K.bspline_design
    return [bspline(np.linspace(0.0, 1.0, nj), 4, pj) for nj, pj in zip(n, p)]


def tensor_h(factors, B):
    """eta = H(X, B) by successive mode products (input generation only).

    Each mode product is accumulated column by column of the factor in
    ascending order with separate elementwise multiplies and adds, over the
    rows where that column is nonzero, so the result is bit-reproducible on
    any host (no BLAS, whose kernel choice and summation order depend on the
    CPU): the parity fixtures in tests/golden/ are keyed to these bytes."""
    out = np.asarray(B, dtype=np.float64)
    for j, X in enumerate(factors):
        X = np.asarray(X, dtype=np.float64)
        src = np.moveaxis(out, j, 0)
        acc = np.zeros((X.shape[0],) + src.shape[1:])
        for k in range(X.shape[1]):
            rows = np.flatnonzero(X[:, k])
            if rows.size == 0:
                continue
            lo, hi = rows[0], rows[-1] + 1
            col = X[lo:hi, k].reshape((hi - lo,) + (1,) * (src.ndim - 1))
            acc[lo:hi] = acc[lo:hi] + col * src[k][None]
        out = np.moveaxis(acc, 0, j)
    return np.asfortranarray(out)


def _sparse_coef(rng, p, frac):
    B = np.zeros(p)
    mask = rng.random(p) < frac
    B[mask] = rng.standard_normal(int(mask.sum()))
    return B


CONFIGS = {
    "C1": dict(family="gaussian", n=(40, 40, 40), p=(10, 10, 10), n_lambda=100),
    "C2": dict(family="gaussian", n=(100, 100, 500), p=(30, 30, 120), n_lambda=50),
    "C3": dict(family="poisson", n=(64, 64, 365), p=(20, 20, 60), n_lambda=50),
    "C4": dict(family="gaussian", n=(4096, 4096), p=(256, 256), n_lambda=30),
    "C5": dict(family="poisson", n=(256, 256, 1024), p=(64, 64, 256), n_lambda=20),
}


def make(name: str, bspline=None):
    """Returns dict(design=[[X1..Xd]], y, family, n_lambda, lambda_min_ratio, meta).

    `bspline` builds the factors (default: the product's kg_bspline_design;
    the CPU-only callers -- the reference arm of bench.py and the fixture
    script -- pass their own bit-identical builder so they never load the
    product library)."""
    cfg = dict(CONFIGS[name])
    k = int(name[1])
    rng = np.random.default_rng(SEED0 + k)
    n, p = cfg["n"], cfg["p"]
    X = _factors(n, p, bspline)
    meta = {}
    if name == "C1":
        B = _sparse_coef(rng, p, 0.05)
        y = tensor_h(X, B) + rng.standard_normal(n)
    elif name == "C2":
        grids = np.meshgrid(*[np.linspace(0, 1, nj) for nj in n], indexing="ij")
        f = np.zeros(n)
        for _ in range(8):
            amp = rng.uniform(1, 3) * rng.choice([-1.0, 1.0])
            c = rng.uniform(0.1, 0.9, 3)
            w = rng.uniform(0.05, 0.25, 3)
            f += amp * np.exp(-sum(((g - ci) / wi) ** 2 for g, ci, wi in zip(grids, c, w)) / 2.0)
        y = f + rng.normal(0.0, 0.5, n)
    elif name in ("C3", "C5"):
        frac = 0.10 if name == "C3" else 0.02
        B = _sparse_coef(rng, p, frac)
        h = tensor_h(X, B)
        s = np.log(50.0) / h.max()
        eta = s * h
        y = rng.poisson(np.exp(eta)).astype(np.float64)
        meta["zero_fraction"] = float(np.mean(y == 0))
        meta["scale"] = float(s)
    elif name == "C4":
        B = _sparse_coef(rng, p, 0.02)
        y = tensor_h(X, B) + rng.standard_normal(n)
    else:
        raise KeyError(name)
    return dict(design=[X], y=np.asfortranarray(y), family=cfg["family"], n_lambda=cfg["n_lambda"],
                lambda_min_ratio=1e-4, n=n, p=p, meta=meta)
