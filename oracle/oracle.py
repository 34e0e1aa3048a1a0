"""ctypes front end of the CPU oracle — TEST INFRASTRUCTURE ONLY.

Mirrors the reference's Python module surface (proj/bindings/kronglm_py.cpp:115-269:
``rho``, ``h_map``, ``g_map``, ``lambda_max``, ``fit_path``, ``bspline_design``,
``default_basis_count``, ``linear_index``) on top of ``liborc.so`` (the Eigen-free
restatement in kronglm_oracle.cpp), plus the lower-level pieces the reference's
C++ tests exercise (family maps, prox, fista_solve, outer_solve, ...).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs import
this module.  Parity status: "parity unpinned" (see kronglm_oracle.cpp).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, os.environ.get("KRONGLM_ORACLE_LIB", "liborc.so"))
_lib = None
_lock = threading.Lock()

FAMILIES = {"gaussian": 0, "binomial": 1, "poisson": 2, "gamma": 3}
PENALTIES = {"lasso": 0, "ridge": 1, "elasticnet": 2, "elastic_net": 2}
WEIGHT_MODES = {"exact": 0, "unit": 1, "one": 1, "tensor": 2, "tensor_approx": 2}
TRACE_KEYS = ["objective", "alpha", "delta_k", "lipschitz", "inner_iterations", "inner_converged", "armijo_j"]
STATUS = ["converged", "max_iterations", "line_search_failed", "inner_divergence"]

_P = C.POINTER
_d = C.c_double
_i64 = C.c_int64


class EvalError(RuntimeError):
    """Entrywise evaluation failure (family.hpp:53-61); ``cell`` is the 0-based flat index."""

    def __init__(self, msg, cell):
        super().__init__(msg)
        self.cell = cell


class DivergenceError(RuntimeError):
    pass


class PowerIterationError(RuntimeError):
    pass


class _Cfg(C.Structure):
    _fields_ = [
        ("n_lambda", _i64), ("lambda_min_ratio", _d), ("max_outer", _i64),
        ("armijo_alpha0", _d), ("armijo_b", _d), ("armijo_v", _d),
        ("armijo_max_backtracks", _i64), ("weight_mode", _i64), ("outer_tol", _d),
        ("nu", _d), ("inner_max_iters", _i64), ("inner_tol", _d),
        ("extrapolation", _i64), ("monitor_every", _i64),
    ]


def make_cfg(n_lambda=100, lambda_min_ratio=1e-4, maxit=100, alpha0=1.0, armijo_b=0.5,
             armijo_v=0.1, armijo_max_backtracks=50, iwls="exact", tol=1e-8, nu=1.0,
             inner_maxit=2000, inner_tol=1e-8, extrapolation="fista", monitor_every=1):
    return _Cfg(n_lambda, lambda_min_ratio, maxit, alpha0, armijo_b, armijo_v,
                armijo_max_backtracks, WEIGHT_MODES[iwls], tol, nu, inner_maxit, inner_tol,
                0 if extrapolation == "fista" else 1, monitor_every)


def _declare(L):
    vp, pd, pi = C.c_void_p, _P(_d), _P(_i64)
    D = [_i64, _i64, pi, pi, _P(pd)]  # c, d, n[], p[], X[]
    sig = {
        "orc_set_threads": [C.c_int],
        "orc_linear_index": [_i64, pi, pi, pi],
        "orc_rho": [_i64, _i64, pd, _i64, pi, pd, pd],
        "orc_h_map": D + [pd, pd],
        "orc_g_map": D + [pd, pd],
        "orc_xtwx_apply": D + [pd, pd, pd],
        "orc_family_map": [C.c_int, _d, _i64, pd, pd, pd, C.c_int, pd],
        "orc_loglik": [C.c_int, _d, _i64, pd, pd, pd, pd],
        "orc_validate": [C.c_int, _i64, pd, pd],
        "orc_deviance": [C.c_int, _i64, pd, pd, pd, pd],
        "orc_path_n_outer": [vp, _i64], "orc_path_trace": [vp, _i64, _i64, pd],
        "orc_penalty_value": [C.c_int, _d, _i64, pd, pd],
        "orc_prox": [C.c_int, _d, _d, _i64, pd, pd],
        "orc_lambda_max": D + [C.c_int, _d, pd, pd, C.c_int, _d, pd],
        "orc_spectral_radius": [_i64, pd, pd],
        "orc_lipschitz_upper": D + [pd, pd],
        "orc_fista_solve": D + [pd, pd, _P(pd), _d, C.c_int, _d, vp, pd, pd, pd, pd, _i64],
        "orc_outer_solve": D + [C.c_int, _d, pd, pd, _d, C.c_int, _d, vp, pd, pd, pd, pd, _i64],
        "orc_fit_path": D + [C.c_int, _d, pd, pd, C.c_int, _d, vp, pd, _i64, _P(vp)],
        "orc_path_n_models": [vp], "orc_path_lambda_max": [vp], "orc_path_truncated": [vp],
        "orc_path_model": [vp, _i64, pd], "orc_path_coef": [vp, _i64, pd], "orc_path_free": [vp],
        "orc_bspline_design": [_i64, pd, _i64, _i64, pd],
        "orc_default_basis_count": [_i64, _i64, pi],
        "orc_mse_heldout": D + [C.c_int, pd, _i64, pd, pd, pd, pi],
        "orc_bin_scatter": [_i64, _i64, pd, pd, pd, pi, pd, pi],
    }
    for name, args in sig.items():
        getattr(L, name).argtypes = args
    for name in ["orc_linear_index", "orc_rho", "orc_h_map", "orc_g_map", "orc_xtwx_apply", "orc_family_map",
                 "orc_loglik", "orc_validate", "orc_deviance", "orc_penalty_value", "orc_prox", "orc_lambda_max",
                 "orc_spectral_radius", "orc_lipschitz_upper", "orc_fista_solve", "orc_outer_solve",
                 "orc_fit_path", "orc_bspline_design", "orc_default_basis_count", "orc_mse_heldout", "orc_bin_scatter"]:
        getattr(L, name).restype = C.c_int


def build():
    """Compile liborc.so with the committed Makefile (no reference sources involved)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(_LIB_PATH):
                build()
            L = C.CDLL(_LIB_PATH)
            L.orc_last_error.restype = C.c_char_p
            L.orc_last_cell.restype = _i64
            L.orc_path_n_models.restype = _i64
            L.orc_path_lambda_max.restype = _d
            L.orc_path_truncated.restype = C.c_int
            L.orc_path_n_outer.restype = _i64
            _declare(L)
            _lib = L
    return _lib


def _check(rc):
    if rc == 0:
        return
    L = lib()
    msg = L.orc_last_error().decode()
    if rc == 1:
        raise ValueError(msg)
    if rc == 2:
        raise EvalError(msg, int(L.orc_last_cell()))
    if rc == 4:
        raise DivergenceError(msg)
    if rc == 5:
        raise PowerIterationError(msg)
    raise RuntimeError(msg)


def set_threads(t: int):
    lib().orc_set_threads(int(t))


def _f(a):
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def _ptr(a):
    return a.ctypes.data_as(_P(_d))


class _Design:
    """Flattened tensor design: components[r][j] is an n_j x p_{r,j} factor."""

    def __init__(self, design):
        comps = [[_f(x) for x in comp] for comp in design]
        if not comps or not comps[0]:
            raise ValueError("TensorDesign: need at least one component and factor")
        self.c, self.d = len(comps), len(comps[0])
        for comp in comps:
            if len(comp) != self.d:
                raise ValueError("TensorDesign: components must share the array order d")
            for x in comp:
                if x.ndim != 2:
                    raise ValueError("expected a 2-d array")
        self.comps = comps
        self.n = [comps[0][j].shape[0] for j in range(self.d)]
        self.p = [[x.shape[1] for x in comp] for comp in comps]
        self._n = (_i64 * self.d)(*self.n)
        self._p = (_i64 * (self.c * self.d))(*[q for row in self.p for q in row])
        self._X = (_P(_d) * (self.c * self.d))(*[_ptr(x) for comp in comps for x in comp])
        self.block_dims = [tuple(row) for row in self.p]
        self.p_total = int(sum(int(np.prod(b)) for b in self.block_dims))
        self.row_dims = tuple(self.n)

    def args(self):
        return (self.c, self.d, self._n, self._p, self._X)

    def blocks(self, flat):
        out, off = [], 0
        for b in self.block_dims:
            k = int(np.prod(b))
            out.append(np.asfortranarray(flat[off:off + k].reshape(b, order="F")))
            off += k
        return out

    def flat(self, coef):
        if len(coef) != self.c:
            raise ValueError("wrong number of coefficient blocks")
        parts = []
        for r, b in enumerate(coef):
            b = _f(b)
            if b.shape != self.block_dims[r]:
                raise ValueError(f"coefficient block {r} does not match the design")
            parts.append(b.ravel(order="F"))
        return np.ascontiguousarray(np.concatenate(parts))


def linear_index(multi_index, dims):
    d = len(dims)
    out = _i64()
    _check(lib().orc_linear_index(d, (_i64 * d)(*multi_index), (_i64 * d)(*dims), C.byref(out)))
    return out.value


def rho(x, a):
    x, a = _f(x), _f(a)
    if a.ndim == 0:
        a = a.reshape(1)
    ext = list(a.shape)
    out_shape = tuple(ext[1:]) + (x.shape[0],)
    out = np.zeros(int(np.prod(out_shape)))
    _check(lib().orc_rho(x.shape[0], x.shape[1], _ptr(x), len(ext), (_i64 * len(ext))(*ext), _ptr(a),
                         _ptr(out)))
    return out.reshape(out_shape, order="F")


def h_map(design, coef):
    D = _Design(design)
    th = D.flat(coef)
    eta = np.zeros(int(np.prod(D.row_dims)))
    _check(lib().orc_h_map(*D.args(), _ptr(th), _ptr(eta)))
    return eta.reshape(D.row_dims, order="F")


def mse_heldout(design, family, coefficients, y_full, heldout_mask):
    """kronglm::mse_heldout (path.cpp:91-126) over a list of coefficient sets."""
    D = _Design(design)
    flat = np.ascontiguousarray(np.stack([D.flat(c) for c in coefficients])) if coefficients else np.zeros((0, D.p_total))
    y = _f(y_full).ravel(order="F")
    m = _f(heldout_mask).ravel(order="F")
    out = np.zeros(max(len(coefficients), 1))
    arg = C.c_int64()
    _check(lib().orc_mse_heldout(*D.args(), FAMILIES[family], _ptr(flat), len(coefficients), _ptr(y), _ptr(m),
                                 _ptr(out), C.byref(arg)))
    return {"mse": [float(v) for v in out[:len(coefficients)]], "argmin": int(arg.value)}


def g_map(design, u):
    D = _Design(design)
    u = _f(u)
    if u.shape != D.row_dims:
        raise ValueError("g_map: array dimensions do not match")
    out = np.zeros(D.p_total)
    _check(lib().orc_g_map(*D.args(), _ptr(u), _ptr(out)))
    return D.blocks(out)


def xtwx_apply(design, v, coef):
    D = _Design(design)
    v = _f(v)
    th = D.flat(coef)
    out = np.zeros(D.p_total)
    _check(lib().orc_xtwx_apply(*D.args(), _ptr(v), _ptr(th), _ptr(out)))
    return D.blocks(out)


def _family_map(what, family, eta, y=None, a=None, dispersion=1.0):
    eta = np.ascontiguousarray(np.asarray(eta, dtype=np.float64).ravel(order="F"))
    n = eta.size
    y = np.zeros(n) if y is None else np.ascontiguousarray(np.asarray(y, np.float64).ravel(order="F"))
    a = np.ones(n) if a is None else np.ascontiguousarray(np.asarray(a, np.float64).ravel(order="F"))
    out = np.zeros(n)
    _check(lib().orc_family_map(FAMILIES[family], _d(dispersion), n, _ptr(y), _ptr(a), _ptr(eta), what,
                                _ptr(out)))
    return out


def mean(family, eta, dispersion=1.0):
    return _family_map(0, family, eta, dispersion=dispersion)


def score(family, y, eta, a=None, dispersion=1.0):
    return _family_map(1, family, eta, y, a, dispersion)


def glm_weights(family, eta, dispersion=1.0):
    return _family_map(2, family, eta, dispersion=dispersion)


def working_response(family, y, eta, a=None, dispersion=1.0):
    return _family_map(3, family, eta, y, a, dispersion)


def loglik(family, y, eta, a=None, dispersion=1.0):
    eta = np.ascontiguousarray(np.asarray(eta, np.float64).ravel(order="F"))
    n = eta.size
    y = np.ascontiguousarray(np.asarray(y, np.float64).ravel(order="F"))
    a = np.ones(n) if a is None else np.ascontiguousarray(np.asarray(a, np.float64).ravel(order="F"))
    out = _d()
    _check(lib().orc_loglik(FAMILIES[family], _d(dispersion), n, _ptr(y), _ptr(a), _ptr(eta), C.byref(out)))
    return out.value


def deviance(family, y, eta, a=None):
    """Deviance from eta (SURVEY 8(d) parity protocol; family.cpp conventions)."""
    eta = np.ascontiguousarray(np.asarray(eta, np.float64).ravel(order="F"))
    n = eta.size
    y = np.ascontiguousarray(np.asarray(y, np.float64).ravel(order="F"))
    a = np.ones(n) if a is None else np.ascontiguousarray(np.asarray(a, np.float64).ravel(order="F"))
    out = _d()
    _check(lib().orc_deviance(FAMILIES[family], n, _ptr(y), _ptr(a), _ptr(eta), C.byref(out)))
    return out.value


def validate(family, y, a=None):
    y = np.ascontiguousarray(np.asarray(y, np.float64).ravel(order="F"))
    a = np.ones(y.size) if a is None else np.ascontiguousarray(np.asarray(a, np.float64).ravel(order="F"))
    _check(lib().orc_validate(FAMILIES[family], y.size, _ptr(y), _ptr(a)))


def penalty_value(theta, penalty="lasso", alpha=0.0):
    th = np.ascontiguousarray(np.asarray(theta, np.float64).ravel())
    out = _d()
    _check(lib().orc_penalty_value(PENALTIES[penalty], _d(alpha), th.size, _ptr(th), C.byref(out)))
    return out.value


def prox(z, gamma, penalty="lasso", alpha=0.0):
    z = np.ascontiguousarray(np.asarray(z, np.float64).ravel())
    out = np.zeros_like(z)
    _check(lib().orc_prox(PENALTIES[penalty], _d(alpha), _d(gamma), z.size, _ptr(z), _ptr(out)))
    return out


def _data(D, y, weights):
    y = _f(y)
    if y.shape != D.row_dims:
        raise ValueError("data dims do not match the design")
    a = None if weights is None else _f(weights)
    return y, a


def lambda_max(design, family, y, weights=None, penalty="lasso", alpha=0.0, dispersion=1.0):
    D = _Design(design)
    y, a = _data(D, y, weights)
    out = _d()
    _check(lib().orc_lambda_max(*D.args(), FAMILIES[family], _d(dispersion), _ptr(y),
                                _ptr(a) if a is not None else None, PENALTIES[penalty], _d(alpha),
                                C.byref(out)))
    return out.value


def spectral_radius(A):
    A = _f(A)
    out = _d()
    _check(lib().orc_spectral_radius(A.shape[0], _ptr(A), C.byref(out)))
    return out.value


def lipschitz_upper(design, v):
    D = _Design(design)
    v = _f(v)
    out = _d()
    _check(lib().orc_lipschitz_upper(*D.args(), _ptr(v), C.byref(out)))
    return out.value


def fista_solve(design, v, z, lam, penalty="lasso", alpha=0.0, init=None, tensor_weights=None,
                record_history=False, **cfg):
    D = _Design(design)
    v, z = _f(v), _f(z)
    th0 = np.zeros(D.p_total) if init is None else D.flat(init)
    c = make_cfg(**cfg)
    out = np.zeros(D.p_total)
    info = np.zeros(6)
    tw = None
    if tensor_weights is not None:
        tws = [np.ascontiguousarray(np.asarray(w, np.float64)) for w in tensor_weights]
        tw = (_P(_d) * len(tws))(*[_ptr(w) for w in tws])
    cap = int(c.inner_max_iters) + 2 if record_history else 0
    hist = np.zeros(2 * cap) if record_history else None
    _check(lib().orc_fista_solve(*D.args(), _ptr(v), _ptr(z), tw, _d(lam), PENALTIES[penalty], _d(alpha),
                                 C.byref(c), _ptr(th0), _ptr(out), _ptr(info),
                                 _ptr(hist) if hist is not None else None, cap))
    res = {"coef": D.blocks(out), "coef_flat": out, "objective": info[0], "iterations": int(info[1]),
           "converged": bool(info[2]), "backtracks": int(info[3]), "lipschitz": info[4]}
    if record_history:
        k = int(info[5])
        res["history"] = [(int(hist[2 * i]), hist[2 * i + 1]) for i in range(k)]
    return res


def outer_solve(design, family, y, lam, weights=None, penalty="lasso", alpha=0.0, init=None,
                dispersion=1.0, **cfg):
    D = _Design(design)
    y, a = _data(D, y, weights)
    th0 = np.zeros(D.p_total) if init is None else D.flat(init)
    c = make_cfg(**cfg)
    out = np.zeros(D.p_total)
    info = np.zeros(5)
    cap = int(c.max_outer) + 1
    rec = np.zeros(7 * cap)
    _check(lib().orc_outer_solve(*D.args(), FAMILIES[family], _d(dispersion), _ptr(y),
                                 _ptr(a) if a is not None else None, _d(lam), PENALTIES[penalty], _d(alpha),
                                 C.byref(c), _ptr(th0), _ptr(out), _ptr(info), _ptr(rec), cap))
    k = int(info[1])
    recs = [dict(zip(["objective", "alpha", "delta_k", "lipschitz", "inner_iterations", "inner_converged",
                      "armijo_j"], rec[7 * i:7 * i + 7])) for i in range(k)]
    return {"coef": D.blocks(out), "coef_flat": out, "status": STATUS[int(info[0])], "iterations": recs,
            "weight_evaluations": int(info[2]), "initial_objective": info[3], "final_objective": info[4]}


def fit_path(design, family, y, weights=None, penalty="lasso", alpha=0.0, n_lambda=100,
             lambda_min_ratio=1e-4, lambdas=None, iwls="exact", nu=1.0, tol=1e-8, maxit=100,
             inner_tol=1e-8, inner_maxit=2000, dispersion=1.0, monitor_every=1):
    """Same signature and result keys as kronglm.fit_path (kronglm_py.cpp:159-217), plus
    per-model ``inner_iters`` and ``status`` diagnostics."""
    D = _Design(design)
    y, a = _data(D, y, weights)
    c = make_cfg(n_lambda=n_lambda, lambda_min_ratio=lambda_min_ratio, maxit=maxit, iwls=iwls, tol=tol,
                 nu=nu, inner_maxit=inner_maxit, inner_tol=inner_tol, monitor_every=monitor_every)
    if penalty not in PENALTIES:
        raise ValueError("unknown penalty: " + penalty)
    if family not in FAMILIES:
        raise ValueError("unknown family: " + family)
    lam = None if lambdas is None else np.ascontiguousarray(np.asarray(lambdas, np.float64))
    h = C.c_void_p()
    L = lib()
    _check(L.orc_fit_path(*D.args(), FAMILIES[family], _d(dispersion), _ptr(y),
                          _ptr(a) if a is not None else None, PENALTIES[penalty], _d(alpha), C.byref(c),
                          _ptr(lam) if lam is not None else None, 0 if lam is None else lam.size,
                          C.byref(h)))
    try:
        m = L.orc_path_n_models(h)
        info = np.zeros(6)
        out = {"lambdas": [], "objectives": [], "lambda_max": L.orc_path_lambda_max(h),
               "truncated": bool(L.orc_path_truncated(h)), "coefficients": [], "nonzero": [],
               "outer_iters": [], "converged": [], "inner_iters": [], "status": [], "traces": []}
        for t in range(m):
            L.orc_path_model(h, _i64(t), _ptr(info))
            flat = np.zeros(D.p_total)
            L.orc_path_coef(h, _i64(t), _ptr(flat))
            out["lambdas"].append(info[0])
            out["objectives"].append(info[1])
            out["outer_iters"].append(int(info[2]))
            out["inner_iters"].append(int(info[3]))
            out["status"].append(STATUS[int(info[4])])
            out["converged"].append(bool(info[5]))
            out["coefficients"].append(D.blocks(flat))
            out["nonzero"].append(int(np.count_nonzero(flat)))
            rec = np.zeros(7)
            tr = []
            for k in range(L.orc_path_n_outer(h, _i64(t))):
                L.orc_path_trace(h, _i64(t), _i64(k), _ptr(rec))
                tr.append(dict(zip(TRACE_KEYS, [float(rec[0]), float(rec[1]), float(rec[2]), float(rec[3]),
                                                int(rec[4]), bool(rec[5]), int(rec[6])])))
            out["traces"].append(tr)
        return out
    finally:
        L.orc_path_free(h)


def bspline_design(points, order=4, n_basis=0):
    pts = np.ascontiguousarray(np.asarray(points, np.float64))
    out = np.zeros((pts.size, n_basis), order="F")
    _check(lib().orc_bspline_design(pts.size, _ptr(pts), order, n_basis, _ptr(out)))
    return out


def bin_scatter(points, bounds, bins):
    """bin_scatter (bspline.cpp:106-153): (counts array, dropped)."""
    pts = np.ascontiguousarray(np.asarray(points, np.float64))
    bins = [int(b) for b in bins]
    d = len(bins)
    if d == 0 or len(bounds) != d:
        raise ValueError("bin_scatter: bounds and bins must agree on the dimension")
    pts = pts.reshape(-1, d) if pts.size else np.zeros((0, d))
    lo = np.array([float(b[0]) for b in bounds])
    hi = np.array([float(b[1]) for b in bounds])
    bn = np.array(bins, dtype=np.int64)
    counts = np.zeros(int(np.prod(bins)))
    drop = _i64()
    _check(lib().orc_bin_scatter(pts.shape[0], d, _ptr(pts), _ptr(lo), _ptr(hi),
                                 bn.ctypes.data_as(_P(_i64)), _ptr(counts), C.byref(drop)))
    return counts.reshape(bins, order="F"), drop.value


def default_basis_count(n_points, ratio):
    out = _i64()
    _check(lib().orc_default_basis_count(n_points, ratio, C.byref(out)))
    return out.value
