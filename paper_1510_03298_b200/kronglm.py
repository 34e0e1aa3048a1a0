"""Drop-in Python surface of the reference ``kronglm`` module on the B200 path.

Same names, arguments, defaults, result keys and error types as the
reference's pybind11 module (proj/bindings/kronglm_py.cpp:115-269):
``linear_index``, ``rho``, ``h_map``, ``g_map``, ``lambda_max``,
``fit_path``, ``predict``, ``bspline_design``, ``default_basis_count``.
Arrays cross the boundary as Fortran-order float64 numpy arrays; every
computation runs in libkronglm_b200.so on the GPU (no CPU fallback).

Lower-level handles (:class:`Context`, :class:`Design`, :class:`Observation`,
:func:`fit_path_resident`) expose the resident-HBM workflow the bench uses:
upload once, fit many paths.
"""
from __future__ import annotations

import ctypes as C
import threading
import weakref

import numpy as np

from . import _lib
from ._lib import EvalError, InvalidArgument, KgError, PathCfg  # noqa: F401

FAMILIES = {"gaussian": 0, "binomial": 1, "poisson": 2, "gamma": 3}
PENALTIES = {"lasso": 0, "ridge": 1, "elasticnet": 2, "elastic_net": 2}
WEIGHT_MODES = {"exact": 0, "unit": 1, "one": 1, "tensor": 2, "tensor_approx": 2}
STATUS = ["converged", "max_iterations", "line_search_failed", "inner_divergence"]

_pd = C.POINTER(C.c_double)
_i64 = C.c_int64
_pi = C.POINTER(_i64)


def _f(a):
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def _ptr(a):
    return a.ctypes.data_as(_pd)


# ------------------------------------------------------------------ handles
class Context:
    """One CUDA device + stream (kg_ctx)."""

    def __init__(self, device: int = 0, _handle=None, rank: int = 0, world: int = 1):
        L = _lib.load()
        h = _handle
        if h is None:
            h = C.c_void_p()
            _lib.check(L.kg_ctx_create(int(device), C.byref(h)))
        self.h = h
        self.device = device
        self.rank, self.world = int(rank), int(world)
        self._children = weakref.WeakSet()  # designs / observations / results on this context

    @classmethod
    def sharded(cls, device: int, rank: int, world: int, unique_id: bytes | None):
        """Last-mode sharded context (kg_ctx_create_sharded): rank `rank` of
        `world` owns slab rank of the last observation mode; `unique_id` is
        nccl_unique_id() from rank 0 broadcast to every rank (None: local
        partials only, no communicator)."""
        h = C.c_void_p()
        buf = None
        if unique_id is not None:
            if len(unique_id) != 128:
                raise ValueError("nccl unique id must be 128 bytes")
            buf = C.create_string_buffer(bytes(unique_id), 128)
        _lib.check(_lib.load().kg_ctx_create_sharded(int(device), int(rank), int(world), buf, C.byref(h)))
        return cls(device, _handle=h, rank=rank, world=world)

    def close(self):
        if getattr(self, "h", None):
            for ch in list(getattr(self, "_children", ())):  # the C objects must go before their context
                ch.close()
            _lib.load().kg_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def check(self, st):
        _lib.check(st, self.h)

    @property
    def stream(self) -> int:
        return _lib.load().kg_ctx_stream(self.h)

    def synchronize(self):
        self.check(_lib.load().kg_ctx_synchronize(self.h))

    @property
    def launches(self) -> int:
        return int(_lib.load().kg_launch_count(self.h))

    def reset_launches(self):
        _lib.load().kg_launch_count_reset(self.h)


_ctx_local = threading.local()


def nccl_unique_id() -> bytes:
    """128-byte ncclUniqueId for Context.sharded (made on rank 0, broadcast by the caller)."""
    buf = C.create_string_buffer(128)
    _lib.check(_lib.load().kg_nccl_unique_id(buf))
    return buf.raw


def shard_rows(n_last: int, rank: int, world: int) -> tuple[int, int]:
    """Rows [lo, hi) of the last mode owned by `rank` (kg_design_create's split)."""
    return n_last * rank // world, n_last * (rank + 1) // world


def default_context(device: int = 0) -> Context:
    ctxs = getattr(_ctx_local, "ctxs", None)
    if ctxs is None:
        ctxs = _ctx_local.ctxs = {}
    if device not in ctxs:
        ctxs[device] = Context(device)
    return ctxs[device]


class Design:
    """TensorDesign: components[r][j] is the n_j x p_{r,j} factor (design.hpp:13-45)."""

    def __init__(self, components, ctx: Context | None = None):
        self.ctx = ctx or default_context()
        comps = [[_f(x) for x in comp] for comp in components]
        if not comps or not comps[0]:
            raise ValueError("TensorDesign: need at least one component and one marginal factor")
        self.c, self.d = len(comps), len(comps[0])
        for comp in comps:
            if len(comp) != self.d:
                raise ValueError("TensorDesign: components must share the array order d")
            for x in comp:
                if x.ndim != 2:
                    raise ValueError("expected a 2-d array")
        rows = [comps[0][j].shape[0] for j in range(self.d)]
        for comp in comps:
            if [x.shape[0] for x in comp] != rows:
                raise ValueError("TensorDesign: factor row counts differ across components")
        self.row_dims = tuple(rows)
        lo, hi = shard_rows(rows[-1], self.ctx.rank, self.ctx.world)
        self.local_row_dims = tuple(rows[:-1]) + (hi - lo,)  # this rank's slab (= row_dims unsharded)
        self.block_dims = [tuple(x.shape[1] for x in comp) for comp in comps]
        self.p = int(sum(int(np.prod(b)) for b in self.block_dims))
        self.n = int(np.prod(rows))
        n_arr = (_i64 * self.d)(*rows)
        p_arr = (_i64 * (self.c * self.d))(*[q for b in self.block_dims for q in b])
        X = (_pd * (self.c * self.d))(*[_ptr(x) for comp in comps for x in comp])
        h = C.c_void_p()
        self.ctx.check(_lib.load().kg_design_create(self.ctx.h, self.c, self.d, n_arr, p_arr, X, C.byref(h)))
        self.h = h
        self.ctx._children.add(self)

    def close(self):
        if getattr(self, "h", None):
            _lib.load().kg_design_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def spectral(self, r, j):
        out = C.c_double()
        self.ctx.check(_lib.load().kg_design_spectral(self.h, r, j, C.byref(out)))
        return out.value

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

    def blocks(self, flat):
        out, off = [], 0
        for b in self.block_dims:
            k = int(np.prod(b))
            out.append(np.asfortranarray(flat[off:off + k].reshape(b, order="F")))
            off += k
        return out


class Observation:
    """ObservationData(y[, a]) resident in HBM (family.hpp:40-47).

    ``y``/``weights`` are numpy arrays (uploaded) or objects exposing
    ``data_ptr()`` (e.g. CUDA torch tensors; copied device to device)."""

    def __init__(self, design: Design, y, weights=None):
        self.design = design
        self.ctx = design.ctx
        L = _lib.load()
        h = C.c_void_p()
        if hasattr(y, "data_ptr"):
            yp = C.c_void_p(y.data_ptr())
            ap = C.c_void_p(weights.data_ptr()) if weights is not None else None
            self.ctx.check(L.kg_obs_create(self.ctx.h, design.h, yp, ap, 1, C.byref(h)))
        else:
            y = _f(y)
            if y.shape != design.local_row_dims:
                raise ValueError("data dims do not match the design")
            a = None
            if weights is not None:
                a = _f(weights)
                if a.shape != design.local_row_dims:
                    raise ValueError("ObservationData: response and weight dims differ")
            self.ctx.check(L.kg_obs_create(self.ctx.h, design.h, y.ctypes.data_as(C.c_void_p),
                                           a.ctypes.data_as(C.c_void_p) if a is not None else None, 0,
                                           C.byref(h)))
        self.h = h
        self.ctx._children.add(self)

    def close(self):
        if getattr(self, "h", None):
            _lib.load().kg_obs_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def make_cfg(n_lambda=100, lambda_min_ratio=1e-4, iwls="exact", nu=1.0, tol=1e-8, maxit=100, inner_tol=1e-8,
             inner_maxit=2000, monitor_every=1, extrapolation="fista", armijo_alpha0=1.0, armijo_b=0.5,
             armijo_v=0.1, armijo_max_backtracks=50):
    if iwls not in WEIGHT_MODES:
        raise ValueError("unknown weight mode: " + str(iwls))
    cfg = PathCfg()
    _lib.load().kg_path_cfg_default(C.byref(cfg))
    cfg.n_lambda = int(n_lambda)
    cfg.lambda_min_ratio = float(lambda_min_ratio)
    cfg.weight_mode = WEIGHT_MODES[iwls]
    cfg.nu = float(nu)
    cfg.outer_tol = float(tol)
    cfg.max_outer = int(maxit)
    cfg.inner_tol = float(inner_tol)
    cfg.inner_max_iters = int(inner_maxit)
    cfg.monitor_every = int(monitor_every)
    cfg.extrapolation = 0 if extrapolation == "fista" else 1
    cfg.armijo_alpha0 = float(armijo_alpha0)
    cfg.armijo_b = float(armijo_b)
    cfg.armijo_v = float(armijo_v)
    cfg.armijo_max_backtracks = int(armijo_max_backtracks)
    return cfg


class PathResult:
    """FitPath (path.hpp:18-27); coefficients stay in HBM until read."""

    def __init__(self, design: Design, h):
        self.design = design
        self.h = h
        design.ctx._children.add(self)
        L = _lib.load()
        self.n_models = int(L.kg_result_n_models(h))
        self.truncated = bool(L.kg_result_truncated(h))
        self.lambda_max = float(L.kg_result_lambda_max(h))
        self.lambdas = [L.kg_result_lambda(h, t) for t in range(self.n_models)]
        self.objectives = [L.kg_result_objective(h, t) for t in range(self.n_models)]
        self.outer_iters = [int(L.kg_result_outer_iters(h, t)) for t in range(self.n_models)]
        self.inner_iters = [int(L.kg_result_inner_iters(h, t)) for t in range(self.n_models)]
        self.status = [STATUS[L.kg_result_status(h, t)] for t in range(self.n_models)]
        self.initial_objectives = [L.kg_result_initial_objective(h, t) for t in range(self.n_models)]
        self.traces = [self._trace(L, t) for t in range(self.n_models)]

    def _trace(self, L, t):
        """OuterTrace records of model t (outer.hpp:26-47; FitPath::diagnostics, path.hpp:23)."""
        k = int(L.kg_result_n_outer(self.h, t))
        recs = (_lib.OuterRecord * max(k, 1))()
        if k > 0 and L.kg_result_trace(self.h, t, recs) != 0:
            raise RuntimeError("kg_result_trace failed")
        return [{"objective": r.objective, "alpha": r.alpha, "delta_k": r.delta_k, "lipschitz": r.lipschitz,
                 "inner_iterations": int(r.inner_iterations), "inner_converged": bool(r.inner_converged),
                 "armijo_j": int(r.armijo_j)} for r in recs[:k]]

    def deviance(self, obs: "Observation", family: str) -> list:
        """Deviance of every model against ``obs`` (family.cpp conventions),
        eta = H(theta_t) and the sum computed on the device."""
        if family not in FAMILIES:
            raise ValueError("unknown family: " + str(family))
        out = np.zeros(max(self.n_models, 1))
        D = self.design
        D.ctx.check(_lib.load().kg_result_deviance(D.ctx.h, D.h, obs.h, self.h, FAMILIES[family], _ptr(out)))
        return [float(v) for v in out[:self.n_models]]

    def coef(self, t) -> np.ndarray:
        out = np.zeros(self.design.p)
        self.design.ctx.check(_lib.load().kg_result_coef(self.h, t, _ptr(out)))
        return out

    def coefs(self, out=None) -> np.ndarray:
        """All models' coefficients, n_models x p, in one device-to-host copy
        (into ``out[:n_models]`` when given: C-contiguous float64, >= n_models rows)."""
        if out is None:
            out = np.zeros((self.n_models, self.design.p))
        else:
            if (out.dtype != np.float64 or not out.flags.c_contiguous or out.ndim != 2
                    or out.shape[1] != self.design.p or out.shape[0] < self.n_models):
                raise ValueError("coefs: out must be a C-contiguous float64 (>= n_models, p) array")
            out = out[:self.n_models]
        if self.n_models:
            self.design.ctx.check(_lib.load().kg_result_coefs(self.h, 0, self.n_models, _ptr(out)))
        return out

    def nonzeros(self) -> list:
        """Nonzero count of every model's coefficients, counted on the device."""
        if not self.n_models:
            return []
        out = (_i64 * self.n_models)()
        self.design.ctx.check(_lib.load().kg_result_nonzeros(self.h, out))
        return [int(v) for v in out]

    def close(self):
        if getattr(self, "h", None):
            _lib.load().kg_result_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def fit_path_resident(design: Design, obs: Observation, family="gaussian", penalty="lasso", alpha=0.0,
                      lambdas=None, dispersion=1.0, **cfg) -> PathResult:
    if family not in FAMILIES:
        raise ValueError("unknown family: " + str(family))
    if penalty not in PENALTIES:
        raise ValueError("unknown penalty: " + str(penalty))
    c = make_cfg(**cfg)
    lam = None
    if lambdas is not None:
        lam = np.ascontiguousarray(np.asarray(lambdas, dtype=np.float64))
    h = C.c_void_p()
    design.ctx.check(_lib.load().kg_fit_path(design.ctx.h, design.h, obs.h, FAMILIES[family], float(dispersion),
                                             PENALTIES[penalty], float(alpha), C.byref(c),
                                             _ptr(lam) if lam is not None else None,
                                             0 if lam is None else lam.size, C.byref(h)))
    return PathResult(design, h)


def outer_solve(design, family, y, lam, weights=None, penalty="lasso", alpha=0.0, dispersion=1.0, **cfg):
    """kronglm::outer_solve (outer.hpp:56-60) at one lambda from theta = 0.
    Returns {"coef", "coef_flat", "status", "iterations" (OuterTrace records),
    "initial_objective", "final_objective"} like the C++ OuterResult."""
    if family not in FAMILIES:
        raise ValueError("unknown family: " + str(family))
    if penalty not in PENALTIES:
        raise ValueError("unknown penalty: " + str(penalty))
    D = _design(design)
    obs = Observation(D, y, weights)
    c = make_cfg(**cfg)
    h = C.c_void_p()
    D.ctx.check(_lib.load().kg_outer_solve(D.ctx.h, D.h, obs.h, FAMILIES[family], float(dispersion),
                                           PENALTIES[penalty], float(alpha), C.byref(c), float(lam), C.byref(h)))
    res = PathResult(D, h)
    flat = res.coef(0)
    out = {"coef": D.blocks(flat), "coef_flat": flat, "status": res.status[0], "iterations": res.traces[0],
           "initial_objective": res.initial_objectives[0], "final_objective": res.objectives[0]}
    res.close()
    return out


# ----------------------------------------------- reference module surface
def linear_index(multi_index, dims):
    """Column-major 1-based linear position (array.cpp:22-36)."""
    d = len(dims)
    if len(multi_index) != d:
        raise ValueError("linear_index: index arity does not match dims")
    r = _lib.load().kg_linear_index(d, (_i64 * d)(*multi_index), (_i64 * d)(*dims))
    if r < 0:
        raise ValueError("linear_index: index out of range")
    return int(r)


def rho(x, a):
    """Rotated contraction of a matrix against the first array dimension (array.cpp:51-72)."""
    x, a = _f(x), _f(a)
    if x.ndim != 2:
        raise ValueError("expected a 2-d array")
    if a.shape[0] != x.shape[1]:
        raise ValueError(f"rho: matrix has {x.shape[1]} columns but array's first extent is {a.shape[0]}")
    ctx = default_context()
    ext = list(a.shape)
    out_shape = tuple(ext[1:]) + (x.shape[0],)
    out = np.zeros(int(np.prod(out_shape)))
    ctx.check(_lib.load().kg_rho(ctx.h, x.shape[0], _ptr(x), len(ext), (_i64 * len(ext))(*ext), _ptr(a),
                                 _ptr(out)))
    return out.reshape(out_shape, order="F")


def _design(design):
    return design if isinstance(design, Design) else Design(design)


def h_map(design, coef):
    """Linear predictor array, vec = X theta (design.cpp:89-102)."""
    D = _design(design)
    th = D.flat(coef)
    eta = np.zeros(int(np.prod(D.local_row_dims)))
    D.ctx.check(_lib.load().kg_h_map(D.ctx.h, D.h, _ptr(th), _ptr(eta)))
    return eta.reshape(D.local_row_dims, order="F")


def g_map(design, u):
    """Adjoint of h_map, vec = X^T vec(u) (design.cpp:104-116)."""
    D = _design(design)
    u = _f(u)
    if u.shape != D.local_row_dims:
        raise ValueError("g_map: array dimensions do not match")
    out = np.zeros(D.p)
    D.ctx.check(_lib.load().kg_g_map(D.ctx.h, D.h, _ptr(u), _ptr(out)))
    return D.blocks(out)


def xtwx_apply(design, v, coef):
    """X^T diag(v) X theta (design.cpp:118-124)."""
    D = _design(design)
    v = _f(v)
    th = D.flat(coef)
    out = np.zeros(D.p)
    D.ctx.check(_lib.load().kg_xtwx_apply(D.ctx.h, D.h, _ptr(v), _ptr(th), _ptr(out)))
    return D.blocks(out)


def lambda_max(design, family, y, weights=None):
    """Smallest penalty level with an all-zero solution (penalty.cpp:72-85)."""
    if family not in FAMILIES:
        raise ValueError("unknown family: " + str(family))
    D = _design(design)
    obs = Observation(D, y, weights)
    out = C.c_double()
    D.ctx.check(_lib.load().kg_lambda_max(D.ctx.h, D.h, obs.h, FAMILIES[family], 1.0, 0, 0.0, C.byref(out)))
    return out.value


class _PinnedBlock:
    """One page-locked host block (kg_host_alloc).  Arrays handed out over it
    keep it alive through their ``base`` chain; when the last one dies the
    block returns to a small free list instead of being unpinned, so repeated
    fits reuse it (pinning costs far more than the download it speeds up)."""
    _free: list = []
    _lock = threading.Lock()
    _keep = 4  # cached blocks

    def __init__(self, nbytes):
        self.nbytes = nbytes
        ptr = C.c_void_p()
        if _lib.load().kg_host_alloc(nbytes, C.byref(ptr)) != 0:
            raise MemoryError("kg_host_alloc(%d) failed" % nbytes)
        self.ptr = ptr.value

    @classmethod
    def take(cls, nbytes):
        with cls._lock:
            for i, b in enumerate(cls._free):
                if b.nbytes >= nbytes:
                    return cls._free.pop(i)
        return cls(nbytes)

    def array(self, shape):
        n = int(np.prod(shape))
        raw = (C.c_double * n).from_address(self.ptr)
        raw._block = self  # the ndarray's base keeps the block alive
        return np.frombuffer(raw, dtype=np.float64).reshape(shape)

    def __del__(self):
        try:
            with _PinnedBlock._lock:
                if len(_PinnedBlock._free) < _PinnedBlock._keep:
                    # resurrect into the free list (re-collected only when evicted)
                    _PinnedBlock._free.append(_PinnedBlock._clone(self))
                    return
            _lib.load().kg_host_free(self.ptr)
        except Exception:
            pass

    @classmethod
    def _clone(cls, b):
        c = cls.__new__(cls)
        c.nbytes, c.ptr = b.nbytes, b.ptr
        return c


def fit_path(design, family, y, weights=None, penalty="lasso", alpha=0.0, n_lambda=100, lambda_min_ratio=1e-4,
             lambdas=None, iwls="exact", nu=1.0, tol=1e-8, maxit=100, inner_tol=1e-8, inner_maxit=2000):
    """Warm-started regularization path (path.cpp:29-81); same kwargs and result
    keys as kronglm_py.cpp:159-217, plus ``inner_iters`` and ``status``."""
    D = _design(design)
    obs = Observation(D, y, weights)
    # The coefficients land in a page-locked block (one PCIe-speed copy, no
    # pageable staging); the returned arrays are views into it.
    n_max = len(lambdas) if lambdas is not None else int(n_lambda)
    shape = (max(n_max, 1), D.p)
    buf = _PinnedBlock.take(8 * shape[0] * shape[1]).array(shape)
    res = fit_path_resident(D, obs, family, penalty, alpha, lambdas, n_lambda=n_lambda,
                            lambda_min_ratio=lambda_min_ratio, iwls=iwls, nu=nu, tol=tol, maxit=maxit,
                            inner_tol=inner_tol, inner_maxit=inner_maxit)
    out = {"lambdas": list(res.lambdas), "objectives": list(res.objectives), "lambda_max": res.lambda_max,
           "truncated": res.truncated, "coefficients": [], "nonzero": [], "outer_iters": list(res.outer_iters),
           "converged": [s == "converged" for s in res.status], "inner_iters": list(res.inner_iters),
           "status": list(res.status), "traces": res.traces}
    for flat in res.coefs(out=buf):
        out["coefficients"].append(D.blocks(flat))
    out["nonzero"] = res.nonzeros()
    return out


def mse_heldout(path, family, y_full, heldout_mask):
    """Held-out sum of squared errors per model and the minimizing index
    (kronglm::mse_heldout, path.cpp:91-126), from a PathResult (the
    coefficients stay on the device).  Returns {"mse": [...], "argmin": t}."""
    if family not in FAMILIES:
        raise ValueError("unknown family: " + str(family))
    D = path.design
    y = _f(y_full)
    m = _f(heldout_mask)
    if y.shape != D.local_row_dims or m.shape != D.local_row_dims:
        raise ValueError("mse_heldout: array dims do not match the design")
    out = np.zeros(max(path.n_models, 1))
    arg = _i64()
    D.ctx.check(_lib.load().kg_mse_heldout(D.ctx.h, D.h, path.h, FAMILIES[family], _ptr(y), _ptr(m), _ptr(out),
                                           C.byref(arg)))
    return {"mse": [float(v) for v in out[:path.n_models]], "argmin": int(arg.value)}


def predict(design, family, coef):
    """Linear predictor and fitted mean arrays (path.cpp:83-89)."""
    if family not in FAMILIES:
        raise ValueError("unknown family: " + str(family))
    D = _design(design)
    th = D.flat(coef)
    eta = np.zeros(int(np.prod(D.local_row_dims)))
    mu = np.zeros(eta.size)
    D.ctx.check(_lib.load().kg_predict(D.ctx.h, D.h, FAMILIES[family], _ptr(th), _ptr(eta), _ptr(mu)))
    return eta.reshape(D.local_row_dims, order="F"), mu.reshape(D.local_row_dims, order="F")


def bspline_design(points, order=4, n_basis=0):
    """Marginal B-spline design on a clamped uniform knot vector (bspline.cpp:64-104)."""
    pts = np.ascontiguousarray(np.asarray(points, dtype=np.float64))
    out = np.zeros((pts.size, int(n_basis)), order="F")
    st = _lib.load().kg_bspline_design(pts.size, _ptr(pts), int(order), int(n_basis), _ptr(out))
    if st != 0:
        raise ValueError("bspline_design: invalid grid or basis specification")
    return out


class BinnedCounts(tuple):
    """BinnedCounts (bspline.hpp:33-36): ``counts`` array and ``dropped``."""
    __slots__ = ()

    def __new__(cls, counts, dropped):
        return tuple.__new__(cls, (counts, dropped))

    counts = property(lambda self: self[0])
    dropped = property(lambda self: self[1])


def _bin_args(bounds, bins):
    bins = [int(b) for b in bins]
    d = len(bins)
    if d == 0 or len(bounds) != d:
        raise ValueError("bin_scatter: bounds and bins must agree on the dimension")
    lo = np.array([float(b[0]) for b in bounds])
    hi = np.array([float(b[1]) for b in bounds])
    return bins, d, lo, hi, np.array(bins, dtype=np.int64)


def bin_scatter(points, bounds, bins, ctx: Context | None = None, out=None) -> BinnedCounts:
    """Count points on a regular grid (bspline.cpp:106-153), on the device.

    ``points``: (npts, d) array -- numpy (uploaded) or a CUDA tensor exposing
    ``data_ptr()`` (row-major float64, read in place).  ``bounds``: d pairs
    (lo, hi); ``bins``: d bin counts.  Returns BinnedCounts(counts, dropped),
    counts shaped ``bins`` in column-major order.  For device points the
    counts land in ``out`` (a CUDA float64 buffer of prod(bins) elements, e.g.
    to feed ``Observation``) and ``counts`` is that buffer."""
    ctx = ctx or default_context()
    bins, d, lo, hi, bn = _bin_args(bounds, bins)
    cells = int(np.prod(bins))
    dropped = _i64()
    L = _lib.load()
    if hasattr(points, "data_ptr"):
        if points.dim() != 2 or points.shape[1] != d:
            raise ValueError("bin_scatter: point arity does not match the grid")
        if not points.is_contiguous():
            raise ValueError("bin_scatter: device points must be contiguous (npts x d)")
        if out is None:
            raise ValueError("bin_scatter: device points need a device `out` buffer")
        if out.numel() != cells:
            raise ValueError("bin_scatter: out must hold prod(bins) counts")
        ctx.check(L.kg_bin_scatter(ctx.h, int(points.shape[0]), d, C.c_void_p(points.data_ptr()), _ptr(lo), _ptr(hi),
                                   bn.ctypes.data_as(_pi), 1, C.c_void_p(out.data_ptr()), C.byref(dropped)))
        return BinnedCounts(out, int(dropped.value))
    pts = np.ascontiguousarray(np.asarray(points, dtype=np.float64))
    if pts.size == 0:
        pts = pts.reshape(0, d)
    if pts.ndim != 2 or pts.shape[1] != d:
        raise ValueError("bin_scatter: point arity does not match the grid")
    counts = np.zeros(cells)
    ctx.check(L.kg_bin_scatter(ctx.h, pts.shape[0], d, pts.ctypes.data_as(C.c_void_p), _ptr(lo), _ptr(hi),
                               bn.ctypes.data_as(_pi), 0, counts.ctypes.data_as(C.c_void_p), C.byref(dropped)))
    return BinnedCounts(counts.reshape(bins, order="F"), int(dropped.value))


def bspline_design_device(points, order=4, n_basis=0, ctx: Context | None = None):
    """bspline_design evaluated on the device (bit-identical to bspline_design)."""
    ctx = ctx or default_context()
    pts = np.ascontiguousarray(np.asarray(points, dtype=np.float64))
    out = np.zeros((pts.size, int(n_basis)), order="F")
    ctx.check(_lib.load().kg_bspline_design_dev(ctx.h, pts.size, pts.ctypes.data_as(C.c_void_p), int(order),
                                                int(n_basis), 0, out.ctypes.data_as(C.c_void_p)))
    return out


def default_basis_count(n_points, ratio):
    """Basis-count rule max(ceil(n/ratio), 5) (bspline.cpp:20-26)."""
    r = _lib.load().kg_default_basis_count(int(n_points), int(ratio))
    if r < 0:
        raise ValueError("default_basis_count: arguments must be positive")
    return int(r)
