"""ctypes binding of the C ABI in include/kronglm_b200.h (the drop-in boundary).

There is no fallback: if libkronglm_b200.so is missing or no CUDA device is
present the calls raise."""
import ctypes as C
import os
import threading

from . import build as _build

_P = C.POINTER
_d = C.c_double
_i64 = C.c_int64
_vp = C.c_void_p
_pd = _P(_d)
_pi = _P(_i64)

KG_OK, KG_EINVAL, KG_EEVAL, KG_ERUNTIME, KG_EDIVERGE, KG_EPOWER, KG_ECUDA, KG_ENCCL, KG_ENOMEM = range(9)


class KgError(RuntimeError):
    def __init__(self, status, msg, cell=-1):
        super().__init__(msg)
        self.status = status
        self.cell = cell


class EvalError(KgError):
    """kronglm::EvalError (family.hpp:53-61); ``cell`` is the 0-based flat cell index."""


class InvalidArgument(KgError, ValueError):
    """std::invalid_argument -> Python ValueError (as pybind11 maps it)."""


class OuterRecord(C.Structure):
    """kg_outer_record: one OuterRecord of OuterTrace (outer.hpp:26-47)."""
    _fields_ = [("objective", _d), ("alpha", _d), ("delta_k", _d), ("lipschitz", _d),
                ("inner_iterations", _i64), ("inner_converged", C.c_int32), ("armijo_j", C.c_int32)]


class PathCfg(C.Structure):
    _fields_ = [
        ("n_lambda", _i64), ("lambda_min_ratio", _d), ("max_outer", _i64),
        ("armijo_alpha0", _d), ("armijo_b", _d), ("armijo_v", _d),
        ("armijo_max_backtracks", _i64), ("weight_mode", _i64), ("outer_tol", _d),
        ("nu", _d), ("inner_max_iters", _i64), ("inner_tol", _d),
        ("extrapolation", _i64), ("monitor_every", _i64),
    ]


_SIGS = {
    "kg_path_cfg_default": (None, [_P(PathCfg)]),
    "kg_ctx_create": (C.c_int, [C.c_int, _P(_vp)]),
    "kg_ctx_create_sharded": (C.c_int, [C.c_int, C.c_int, C.c_int, _vp, _P(_vp)]),
    "kg_nccl_unique_id": (C.c_int, [_vp]),
    "kg_ctx_destroy": (None, [_vp]),
    "kg_last_error": (C.c_char_p, [_vp]),
    "kg_last_error_cell": (_i64, [_vp]),
    "kg_ctx_stream": (_vp, [_vp]),
    "kg_ctx_synchronize": (C.c_int, [_vp]),
    "kg_ctx_shard": (None, [_vp, _P(C.c_int), _P(C.c_int)]),
    "kg_design_create": (C.c_int, [_vp, _i64, _i64, _pi, _pi, _P(_pd), _P(_vp)]),
    "kg_design_destroy": (None, [_vp]),
    "kg_design_n": (_i64, [_vp]),
    "kg_design_p": (_i64, [_vp]),
    "kg_design_spectral": (C.c_int, [_vp, _i64, _i64, _pd]),
    "kg_obs_create": (C.c_int, [_vp, _vp, _vp, _vp, C.c_int, _P(_vp)]),
    "kg_obs_destroy": (None, [_vp]),
    "kg_h_map": (C.c_int, [_vp, _vp, _pd, _pd]),
    "kg_g_map": (C.c_int, [_vp, _vp, _pd, _pd]),
    "kg_xtwx_apply": (C.c_int, [_vp, _vp, _pd, _pd, _pd]),
    "kg_rho": (C.c_int, [_vp, _i64, _pd, _i64, _pi, _pd, _pd]),
    "kg_lambda_max": (C.c_int, [_vp, _vp, _vp, C.c_int, _d, C.c_int, _d, _pd]),
    "kg_fit_path": (C.c_int, [_vp, _vp, _vp, C.c_int, _d, C.c_int, _d, _P(PathCfg), _pd, _i64, _P(_vp)]),
    "kg_outer_solve": (C.c_int, [_vp, _vp, _vp, C.c_int, _d, C.c_int, _d, _P(PathCfg), _d, _P(_vp)]),
    "kg_result_n_models": (_i64, [_vp]),
    "kg_result_truncated": (C.c_int, [_vp]),
    "kg_result_lambda_max": (_d, [_vp]),
    "kg_result_lambda": (_d, [_vp, _i64]),
    "kg_result_objective": (_d, [_vp, _i64]),
    "kg_result_outer_iters": (_i64, [_vp, _i64]),
    "kg_result_inner_iters": (_i64, [_vp, _i64]),
    "kg_result_status": (C.c_int, [_vp, _i64]),
    "kg_result_nonzero": (_i64, [_vp, _i64]),
    "kg_result_initial_objective": (_d, [_vp, _i64]),
    "kg_result_n_outer": (_i64, [_vp, _i64]),
    "kg_result_trace": (C.c_int, [_vp, _i64, _P(OuterRecord)]),
    "kg_result_deviance": (C.c_int, [_vp, _vp, _vp, _vp, C.c_int, _pd]),
    "kg_result_nonzeros": (C.c_int, [_vp, C.POINTER(_i64)]),
    "kg_result_coef": (C.c_int, [_vp, _i64, _pd]),
    "kg_result_coefs": (C.c_int, [_vp, _i64, _i64, _pd]),
    "kg_result_free": (None, [_vp]),
    "kg_host_alloc": (C.c_int, [C.c_size_t, _P(_vp)]),
    "kg_host_free": (None, [_vp]),
    "kg_predict": (C.c_int, [_vp, _vp, C.c_int, _pd, _pd, _pd]),
    "kg_bspline_design": (C.c_int, [_i64, _pd, _i64, _i64, _pd]),
    "kg_default_basis_count": (_i64, [_i64, _i64]),
    "kg_bin_scatter": (C.c_int, [_vp, _i64, _i64, _vp, _pd, _pd, _pi, C.c_int, _vp, C.POINTER(_i64)]),
    "kg_bspline_design_dev": (C.c_int, [_vp, _i64, _vp, _i64, _i64, C.c_int, _vp]),
    "kg_linear_index": (_i64, [_i64, _pi, _pi]),
    "kg_halo_plan": (C.c_int, [_i64, _i64, _pd, C.c_int, C.c_int, C.POINTER(_i64)]),
    "kg_slab_gather_plan": (C.c_int, [_i64, _i64, _pd, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                      C.POINTER(C.c_int32)]),
    "kg_design_halo": (C.c_int, [_vp, C.POINTER(_i64)]),
    "kg_time_kernel": (C.c_int, [_vp, _vp, _vp, C.c_int, C.c_int, _pd, _pd]),
    "kg_path_kernel_stats": (C.c_int, [_vp, _pd, _pd, C.POINTER(_i64)]),
    "kg_mse_heldout": (C.c_int, [_vp, _vp, _vp, C.c_int, _pd, _pd, _pd, C.POINTER(_i64)]),
    "kg_launch_count": (_i64, [_vp]),
    "kg_launch_count_reset": (None, [_vp]),
}

EXPORTED = sorted(_SIGS)

_lib = None
_lock = threading.Lock()


def lib_path():
    return _build.LIB


def load(build_if_missing=True):
    """Load libkronglm_b200.so (building it in-tree from csrc/ if absent)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(_build.LIB):
                if not build_if_missing:
                    raise OSError(f"{_build.LIB} is missing; run paper_1510_03298_b200.build.build()")
                _build.build()
            L = C.CDLL(_build.LIB)
            for name, (res, args) in _SIGS.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
    return _lib


def check(status, ctx=None):
    if status == KG_OK:
        return
    L = load()
    msg = L.kg_last_error(ctx).decode() if ctx else f"kronglm_b200 error {status}"
    if status == KG_EINVAL:
        raise InvalidArgument(status, msg)
    if status == KG_EEVAL:
        raise EvalError(status, msg, int(L.kg_last_error_cell(ctx)))
    raise KgError(status, msg)
