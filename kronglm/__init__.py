"""`import kronglm` -- the reference's Python module name (kronglm_py.cpp:115,
PYBIND11_MODULE(kronglm, m)) bound to the B200 path.

A re-export of paper_1510_03298_b200.kronglm: the same functions, keyword
arguments, result keys and exception types as the pybind11 module
(kronglm_py.cpp:115-269), computed by the CUDA library through its C ABI.
Existing callers switch by putting this directory on sys.path."""
from paper_1510_03298_b200.kronglm import *  # noqa: F401,F403
from paper_1510_03298_b200.kronglm import (  # noqa: F401
    Context, Design, EvalError, Observation, PathResult, bspline_design, default_basis_count, fit_path,
    fit_path_resident, g_map, h_map, lambda_max, linear_index, mse_heldout, outer_solve, predict, rho, xtwx_apply,
)
