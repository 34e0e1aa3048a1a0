"""B200-native penalized GLAM solver (arXiv 1510.03298): design-matrix-free
lasso / ridge / elastic-net GLM fits over Kronecker-product designs.

``paper_1510_03298_b200.kronglm`` mirrors the reference ``kronglm`` Python
module; the compute runs in ``libkronglm_b200.so`` (hand-written sm_100a CUDA
behind the C ABI in include/kronglm_b200.h)."""
from . import kronglm  # noqa: F401
from . import build  # noqa: F401  (module: build.build() compiles the CUDA library)

__all__ = ["kronglm", "build"]
