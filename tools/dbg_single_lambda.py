"""Debug helper: the single-lambda boundary case of test_single_lambda_and_boundary."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests import helpers as H  # noqa: E402
from paper_1510_03298_b200 import kronglm as K  # noqa: E402

rng = np.random.default_rng(71)
design = H.make_design(rng, (4, 3), [(2, 3)])
y = rng.standard_normal((4, 3))
p = K.fit_path(design, "gaussian", y, n_lambda=1)
print(os.environ.get("KG_PATH_CW"), os.environ.get("KG_PATH_BS"), p["lambdas"], p["lambda_max"], p["inner_iters"],
      H.flat(p["coefficients"][0]))
