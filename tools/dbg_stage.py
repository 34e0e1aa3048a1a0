"""Compare the whole-path kernel with and without a KG_PATH_DBG switch."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1510_03298_b200 import configs  # noqa: E402
from paper_1510_03298_b200 import kronglm as K  # noqa: E402

d = configs.make(sys.argv[1] if len(sys.argv) > 1 else "C1")
ctx = K.Context(0)
D = K.Design(d["design"], ctx)
O = K.Observation(D, d["y"])
out = {}
for f in ("1", "0"):
    os.environ["KG_PATH_DBG"] = f
    r = K.fit_path_resident(D, O, "gaussian", n_lambda=4, lambda_min_ratio=d["lambda_min_ratio"],
                            inner_maxit=50)
    out[f] = r
    print(f, r.n_models, r.inner_iters, r.status, [float(x) for x in r.objectives], flush=True)
a, b = out["1"], out["0"]
for t in range(min(a.n_models, b.n_models)):
    print(t, float(np.max(np.abs(a.coef(t) - b.coef(t)))))
