import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1510_03298_b200 import kronglm as K
from tests import helpers as H
rng = np.random.default_rng(71)
design = H.make_design(rng, (4, 3), [(2, 3)])
y = rng.standard_normal((4, 3))
for nl in (1, 3):
    p = K.fit_path(design, "gaussian", y, n_lambda=nl)
    print(os.environ.get("KG_GSTEP_NT"), nl, p["inner_iters"], [H.flat(c).tolist() for c in p["coefficients"]], p["objectives"])
