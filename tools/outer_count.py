"""Outer (IRLS) iteration counts of one config's lambda path on cuda:0."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1510_03298_b200 import configs  # noqa: E402
from paper_1510_03298_b200 import kronglm as K  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
d = configs.make(name)
D = K.Design(d["design"])
O = K.Observation(D, d["y"])
for _ in range(2):
    t0 = time.perf_counter()
    r = K.fit_path_resident(D, O, d["family"], n_lambda=d["n_lambda"], lambda_min_ratio=d["lambda_min_ratio"])
    dt = time.perf_counter() - t0
print(name, "outer", sum(r.outer_iters), list(r.outer_iters), "inner", sum(r.inner_iters), f"{dt * 1000:.1f} ms")
