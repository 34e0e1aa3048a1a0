"""Profiling driver: fits one config's lambda path `--paths` times on cuda:0
(the first fit is warm-up).  Used under ncu for launch lists / full captures."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1510_03298_b200 import configs  # noqa: E402
from paper_1510_03298_b200 import kronglm as K  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--paths", type=int, default=2)
ap.add_argument("--n-lambda", type=int, default=None)
args = ap.parse_args()
d = configs.make(args.config)
ctx = K.Context(0)
D = K.Design(d["design"], ctx)
O = K.Observation(D, d["y"])
for i in range(args.paths):
    ctx.reset_launches()
    t0 = time.perf_counter()
    r = K.fit_path_resident(D, O, d["family"], n_lambda=args.n_lambda or d["n_lambda"],
                            lambda_min_ratio=d["lambda_min_ratio"])
    dt = time.perf_counter() - t0
    print(f"path {i}: models={r.n_models} inner={sum(r.inner_iters)} launches={ctx.launches} "
          f"wall={dt * 1000:.1f} ms per-model-inner={r.inner_iters[:8]}", flush=True)
