"""Wall-clock breakdown of the public kronglm.fit_path call (design upload,
observation upload, path fit, coefficient download) for one config."""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1510_03298_b200 import configs  # noqa: E402
from paper_1510_03298_b200 import kronglm as K  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()
d = configs.make(args.config)
for rep in range(args.reps):
    t = [time.perf_counter()]
    D = K._design(d["design"])
    t.append(time.perf_counter())
    O = K.Observation(D, d["y"])
    t.append(time.perf_counter())
    r = K.fit_path_resident(D, O, d["family"], n_lambda=d["n_lambda"], lambda_min_ratio=d["lambda_min_ratio"])
    t.append(time.perf_counter())
    cs = list(r.coefs())
    t.append(time.perf_counter())
    blocks = [D.blocks(c) for c in cs]
    t.append(time.perf_counter())
    dt = np.diff(t) * 1000
    print(f"rep {rep}: design {dt[0]:.1f} ms  obs {dt[1]:.1f}  path {dt[2]:.1f}  coef D2H {dt[3]:.1f}  "
          f"blocks {dt[4]:.1f}  total {sum(dt):.1f}", flush=True)

# the public call itself, timed and profiled (after the warm-up above)
import cProfile  # noqa: E402
import pstats  # noqa: E402

for rep in range(3):
    t0 = time.perf_counter()
    out = K.fit_path(d["design"], d["family"], d["y"], n_lambda=d["n_lambda"], lambda_min_ratio=d["lambda_min_ratio"])
    print(f"fit_path rep {rep}: {1000 * (time.perf_counter() - t0):.1f} ms", flush=True)
pr = cProfile.Profile()
pr.enable()
out = K.fit_path(d["design"], d["family"], d["y"], n_lambda=d["n_lambda"], lambda_min_ratio=d["lambda_min_ratio"])
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
