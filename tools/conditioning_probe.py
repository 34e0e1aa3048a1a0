#!/usr/bin/env python
"""How far apart do two valid rounding orders of the SAME algorithm end up on
a config path?  Runs the oracle restatement twice on identical inputs -- the
checker build (liborc.so, -ffp-contract=off) and the FMA-contracted build
(liborc_fma.so, every a*b+c rounded once) -- and compares them model by model
with the parity protocol's measures.  This is the conditioning floor of the
coefficient criterion: any implementation whose arithmetic differs from the
reference's in rounding (the reference's own Eigen build included) cannot be
expected to agree more closely than this.

    python tools/conditioning_probe.py C3 [--threads 8] > profiles/r02_conditioning_C3.json
"""
import argparse
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def one(name, lib, threads, out):
    code = f"""
import sys, json, numpy as np
sys.path.insert(0, {ROOT!r})
from oracle import oracle as O
from paper_1510_03298_b200 import configs
O.set_threads({threads})
d = configs.make({name!r}, bspline=O.bspline_design)
r = O.fit_path(d["design"], d["family"], d["y"], n_lambda=d["n_lambda"], lambda_min_ratio=d["lambda_min_ratio"])
flat = np.stack([np.concatenate([np.asarray(b).ravel(order="F") for b in c]) for c in r["coefficients"]])
np.savez({out!r}, coef=flat, obj=np.array(r["objectives"]), inner=np.array(r["inner_iters"]),
         outer=np.array(r["outer_iters"]))
"""
    env = dict(os.environ, KRONGLM_ORACLE_LIB=lib)
    subprocess.run([sys.executable, "-c", code], check=True, env=env)
    return np.load(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    a = ap.parse_args()
    A = one(a.config, "liborc.so", a.threads, f"/tmp/cond_{a.config}_off.npz")
    B = one(a.config, "liborc_fma.so", a.threads, f"/tmp/cond_{a.config}_fma.npz")
    rows = []
    m = min(len(A["obj"]), len(B["obj"]))
    for t in range(m):
        x, y = A["coef"][t], B["coef"][t]
        rows.append({"t": t, "coef_rel": float(np.max(np.abs(x - y)) / max(np.max(np.abs(x)), 1e-300)),
                     "obj_rel": float(abs(A["obj"][t] - B["obj"][t]) / abs(A["obj"][t])),
                     "same_support": bool(np.array_equal(x != 0, y != 0)),
                     "inner": [int(A["inner"][t]), int(B["inner"][t])]})
    print(json.dumps({"config": a.config, "compare": "oracle -ffp-contract=off vs -ffp-contract=fast -mfma",
                      "max_coef_rel": max(r["coef_rel"] for r in rows), "rows": rows}))


if __name__ == "__main__":
    main()
