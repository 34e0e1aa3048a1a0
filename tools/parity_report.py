#!/usr/bin/env python
"""Per-model parity table of the CUDA path against the committed oracle
fixtures (tests/golden/path_C*.npz): coefficient relative error (full models),
fingerprint check, objective / deviance relative error, iteration counts and
support equality.  Writes one JSON line per config.

    python tools/parity_report.py C1 C2 C3 C4 C5 > gpurun_out/parity.jsonl
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1510_03298_b200 import configs  # noqa: E402
from paper_1510_03298_b200 import kronglm as K  # noqa: E402
from tests.test_gpu_fixtures import coef_tolerance, coefs_of, fingerprint_ok, load, rel, sha, supports_of  # noqa: E402


def report(name):
    fx = load(name)
    meta = fx["meta"]
    d = configs.make(name)
    same_inputs = sha(d["y"]) == meta["y_sha256"]
    design = K.Design(d["design"])
    obs = K.Observation(design, d["y"])
    fam = d["family"]
    if meta["prefix"]:
        res = K.fit_path_resident(design, obs, fam, lambdas=fx["lambdas"])
    else:
        res = K.fit_path_resident(design, obs, fam, n_lambda=d["n_lambda"], lambda_min_ratio=d["lambda_min_ratio"])
    want, supp = coefs_of(fx), supports_of(fx)
    tol = coef_tolerance(name, meta["models"])
    got = res.coefs()
    dev = res.deviance(obs, fam)
    rows = []
    for t in range(min(res.n_models, meta["models"])):
        g = got[t]
        row = {"t": t, "nnz": int(np.count_nonzero(g)), "same_support": bool(np.array_equal(g != 0, supp[t])),
               "inner": [res.inner_iters[t], int(fx["inner_iters"][t])],
               "outer": [res.outer_iters[t], int(fx["outer_iters"][t])],
               "obj_rel": rel(res.objectives[t], fx["objectives"][t]), "dev_rel": rel(dev[t], fx["deviance"][t]),
               "fingerprints_ok": bool(fingerprint_ok(g, fx["fingerprints"][t], meta["fp_seed"]))}
        row["coef_tol"] = tol[t]
        if t in want:
            w = want[t]
            row["coef_rel"] = float(np.max(np.abs(g - w)) / max(np.max(np.abs(w)), 1e-300))
            row["within_tol"] = row["coef_rel"] <= tol[t]
        rows.append(row)
    out = {"config": name, "same_inputs": same_inputs, "models": [res.n_models, meta["models"]],
           "max_coef_rel": max((r.get("coef_rel", 0.0) for r in rows), default=None),
           "max_obj_rel": max((r["obj_rel"] for r in rows), default=None),
           "max_dev_rel": max((r["dev_rel"] for r in rows), default=None),
           "all_supports_equal": all(r["same_support"] for r in rows),
           "all_coefs_within_tol": all(r.get("within_tol", True) for r in rows),
           "models_at_1e-8": sum(1 for r in rows if r["coef_tol"] <= 1e-8),
           "all_iteration_counts_equal": all(r["inner"][0] == r["inner"][1] and r["outer"][0] == r["outer"][1]
                                             for r in rows),
           "rows": rows}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    for c in sys.argv[1:]:
        report(c)
