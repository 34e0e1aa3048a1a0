#!/usr/bin/env python
"""Generates the config-size parity fixtures tests/golden/path_C{k}.npz from
the CPU oracle (oracle/, the Eigen-free restatement of the reference fit path;
TEST INFRASTRUCTURE ONLY) on the seeded BASELINE config inputs
(paper_1510_03298_b200/configs.py, factors built with the oracle's
bspline_design so this script never loads the product library).

Per config and per fitted model t the fixture holds what the north-star parity
protocol compares:
  * lambda_t, objective F_t, deviance D_t = dev(y, H(theta_t)) (oracle
    deviance(), family.cpp conventions), outer/inner iteration counts, status;
  * the support {i : theta_t[i] != 0} as a packed bitmap, for every model;
  * the nonzero values of theta_t (so the whole vector is reconstructed) for
    the models in FULL (the first three, every tenth and the last; all of
    them when p is small) -- kept to a few MB per config;
  * for every model, size-independent fingerprints of theta_t: max |theta|,
    sum |theta|, sum theta^2 and three projections <r_k, theta> on seeded
    N(0,1) vectors r_k (default_rng(FP_SEED + k)), which a 1e-8 relative
    coefficient match implies to within 1e-8 max|theta| ||r_k||_1;
  * every OuterTrace record (objective, alpha, Delta_k, L-hat, inner
    iterations, inner convergence, Armijo j; outer.hpp:26-47);
  * sha256 of y and of every factor, so a test can tell "different inputs"
    from "different results".

Full paths (C1, C2, C3) run the auto grid (path.cpp:29-45).  C4 and C5 run a
prefix: the first K lambdas of the same grid passed explicitly (path.cpp:47-81
with lambda_sequence(lambda_max) truncated), which is what fit_path does for
those models.  Run on this CPU container:

    python tests/golden/make_path_fixtures.py C1 C2 C3 C4 C5 spectral [--threads 8]
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_1510_03298_b200 import configs  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
PREFIX = {}  # configs fitted as a lambda prefix (none: every config is a full path; ~3 h of CPU for C5)
FP_SEED = 1510032980
FULL_VALUES_MAX = 400_000  # nonzero values stored in full before switching to the FULL subset


def fingerprints(th: np.ndarray) -> np.ndarray:
    p = th.size
    proj = [float(np.random.default_rng(FP_SEED + k).standard_normal(p) @ th) for k in range(3)]
    return np.array([np.max(np.abs(th)) if p else 0.0, float(np.sum(np.abs(th))), float(th @ th)] + proj)


def full_models(m: int, flat) -> list:
    if sum(int(np.count_nonzero(f)) for f in flat) <= FULL_VALUES_MAX:
        return list(range(m))
    return sorted({0, 1, 2, m - 1} | set(range(0, m, 10)))


def sha(a) -> str:
    return hashlib.sha256(np.asfortranarray(a).tobytes(order="F")).hexdigest()


def grid(lmax, nl, ratio):
    """lambda_sequence (path.cpp:8-27) for the explicit-prefix configs."""
    step = np.log(ratio) / (nl - 1)
    return [lmax] + [lmax * float(np.exp(step * t)) for t in range(1, nl)]


def run(name: str, threads: int):
    O.set_threads(threads)
    d = configs.make(name, bspline=O.bspline_design)
    design, y, fam = d["design"], d["y"], d["family"]
    t0 = time.time()
    lmax = O.lambda_max(design, fam, y)
    if name in PREFIX:
        lams = grid(lmax, d["n_lambda"], d["lambda_min_ratio"])[:PREFIX[name]]
        r = O.fit_path(design, fam, y, lambdas=lams)
        r["lambda_max"] = lmax
    else:
        r = O.fit_path(design, fam, y, n_lambda=d["n_lambda"], lambda_min_ratio=d["lambda_min_ratio"])
    fit_s = time.time() - t0
    m = len(r["lambdas"])
    flat = [np.concatenate([np.asarray(b).ravel(order="F") for b in c]) for c in r["coefficients"]]
    p = flat[0].size
    dev = []
    for c in r["coefficients"]:
        eta = O.h_map(design, c)
        dev.append(O.deviance(fam, y, eta))
    supp = np.stack([np.packbits(f != 0) for f in flat])
    full = full_models(m, flat)
    vals = np.concatenate([flat[t][flat[t] != 0] for t in full]) if m else np.zeros(0)
    nz = np.array([int(np.count_nonzero(f)) for f in flat], dtype=np.int64)
    fps = np.stack([fingerprints(f) for f in flat])
    tr_off = np.cumsum([0] + [len(t) for t in r["traces"]]).astype(np.int64)
    keys = O.TRACE_KEYS
    tr = np.array([[float(rec[k]) for k in keys] for t in r["traces"] for rec in t]).reshape(-1, len(keys))
    meta = {"config": name, "family": fam, "n": list(d["n"]), "p": list(d["p"]), "n_lambda": d["n_lambda"],
            "lambda_min_ratio": d["lambda_min_ratio"], "models": m, "prefix": name in PREFIX,
            "truncated": bool(r["truncated"]), "y_sha256": sha(y),
            "factor_sha256": [sha(x) for x in design[0]], "p_total": p, "oracle_threads": threads,
            "oracle_fit_seconds": fit_s, "trace_keys": keys, "meta": d["meta"], "full_models": full,
            "fp_seed": FP_SEED}
    path = os.path.join(OUT, f"path_{name}.npz")
    np.savez_compressed(path, meta=np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8),
                        lambdas=np.array(r["lambdas"]), lambda_max=np.array([r["lambda_max"]]),
                        objectives=np.array(r["objectives"]), deviance=np.array(dev),
                        outer_iters=np.array(r["outer_iters"], dtype=np.int64),
                        inner_iters=np.array(r["inner_iters"], dtype=np.int64),
                        status=np.array([O.STATUS.index(s) for s in r["status"]], dtype=np.int64),
                        nonzero=nz, support=supp, values=vals, fingerprints=fps, traces=tr, trace_offsets=tr_off)
    print(f"{name}: {m} models, {sum(r['inner_iters'])} FISTA iterations, oracle {fit_s:.1f} s, "
          f"{os.path.getsize(path) / 1e6:.2f} MB -> {path}", flush=True)


def spectral():
    """spectral_radius(X_j^T X_j) of every config factor (spectral.cpp:8-42:
    fixed-seed power iteration, two settled steps at 1e-14) ->
    spectral_radii.json; includes the p_j = 256 factors of C4 and C5
    (~1e5 iterations)."""
    out = []
    for name, cfg in configs.CONFIGS.items():
        for j, (nj, pj) in enumerate(zip(cfg["n"], cfg["p"])):
            X = O.bspline_design(np.linspace(0.0, 1.0, nj), 4, pj)
            t0 = time.time()
            rho = O.spectral_radius(np.asfortranarray(X.T @ X))
            out.append({"config": name, "mode": j, "n": nj, "p": pj, "rho": rho, "x_sha256": sha(X),
                        "oracle_seconds": time.time() - t0})
            print(f"{name} mode {j}: {nj}x{pj} rho = {rho!r} ({time.time() - t0:.1f} s)", flush=True)
    with open(os.path.join(OUT, "spectral_radii.json"), "w") as f:
        json.dump(out, f, indent=1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+", help="C1..C5, or 'spectral'")
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    a = ap.parse_args()
    for c in a.configs:
        if c == "spectral":
            spectral()
        else:
            run(c, a.threads)


if __name__ == "__main__":
    main()
