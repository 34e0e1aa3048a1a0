"""Command line front end of the fit path (the reference's ``kronglm`` tool,
proj/tools/main.cpp: ``fit`` and ``predict``), on the B200 solver.

  python -m paper_1510_03298_b200.cli fit --response y.glam (--design X1.csv ... | --bspline)
         --family poisson --out DIR [--weights a.glam] [--penalty ...] [--nlambda ...] ...
  python -m paper_1510_03298_b200.cli predict --fit DIR --out DIR [--truth y.glam --mask m.glam] [--eta]

Same options, defaults, output files (path.json, coef_L%03d_C%d.glam,
mu_L%03d.glam, eta_L%03d.glam, mse.tsv) and exit codes (0 ok, 1 error,
3 truncated path) as main.cpp:30-32, 130-323, 463-535.  The simulator and the
dense benchmark subcommands are outside the fit path and are not
provided.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

from . import glamio
from . import kronglm as K

EXIT_OK, EXIT_ERROR, EXIT_TRUNCATED = 0, 1, 3
LINKS = {"gaussian": "identity", "binomial": "logit", "poisson": "log", "gamma": "log"}


def _family(name: str) -> str:  # family_from_name (family.cpp:58-64)
    if name not in LINKS:
        raise ValueError("unknown family: " + name)
    return name


def _weight_mode(name: str) -> str:  # weight_mode_from_name (outer.cpp:17-22)
    if name == "exact":
        return "exact"
    if name in ("unit", "one"):
        return "unit"
    if name in ("tensor", "tensor_approx"):
        return "tensor"
    raise ValueError("unknown weight mode: " + name)


def _penalty(name: str) -> str:  # main.cpp:123-128
    if name in ("lasso", "ridge"):
        return name
    if name in ("elasticnet", "elastic_net"):
        return "elasticnet"
    raise ValueError("unknown penalty: " + name)


def _float_list(text: str):
    return [float(v) for v in text.split(",")]


def _tag(t: int) -> str:
    return "L%03d" % t


def _add_design_flags(p):  # main.cpp:41-50
    p.add_argument("--design", action="append", default=[],
                   help="marginal design matrix CSV, repeated per dimension per component")
    p.add_argument("--bspline", action="store_true", help="build a B-spline design on the grid indices 1..n_j")
    p.add_argument("--basis-ratio", type=int, default=5, help="basis-count rule p_j = max(ceil(n_j/ratio), 5)")
    p.add_argument("--order", type=int, default=4, help="B-spline order (4 = cubic)")


def build_design(files, bspline, basis_ratio, order, dims):
    """main.cpp:52-93."""
    if bspline:
        if files:
            raise ValueError("give either --design files or --bspline, not both")
        return [[K.bspline_design(np.arange(1.0, n + 1.0), order, K.default_basis_count(n, basis_ratio))
                 for n in dims]]
    d = len(dims)
    if not files or len(files) % d != 0:
        raise ValueError("need --bspline or c*d --design files (d = response dimension count)")
    comps, nxt = [], 0
    for _ in range(len(files) // d):
        factors = []
        for j in range(d):
            m = glamio.read_csv_matrix(files[nxt])
            nxt += 1
            if m.shape[0] != dims[j]:
                raise ValueError(f"design file {files[nxt - 1]} has {m.shape[0]} rows but dimension {j + 1} "
                                 f"needs {dims[j]}")
            factors.append(m)
        comps.append(factors)
    return comps


def run_fit(a) -> int:
    """main.cpp:130-236."""
    y = glamio.read_array(a.response)
    w = glamio.read_array(a.weights) if a.weights else None
    fam = _family(a.family)
    pen = _penalty(a.penalty)
    alpha = a.alpha if pen == "elasticnet" else 0.0  # PenaltySpec::lasso()/ridge() carry alpha 0
    iwls = _weight_mode(a.iwls)
    dims = list(y.shape)
    comps = build_design(a.design, a.bspline, a.basis_ratio, a.order, dims)
    lambdas = sorted((v for grp in a.lambdas for v in grp), reverse=True) if a.lambdas else None
    D = K.Design(comps)
    obs = K.Observation(D, y, w)
    res = K.fit_path_resident(D, obs, fam, pen, alpha, lambdas, n_lambda=a.nlambda,
                              lambda_min_ratio=a.lambda_min_ratio, iwls=iwls, nu=a.nu, tol=a.tol, maxit=a.maxit,
                              inner_tol=a.inner_tol, inner_maxit=a.inner_maxit)
    os.makedirs(a.out, exist_ok=True)
    meta = {"format": "kronglm-path", "version": 1, "family": fam, "link": LINKS[fam], "penalty": pen,
            "alpha": alpha, "iwls": iwls, "nu": a.nu, "lambda_max": res.lambda_max, "truncated": res.truncated,
            "response_dims": dims, "n_components": len(comps),
            "coef_dims": [list(b) for b in D.block_dims]}
    meta["design"] = ({"kind": "bspline", "basis_ratio": a.basis_ratio, "order": a.order} if a.bspline
                      else {"kind": "csv", "files": list(a.design)})
    models = []
    coefs = res.coefs()
    for t in range(res.n_models):
        flat = coefs[t]
        files = []
        for r, block in enumerate(D.blocks(flat)):
            name = f"coef_{_tag(t)}_C{r}.glam"
            glamio.write_array(os.path.join(a.out, name), block)
            files.append(name)
        models.append({"lambda": res.lambdas[t], "objective": res.objectives[t],
                       "nonzero": int(np.count_nonzero(flat)), "outer_iters": res.outer_iters[t],
                       "inner_iters": res.inner_iters[t], "converged": res.status[t] == "converged",
                       "coef_files": files})
        if a.save_mu:
            _, mu = K.predict(D, fam, D.blocks(flat))
            glamio.write_array(os.path.join(a.out, f"mu_{_tag(t)}.glam"), mu)
    meta["models"] = models
    with open(os.path.join(a.out, "path.json"), "w") as f:
        f.write(json.dumps(meta, indent=2, sort_keys=True) + "\n")  # nlohmann::json keeps keys sorted
    print(f"fitted {res.n_models} models" + (" (path truncated)" if res.truncated else ""))
    return EXIT_TRUNCATED if res.truncated else EXIT_OK


def run_predict(a) -> int:
    """main.cpp:249-323."""
    try:
        with open(os.path.join(a.fit, "path.json")) as f:
            meta = json.load(f)
    except OSError:
        raise RuntimeError("cannot open " + a.fit + "/path.json") from None
    if meta.get("format", "") != "kronglm-path":
        raise RuntimeError("not a fit directory: " + a.fit)
    fam = _family(meta["family"])
    dims = [int(e) for e in meta["response_dims"]]
    files, bspline, ratio, order = list(a.design), a.bspline, a.basis_ratio, a.order
    if not files and not bspline:  # reconstruct the design from the fit metadata
        dm = meta["design"]
        if dm["kind"] == "bspline":
            bspline, ratio, order = True, int(dm["basis_ratio"]), int(dm["order"])
        else:
            files = list(dm["files"])
    comps = build_design(files, bspline, ratio, order, dims)
    D = K.Design(comps)
    lambdas, fits = [], []
    for model in meta["models"]:
        lambdas.append(float(model["lambda"]))
        blocks = []
        for r, name in enumerate(model["coef_files"][:len(comps)]):
            blk = glamio.read_array(os.path.join(a.fit, name))
            if tuple(blk.shape) != tuple(D.block_dims[r]):
                raise RuntimeError("coefficient file dims do not match the design")
            blocks.append(blk)
        fits.append(blocks)
    os.makedirs(a.out, exist_ok=True)
    mus = []
    for t, blocks in enumerate(fits):
        eta, mu = K.predict(D, fam, blocks)
        mus.append(mu)
        glamio.write_array(os.path.join(a.out, f"mu_{_tag(t)}.glam"), mu)
        if a.eta:
            glamio.write_array(os.path.join(a.out, f"eta_{_tag(t)}.glam"), eta)
    if a.truth:
        if not a.mask:
            raise ValueError("--truth needs --mask")
        truth = glamio.read_array(a.truth)
        mask = glamio.read_array(a.mask)
        if list(truth.shape) != dims or list(mask.shape) != dims:
            raise ValueError("mse_heldout: array dims do not match the design")
        mf = mask.ravel(order="F")
        if np.any((mf != 0.0) & (mf != 1.0)):
            raise ValueError("mse_heldout: mask entries must be 0 or 1")
        if not np.any(mf == 1.0):
            raise ValueError("mse_heldout: empty held-out mask")
        if not fits:
            raise ValueError("mse_heldout: empty path")
        sel = mf == 1.0
        tf = truth.ravel(order="F")[sel]
        mse, argmin = [], 0
        for t, mu in enumerate(mus):  # path.cpp:111-121, ascending cell order
            d = mu.ravel(order="F")[sel] - tf
            s = float(np.cumsum(d * d)[-1])  # sequential sum, as the reference loop
            mse.append(s)
            if s < mse[argmin]:
                argmin = t
        with open(os.path.join(a.out, "mse.tsv"), "w") as f:
            f.write("model\tlambda\tmse\targmin\n")
            for t in range(len(mse)):
                f.write("%d\t%.17g\t%.17g\t%d\n" % (t, lambdas[t], mse[t], 1 if t == argmin else 0))
        print(f"minimal held-out MSE at model {argmin} (lambda = {lambdas[argmin]:g})")
    return EXIT_OK


def parser():
    ap = argparse.ArgumentParser(prog="kronglm", description="penalized GLAM fits on B200")
    sub = ap.add_subparsers(dest="cmd")
    f = sub.add_parser("fit", help="fit a regularization path")
    f.add_argument("--response", required=True, help="response ArrayFile")
    f.add_argument("--weights", default="", help="prior observation weight ArrayFile")
    _add_design_flags(f)
    f.add_argument("--family", required=True, help="gaussian|binomial|poisson|gamma")
    f.add_argument("--penalty", default="lasso", help="lasso|ridge|elasticnet")
    f.add_argument("--alpha", type=float, default=0.0, help="elastic net quadratic mix")
    f.add_argument("--nlambda", type=int, default=100)
    f.add_argument("--lambda-min-ratio", type=float, default=1e-4)
    f.add_argument("--lambda", dest="lambdas", action="append", type=_float_list, default=None,
                   help="explicit lambda values (comma separated, repeatable)")
    f.add_argument("--nu", type=float, default=1.0, help="inner stepsize policy in [0,1]")
    f.add_argument("--iwls", default="exact", help="exact|unit|tensor")
    f.add_argument("--tol", type=float, default=1e-8, help="outer relative tolerance")
    f.add_argument("--maxit", type=int, default=100, help="outer iteration cap")
    f.add_argument("--inner-tol", type=float, default=1e-8)
    f.add_argument("--inner-maxit", type=int, default=2000)
    f.add_argument("--save-mu", action="store_true", help="also write fitted mean arrays")
    f.add_argument("--out", required=True, help="output directory")
    p = sub.add_parser("predict", help="evaluate fitted models")
    p.add_argument("--fit", required=True, help="directory written by fit")
    _add_design_flags(p)
    p.add_argument("--truth", default="", help="true response ArrayFile for MSE")
    p.add_argument("--mask", default="", help="0/1 held-out mask ArrayFile")
    p.add_argument("--eta", action="store_true", help="also write linear predictor arrays")
    p.add_argument("--out", required=True, help="output directory")
    return ap


def main(argv=None) -> int:
    args = parser().parse_args(argv)
    try:
        if args.cmd == "fit":
            return run_fit(args)
        if args.cmd == "predict":
            return run_predict(args)
    except Exception as err:  # main.cpp:530-532
        print("error: " + str(err), file=sys.stderr)
        return EXIT_ERROR
    return EXIT_ERROR


if __name__ == "__main__":
    sys.exit(main())
