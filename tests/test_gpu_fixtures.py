"""Config-size parity: the CUDA path, through the C ABI, against the committed
oracle fixtures of every BASELINE config (tests/golden/path_C{k}.npz, made by
tests/golden/make_path_fixtures.py from the CPU restatement on the same seeded
inputs).

North-star parity protocol, per fitted model:
  * identical truncation and status;
  * identical support {i : theta_i != 0};
  * coefficients within 1e-8 relative (max |d theta| / max |theta|);
  * objective and deviance within 1e-8 relative;
  * identical inner and outer iteration counts, and per outer iteration
    (OuterTrace, outer.hpp:26-47) identical Armijo j and step alpha.
C1-C3 are full auto-grid paths (path.cpp:29-45); C4 and C5 are the first
lambdas of the grid passed explicitly (path.cpp:47-81)."""
import hashlib
import json
import os

import numpy as np
import pytest

from paper_1510_03298_b200 import configs
from paper_1510_03298_b200 import kronglm as K

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
REL = 1e-8


def sha(a) -> str:
    return hashlib.sha256(np.asfortranarray(a).tobytes(order="F")).hexdigest()


def load(name):
    z = np.load(os.path.join(GOLDEN, f"path_{name}.npz"))
    fx = {k: z[k] for k in z.files}
    fx["meta"] = json.loads(bytes(z["meta"]).decode())
    return fx


def supports_of(fx):
    p = fx["meta"]["p_total"]
    return [np.unpackbits(fx["support"][t])[:p].astype(bool) for t in range(fx["meta"]["models"])]


def coefs_of(fx):
    """Dense coefficient vectors of the fixture's FULL models (packed support
    + nonzero values); {t: theta_t}."""
    supp = supports_of(fx)
    out, off = {}, 0
    for t in fx["meta"]["full_models"]:
        th = np.zeros(fx["meta"]["p_total"])
        k = int(supp[t].sum())
        th[supp[t]] = fx["values"][off:off + k]
        off += k
        out[t] = th
    return out


def fingerprint_ok(th, fp, seed, rtol=REL):
    """max|theta|, sum|theta|, sum theta^2 and <r_k, theta> (make_path_fixtures.py)
    agree with the oracle's within what an `rtol` relative coefficient match allows."""
    p = th.size
    scale = fp[0]
    tol = rtol * scale
    if abs(np.max(np.abs(th)) - fp[0]) > tol:
        return False
    if abs(np.sum(np.abs(th)) - fp[1]) > tol * p:
        return False
    if abs(th @ th - fp[2]) > 2.0 * tol * np.sum(np.abs(th)) + tol * tol * p:
        return False
    for k in range(3):
        r = np.random.default_rng(seed + k).standard_normal(p)
        if abs(r @ th - fp[3 + k]) > tol * np.sum(np.abs(r)) + 1e-12 * abs(fp[3 + k]):
            return False
    return True


def rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)


def unstable_supports(name):
    """Models whose support differs between the two valid oracle builds of the
    conditioning probe (C3: the last, least-penalised models 47-48, where a
    coefficient sits on the soft-threshold boundary to within the 1e-5 floor)."""
    path = os.path.join(GOLDEN, f"conditioning_{name}.json")
    if not os.path.exists(path):
        return set()
    with open(path) as f:
        return {r["t"] for r in json.load(f)["rows"] if not r["same_support"]}


def coef_tolerance(name, m):
    """Per-model coefficient tolerance: 1e-8 relative (north_star), or 4x the
    conditioning floor where the problem amplifies rounding beyond it -- the
    spread between two valid builds of the oracle itself (no FMA vs FMA
    contraction, tools/conditioning_probe.py -> tests/golden/conditioning_<C>.json).
    On C3 that floor reaches 1e-5 at the last, least-penalised models (with
    identical iteration counts); everywhere else it is below 1e-8."""
    tol = [REL] * m
    path = os.path.join(GOLDEN, f"conditioning_{name}.json")
    if os.path.exists(path):
        with open(path) as f:
            rows = json.load(f)["rows"]
        for r in rows:
            if r["t"] < m:
                tol[r["t"]] = max(REL, 4.0 * r["coef_rel"])
    return tol


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
def test_path_matches_oracle_fixture(name):
    fx = load(name)
    meta = fx["meta"]
    d = configs.make(name)
    # identical inputs first: a mismatch here is a generator problem, not a solver one
    assert sha(d["y"]) == meta["y_sha256"], "config inputs differ from the fixture's"
    assert [sha(x) for x in d["design"][0]] == meta["factor_sha256"]
    design = K.Design(d["design"])
    obs = K.Observation(design, d["y"])
    fam = d["family"]
    if meta["prefix"]:
        res = K.fit_path_resident(design, obs, fam, lambdas=fx["lambdas"])
        lmax = K.lambda_max(d["design"], fam, d["y"])
        assert rel(lmax, float(fx["lambda_max"][0])) <= 1e-13
    else:
        res = K.fit_path_resident(design, obs, fam, n_lambda=d["n_lambda"], lambda_min_ratio=d["lambda_min_ratio"])
        assert rel(res.lambda_max, float(fx["lambda_max"][0])) <= 1e-13
        np.testing.assert_allclose(res.lambdas, fx["lambdas"], rtol=1e-13, atol=0)
    m = meta["models"]
    assert res.n_models == m
    assert res.truncated == meta["truncated"]
    assert [K.STATUS.index(s) for s in res.status] == list(fx["status"])
    assert res.inner_iters == list(fx["inner_iters"]), "inner iteration counts differ"
    assert res.outer_iters == list(fx["outer_iters"]), "outer iteration counts differ"
    want = coefs_of(fx)
    supp = supports_of(fx)
    got = res.coefs()
    dev = res.deviance(obs, fam)
    tol = coef_tolerance(name, m)
    unstable = unstable_supports(name)
    for t in range(m):
        g = got[t]
        if t in unstable:
            # the two oracle builds themselves disagree on this model's support: an
            # entry may flip only where it is zero within the model's tolerance
            diff = (g != 0) != supp[t]
            assert np.all(np.abs(g[diff]) <= tol[t] * float(fx["fingerprints"][t][0])), f"model {t}: support differs"
        else:
            assert np.array_equal(g != 0, supp[t]), f"model {t}: support differs"
            assert int(np.count_nonzero(g)) == int(fx["nonzero"][t])
        if t in want:
            w = want[t]
            scale = max(np.max(np.abs(w)), 1e-300)
            assert np.max(np.abs(g - w)) / scale <= tol[t], f"model {t}: coefficients"
        assert fingerprint_ok(g, fx["fingerprints"][t], meta["fp_seed"], tol[t]), f"model {t}: coefficient fingerprints"
        assert rel(res.objectives[t], fx["objectives"][t]) <= REL, f"model {t}: objective"
        assert rel(dev[t], fx["deviance"][t]) <= REL, f"model {t}: deviance"
    # OuterTrace: one record per outer iteration, same Armijo decisions
    off = fx["trace_offsets"]
    keys = meta["trace_keys"]
    for t in range(m):
        recs = fx["traces"][off[t]:off[t + 1]]
        tr = res.traces[t]
        assert len(tr) == len(recs)
        for r, ref in zip(tr, recs):
            ref = dict(zip(keys, ref))
            assert r["armijo_j"] == int(ref["armijo_j"])
            assert r["alpha"] == ref["alpha"]
            assert r["inner_iterations"] == int(ref["inner_iterations"])
            assert r["inner_converged"] == bool(ref["inner_converged"])
            assert rel(r["objective"], ref["objective"]) <= REL
            # L-hat = max(v)/n * prod(rho_j): the spectral radii agree to ~1e-13 (spectral
            # test); max(v) follows the coefficients, so it gets the model's coefficient tolerance
            assert rel(r["lipschitz"], ref["lipschitz"]) <= max(1e-11, tol[t])
            assert abs(r["delta_k"] - ref["delta_k"]) <= REL * max(1.0, abs(ref["objective"]))
    res.close()
    obs.close()
    design.close()


def test_spectral_radii_of_every_config_factor_match_oracle():
    """spectral_radius (spectral.cpp:8-42) of each config factor, including the
    4096 x 256 (C4) and 1024 x 256 (C5) B-spline factors."""
    with open(os.path.join(GOLDEN, "spectral_radii.json")) as f:
        rows = json.load(f)
    assert {(r["n"], r["p"]) for r in rows} >= {(4096, 256), (1024, 256)}
    for r in rows:
        X = K.bspline_design(np.linspace(0.0, 1.0, r["n"]), 4, r["p"])
        assert sha(X) == r["x_sha256"]
        D = K.Design([[X]])
        # Same seed and stop rule (two consecutive |d rho| <= 1e-14 rho); for the
        # slowly converging p = 256 factors (spectral gap ~1.6e-4) the estimate
        # still creeps by ~1e-14 per step when it stops, so a different
        # summation order can stop a few steps apart: ~1e-12 relative.
        assert rel(D.spectral(0, 0), r["rho"]) <= 1e-11, (r["config"], r["mode"])
        D.close()
