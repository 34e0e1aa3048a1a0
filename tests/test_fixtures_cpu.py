"""CPU checks of the committed parity fixtures (tests/golden/path_C*.npz):
internal consistency, and that the oracle reproduces the C1 fixture from the
seeded config inputs (the generator and the checker are pinned together)."""
import json
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_1510_03298_b200 import configs
from tests.test_gpu_fixtures import coefs_of, fingerprint_ok, load, sha, supports_of

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
def test_fixture_is_self_consistent(name):
    fx = load(name)
    meta = fx["meta"]
    m = meta["models"]
    assert len(fx["lambdas"]) == m and len(fx["deviance"]) == m and fx["fingerprints"].shape == (m, 6)
    assert np.all(np.diff(fx["lambdas"]) < 0)
    supp = supports_of(fx)
    assert [int(s.sum()) for s in supp] == list(fx["nonzero"])
    for t, th in coefs_of(fx).items():
        assert fingerprint_ok(th, fx["fingerprints"][t], meta["fp_seed"])
    assert fx["trace_offsets"][-1] == len(fx["traces"]) == int(np.sum(fx["outer_iters"]))


def test_config_generator_reproduces_fixture_inputs():
    """The seeded generator is host-independent (no BLAS): the C1/C3 inputs hash
    to the fixtures' values (the GPU tests rebuild the inputs the same way)."""
    for name in ("C1", "C3"):
        d = configs.make(name, bspline=O.bspline_design)
        meta = load(name)["meta"]
        assert sha(d["y"]) == meta["y_sha256"]
        assert [sha(x) for x in d["design"][0]] == meta["factor_sha256"]


def test_oracle_reproduces_the_c1_fixture():
    fx = load("C1")
    d = configs.make("C1", bspline=O.bspline_design)
    r = O.fit_path(d["design"], d["family"], d["y"], n_lambda=d["n_lambda"], lambda_min_ratio=d["lambda_min_ratio"])
    assert r["inner_iters"] == list(fx["inner_iters"])
    np.testing.assert_allclose(r["objectives"], fx["objectives"], rtol=1e-12)
    want = coefs_of(fx)
    for t in range(len(r["lambdas"])):
        th = np.concatenate([np.asarray(b).ravel(order="F") for b in r["coefficients"][t]])
        assert np.array_equal(th != 0, supports_of(fx)[t])
        np.testing.assert_allclose(th, want[t], rtol=0, atol=1e-12 * np.max(np.abs(want[t])) + 1e-300)


def test_spectral_fixture_covers_every_config_factor():
    with open(os.path.join(GOLDEN, "spectral_radii.json")) as f:
        rows = json.load(f)
    want = {(c, j) for c, cfg in configs.CONFIGS.items() for j in range(len(cfg["n"]))}
    assert {(r["config"], r["mode"]) for r in rows} == want
    r = next(r for r in rows if r["n"] == 1024 and r["p"] == 256)
    X = O.bspline_design(np.linspace(0.0, 1.0, 1024), 4, 256)
    assert abs(O.spectral_radius(np.asfortranarray(X.T @ X)) - r["rho"]) <= 1e-13 * r["rho"]
