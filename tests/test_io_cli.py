"""File formats and the command line front end, mirroring the reference's
proj/tests/test_io_cli.cpp (array/CSV round trips and error cases; CLI fit ==
library fit; masked-cell invariance; predict / mse.tsv; bad inputs exit
nonzero).  The reference generates its CLI inputs with ``kronglm simulate``
(out of scope); here seeded numpy data of the same kind stands in."""
import json
import os
import struct
import subprocess
import sys

import numpy as np
import pytest

from paper_1510_03298_b200 import cli, glamio

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "gaussian_fixture")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bytes(p):
    with open(p, "rb") as f:
        return f.read()


# ------------------------------------------------------------ array files
def test_array_round_trip_byte_and_value_identical(tmp_path):
    """test_io_cli.cpp:52-71."""
    rng = np.random.default_rng(101)
    a = np.asfortranarray(rng.uniform(-10, 10, size=(3, 4, 2)))
    flat = a.reshape(-1, order="F")
    flat[0], flat[1], flat[2], flat[3] = -0.0, 1e-308, 1.7976931348623157e308, 0.1 + 0.2
    a = flat.reshape((3, 4, 2), order="F")
    glamio.write_array(tmp_path / "a.glam", a)
    b = glamio.read_array(tmp_path / "a.glam")
    assert b.shape == a.shape
    assert a.reshape(-1, order="F").tobytes() == b.reshape(-1, order="F").tobytes()
    glamio.write_array(tmp_path / "b.glam", b)
    assert _bytes(tmp_path / "a.glam") == _bytes(tmp_path / "b.glam")


def test_array_file_layout():
    """io.cpp:91-110: magic, u16 version, u16 ndim, u64 extents, column-major LE f64."""
    import tempfile
    a = np.arange(6, dtype=np.float64).reshape((2, 3), order="F")
    with tempfile.TemporaryDirectory() as d:
        glamio.write_array(os.path.join(d, "x.glam"), a)
        raw = _bytes(os.path.join(d, "x.glam"))
    want = b"GLAM" + struct.pack("<HHQQ", 1, 2, 2, 3) + struct.pack("<6d", 0, 1, 2, 3, 4, 5)
    assert raw == want


def test_array_rejects_bad_magic_version_truncation(tmp_path):
    """test_io_cli.cpp:73-98, plus the remaining io.cpp:112-149 errors."""
    rng = np.random.default_rng(102)
    glamio.write_array(tmp_path / "a.glam", rng.standard_normal((2, 2)))
    raw = _bytes(tmp_path / "a.glam")
    cases = {
        "bad_magic": (b"X" + raw[1:], "bad magic"),
        "bad_version": (raw[:4] + b"\x09" + raw[5:], "unsupported array file version 9"),
        "trunc": (raw[:-5], "payload size does not match the extents"),
        "short_header": (raw[:10], "truncated array file"),
        "zero_dims": (b"GLAM" + struct.pack("<HH", 1, 0), "array file with zero dimensions"),
        "long": (raw + b"\0" * 8, "payload size does not match the extents"),
        "tiny": (b"GL", "truncated array file"),
    }
    for name, (data, msg) in cases.items():
        p = tmp_path / (name + ".glam")
        p.write_bytes(data)
        with pytest.raises(RuntimeError, match=msg):
            glamio.read_array(p)
    with pytest.raises(RuntimeError, match="cannot open"):
        glamio.read_array(tmp_path / "missing.glam")


# ------------------------------------------------------------ CSV matrices
def test_csv_round_trip(tmp_path):
    """test_io_cli.cpp:100-110."""
    rng = np.random.default_rng(103)
    m = rng.standard_normal((5, 3))
    glamio.write_csv_matrix(tmp_path / "m.csv", m)
    back = glamio.read_csv_matrix(tmp_path / "m.csv")
    assert back.shape == (5, 3)
    assert np.array_equal(back, m)


def test_csv_reference_fixture_byte_identical(tmp_path):
    """The reference's committed fixture CSVs (written by io::write_csv_matrix)
    parse to their shapes and re-serialise to the very same bytes."""
    for name, shape in (("X1.csv", (5, 3)), ("X2.csv", (4, 2))):
        m = glamio.read_csv_matrix(os.path.join(GOLDEN, name))
        assert m.shape == shape
        glamio.write_csv_matrix(tmp_path / name, m)
        assert _bytes(tmp_path / name) == _bytes(os.path.join(GOLDEN, name))
    m = glamio.read_csv_matrix(os.path.join(GOLDEN, "X1.csv"))
    assert m[0, 0] == 0.36724096654163113 and m[4, 2] == 1.6876713302350119


def test_csv_parsing_rules_and_errors(tmp_path):
    """io.cpp:151-194: CRLF and blank lines tolerated, a trailing comma ends a
    row, from_chars rejects '+', blanks and empty fields."""
    ok = {"crlf": ("1,2\r\n3,4\r\n", [[1, 2], [3, 4]]),
          "blank": ("\n1,2\n\n3,4\n\n", [[1, 2], [3, 4]]),
          "trailing": ("1,2,\n3,4\n", [[1, 2], [3, 4]]),
          "forms": ("1e3,.5,-2.,-inf\n", [[1e3, 0.5, -2.0, -np.inf]]),
          "noeol": ("7", [[7]])}
    for name, (text, want) in ok.items():
        p = tmp_path / (name + ".csv")
        p.write_text(text)
        assert np.array_equal(glamio.read_csv_matrix(p), np.array(want, dtype=float)), name
    bad = {"plus": ("+1,2\n", "malformed number in row 1"),
           "space": ("1,2\n3, 4\n", "malformed number in row 2"),
           "empty_field": ("1,,2\n", "malformed number in row 1"),
           "sep": ("1;2\n", "expected ',' in row 1"),
           "sep2": ("1,2\n3 ,4\n", "expected ',' in row 2"),
           "exp": ("1e,2\n", "expected ',' in row 1"),
           "ragged": ("1,2\n3\n", "ragged rows"),
           "empty": ("\n\n", "empty matrix file")}
    for name, (text, msg) in bad.items():
        p = tmp_path / (name + ".csv")
        p.write_text(text)
        with pytest.raises(RuntimeError, match=msg):
            glamio.read_csv_matrix(p)
    with pytest.raises(RuntimeError, match="cannot open"):
        glamio.read_csv_matrix(tmp_path / "missing.csv")


# ------------------------------------------------------------ CLI (host-only paths)
def test_cli_bad_inputs_exit_nonzero(tmp_path, capsys):
    """test_io_cli.cpp:333-339 plus the argument checks main.cpp makes before
    any device work."""
    y = tmp_path / "y.glam"
    glamio.write_array(y, np.ones((3, 4)))
    glamio.write_csv_matrix(tmp_path / "X1.csv", np.ones((3, 2)))
    glamio.write_csv_matrix(tmp_path / "X2.csv", np.ones((5, 2)))
    out = str(tmp_path / "o")
    cases = [
        (["fit", "--response", "/nonexistent.glam", "--bspline", "--family", "gaussian", "--out", out],
         "error: cannot open /nonexistent.glam"),
        (["fit", "--response", str(y), "--family", "nosuch", "--bspline", "--out", out], "error: unknown family: nosuch"),
        (["fit", "--response", str(y), "--family", "gaussian", "--penalty", "l0", "--bspline", "--out", out],
         "error: unknown penalty: l0"),
        (["fit", "--response", str(y), "--family", "gaussian", "--iwls", "approx", "--bspline", "--out", out],
         "error: unknown weight mode: approx"),
        (["fit", "--response", str(y), "--family", "gaussian", "--out", out],
         "error: need --bspline or c*d --design files"),
        (["fit", "--response", str(y), "--family", "gaussian", "--bspline", "--design", str(tmp_path / "X1.csv"),
          "--design", str(tmp_path / "X1.csv"), "--out", out], "error: give either --design files or --bspline"),
        (["fit", "--response", str(y), "--family", "gaussian", "--design", str(tmp_path / "X1.csv"),
          "--design", str(tmp_path / "X2.csv"), "--out", out],
         "has 5 rows but dimension 2 needs 4"),
        (["predict", "--fit", str(tmp_path / "nofit"), "--out", out], "error: cannot open"),
    ]
    for argv, msg in cases:
        assert cli.main(argv) == cli.EXIT_ERROR, argv
        assert msg in capsys.readouterr().err
    (tmp_path / "notfit").mkdir()
    (tmp_path / "notfit" / "path.json").write_text('{"format": "other"}')
    assert cli.main(["predict", "--fit", str(tmp_path / "notfit"), "--out", out]) == cli.EXIT_ERROR
    assert "not a fit directory" in capsys.readouterr().err
    with pytest.raises(SystemExit):  # required option missing: argparse usage error
        cli.main(["fit", "--family", "gaussian", "--out", out])


def test_python_m_entry_point(tmp_path):
    r = subprocess.run([sys.executable, "-m", "paper_1510_03298_b200", "fit", "--response", "/nonexistent.glam",
                        "--bspline", "--family", "gaussian", "--out", str(tmp_path / "x")],
                       cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 1
    assert "error: cannot open /nonexistent.glam" in r.stderr


# ------------------------------------------------------------ CLI on the device
def _sim(tmp_path, family, seed, dims=(9, 6, 4), cols=(4, 3, 2)):
    """Stand-in for `kronglm simulate`: dense Gaussian factors, alternating
    decay coefficients (simulate.cpp's shape of data), seeded."""
    rng = np.random.default_rng(seed)
    sim = tmp_path / "sim"
    sim.mkdir(exist_ok=True)
    X = [rng.standard_normal((n, p)) / np.sqrt(p) for n, p in zip(dims, cols)]
    for j, x in enumerate(X):
        glamio.write_csv_matrix(sim / f"X{j + 1}.csv", x)
    p = int(np.prod(cols))
    theta = np.array([(-1) ** (i + 1) * np.exp(-0.1 * i) for i in range(p)]).reshape(cols, order="F")
    eta = theta
    for j, x in enumerate(X):
        eta = np.moveaxis(np.tensordot(x, eta, axes=([1], [j])), 0, j)
    if family == "poisson":
        y = rng.poisson(np.exp(0.5 * eta)).astype(float)
    else:
        y = eta + rng.standard_normal(eta.shape)
    glamio.write_array(sim / "response.glam", np.asfortranarray(y))
    glamio.write_array(sim / "weights.glam", np.asfortranarray(rng.uniform(0.5, 1.5, size=dims)))
    return sim, [str(sim / f"X{j + 1}.csv") for j in range(len(dims))]


def _designs(files):
    out = []
    for f in files:
        out += ["--design", f]
    return out


@pytest.mark.gpu
def test_cli_fit_forced_lambda_above_max_writes_zero(tmp_path):
    """test_io_cli.cpp:125-149."""
    sim, files = _sim(tmp_path, "gaussian", 3)
    base = ["fit", "--response", str(sim / "response.glam")] + _designs(files) + ["--family", "gaussian"]
    assert cli.main(base + ["--nlambda", "1", "--out", str(tmp_path / "probe")]) == 0
    lmax = json.load(open(tmp_path / "probe" / "path.json"))["lambda_max"]
    assert lmax > 0
    assert cli.main(base + ["--lambda", "%.17g" % (2 * lmax), "--out", str(tmp_path / "zero")]) == 0
    coef = glamio.read_array(tmp_path / "zero" / "coef_L000_C0.glam")
    assert coef.shape == (4, 3, 2)
    assert np.max(np.abs(coef)) == 0.0


@pytest.mark.gpu
def test_cli_fit_reproduces_library_fit_exactly(tmp_path):
    """test_io_cli.cpp:151-188: path.json and the coefficient files equal the
    library fit bit for bit; path.json carries main.cpp's keys."""
    from paper_1510_03298_b200 import kronglm as K
    sim, files = _sim(tmp_path, "poisson", 11)
    rc = cli.main(["fit", "--response", str(sim / "response.glam"), "--weights", str(sim / "weights.glam")]
                  + _designs(files) + ["--family", "poisson", "--nlambda", "7", "--lambda-min-ratio", "1e-2",
                                       "--out", str(tmp_path / "fit")])
    assert rc == 0
    meta = json.load(open(tmp_path / "fit" / "path.json"))
    assert sorted(meta) == sorted(["format", "version", "family", "link", "penalty", "alpha", "iwls", "nu",
                                   "lambda_max", "truncated", "response_dims", "n_components", "coef_dims",
                                   "design", "models"])
    assert (meta["format"], meta["version"], meta["family"], meta["link"], meta["penalty"], meta["iwls"]) == \
        ("kronglm-path", 1, "poisson", "log", "lasso", "exact")
    assert meta["response_dims"] == [9, 6, 4] and meta["coef_dims"] == [[4, 3, 2]] and meta["n_components"] == 1
    assert meta["design"] == {"kind": "csv", "files": files}
    D = K.Design([[glamio.read_csv_matrix(f) for f in files]])
    obs = K.Observation(D, glamio.read_array(sim / "response.glam"), glamio.read_array(sim / "weights.glam"))
    res = K.fit_path_resident(D, obs, "poisson", "lasso", 0.0, None, n_lambda=7, lambda_min_ratio=1e-2)
    assert len(meta["models"]) == 7 and res.n_models == 7
    coefs = res.coefs()
    for t, model in enumerate(meta["models"]):
        assert model["lambda"] == res.lambdas[t]
        assert model["objective"] == res.objectives[t]
        assert model["coef_files"] == ["coef_L%03d_C0.glam" % t]
        assert model["nonzero"] == int(np.count_nonzero(coefs[t]))
        coef = glamio.read_array(tmp_path / "fit" / model["coef_files"][0])
        assert np.array_equal(coef.reshape(-1, order="F"), coefs[t])
        assert model["converged"] is True


@pytest.mark.gpu
def test_cli_fit_invariant_to_masked_cells(tmp_path):
    """test_io_cli.cpp:190-220: zero-weight cells may hold anything."""
    sim, files = _sim(tmp_path, "gaussian", 5)
    y = glamio.read_array(sim / "response.glam")
    a = glamio.read_array(sim / "weights.glam")
    af, yf = a.reshape(-1, order="F").copy(), y.reshape(-1, order="F").copy()
    af[::3] = 0.0
    yf[::3] = 77.7
    glamio.write_array(sim / "mask_weights.glam", af.reshape(a.shape, order="F"))
    glamio.write_array(sim / "response_perturbed.glam", yf.reshape(y.shape, order="F"))
    for resp, out in (("response.glam", "fa"), ("response_perturbed.glam", "fb")):
        assert cli.main(["fit", "--response", str(sim / resp), "--weights", str(sim / "mask_weights.glam")]
                        + _designs(files) + ["--family", "gaussian", "--nlambda", "5",
                                             "--out", str(tmp_path / out)]) == 0
    for t in range(5):
        name = "coef_L%03d_C0.glam" % t
        assert _bytes(tmp_path / "fa" / name) == _bytes(tmp_path / "fb" / name)


@pytest.mark.gpu
def test_cli_predict_means_zero_model_and_mse_table(tmp_path, capsys):
    """test_io_cli.cpp:222-266, plus mse.tsv against the library's mse_heldout."""
    from paper_1510_03298_b200 import kronglm as K
    sim, files = _sim(tmp_path, "poisson", 19)
    assert cli.main(["fit", "--response", str(sim / "response.glam")] + _designs(files)
                    + ["--family", "poisson", "--nlambda", "6", "--lambda-min-ratio", "1e-2", "--save-mu",
                       "--out", str(tmp_path / "fit")]) == 0
    truth = glamio.read_array(sim / "response.glam")
    mask = np.zeros(truth.size)
    mask[::2] = 1.0
    mask = mask.reshape(truth.shape, order="F")
    glamio.write_array(tmp_path / "mask.glam", mask)
    capsys.readouterr()
    assert cli.main(["predict", "--fit", str(tmp_path / "fit"), "--truth", str(sim / "response.glam"),
                     "--mask", str(tmp_path / "mask.glam"), "--eta", "--out", str(tmp_path / "pred")]) == 0
    printed = capsys.readouterr().out
    mu0 = glamio.read_array(tmp_path / "pred" / "mu_L000.glam")
    assert np.all(mu0 == 1.0)
    assert np.max(np.abs(glamio.read_array(tmp_path / "pred" / "eta_L000.glam"))) == 0.0
    for t in range(6):  # predict reproduces fit --save-mu exactly
        assert _bytes(tmp_path / "pred" / ("mu_L%03d.glam" % t)) == _bytes(tmp_path / "fit" / ("mu_L%03d.glam" % t))
    lines = open(tmp_path / "pred" / "mse.tsv").read().splitlines()
    assert lines[0] == "model\tlambda\tmse\targmin"
    rows = [ln.split("\t") for ln in lines[1:]]
    assert len(rows) == 6 and sum(r[3] == "1" for r in rows) == 1
    # the same ranking through the library (device) held-out MSE
    D = K.Design([[glamio.read_csv_matrix(f) for f in files]])
    obs = K.Observation(D, truth)
    res = K.fit_path_resident(D, obs, "poisson", "lasso", 0.0, None, n_lambda=6, lambda_min_ratio=1e-2)
    lib = K.mse_heldout(res, "poisson", truth, mask)
    got = [float(r[2]) for r in rows]
    assert np.allclose(got, lib["mse"], rtol=1e-12, atol=0)
    arg = [int(r[0]) for r in rows if r[3] == "1"][0]
    assert arg == lib["argmin"]
    assert f"minimal held-out MSE at model {arg}" in printed


@pytest.mark.gpu
def test_cli_bspline_design_and_truncation_exit(tmp_path):
    """--bspline design reconstruction in predict (main.cpp:265-275) and the
    elastic-net / tensor-weight flags carried into path.json."""
    rng = np.random.default_rng(7)
    y = np.asfortranarray(rng.poisson(2.0, size=(20, 15)).astype(float))
    glamio.write_array(tmp_path / "y.glam", y)
    rc = cli.main(["fit", "--response", str(tmp_path / "y.glam"), "--bspline", "--basis-ratio", "4",
                   "--family", "poisson", "--penalty", "elastic_net", "--alpha", "0.3", "--iwls", "tensor_approx",
                   "--nlambda", "4", "--out", str(tmp_path / "fit")])
    assert rc in (cli.EXIT_OK, cli.EXIT_TRUNCATED)
    meta = json.load(open(tmp_path / "fit" / "path.json"))
    assert meta["design"] == {"kind": "bspline", "basis_ratio": 4, "order": 4}
    assert (meta["penalty"], meta["alpha"], meta["iwls"]) == ("elasticnet", 0.3, "tensor")
    assert meta["coef_dims"] == [[5, 5]]
    assert (rc == cli.EXIT_TRUNCATED) == meta["truncated"]
    assert cli.main(["predict", "--fit", str(tmp_path / "fit"), "--out", str(tmp_path / "pred")]) == 0
    assert len([f for f in os.listdir(tmp_path / "pred") if f.startswith("mu_L")]) == len(meta["models"])


# ------------------------------------------------------------ C++ io header
def test_cpp_io_header_matches_python(tmp_path):
    """include/kronglm_b200_io.hpp and glamio write the same bytes and raise the
    same messages (both restate io.cpp:91-212)."""
    exe = str(tmp_path / "io_roundtrip")
    subprocess.run(["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "io_roundtrip.cpp"), "-o", exe], check=True)
    rng = np.random.default_rng(104)
    glamio.write_array(tmp_path / "a.glam", np.asfortranarray(rng.standard_normal((3, 1, 5, 2))))
    assert subprocess.run([exe, "array", str(tmp_path / "a.glam"), str(tmp_path / "b.glam")]).returncode == 0
    assert _bytes(tmp_path / "a.glam") == _bytes(tmp_path / "b.glam")
    for name in ("X1.csv", "X2.csv"):
        assert subprocess.run([exe, "csv", os.path.join(GOLDEN, name), str(tmp_path / name)]).returncode == 0
        assert _bytes(tmp_path / name) == _bytes(os.path.join(GOLDEN, name))
    raw = _bytes(tmp_path / "a.glam")
    bad_arrays = {"m.glam": b"X" + raw[1:], "v.glam": raw[:4] + b"\x02" + raw[5:], "t.glam": raw[:-1],
                  "h.glam": raw[:9], "z.glam": b"GLAM\x01\x00\x00\x00"}
    bad_csv = {"a.csv": "1,2\n3;4\n", "b.csv": "1,x\n", "c.csv": "1,2\n3\n", "d.csv": "\n", "e.csv": "+1\n"}
    for files, mode, reader in ((bad_arrays, "err-array", glamio.read_array),
                                (bad_csv, "err-csv", glamio.read_csv_matrix)):
        for name, data in files.items():
            p = tmp_path / name
            p.write_bytes(data if isinstance(data, bytes) else data.encode())
            r = subprocess.run([exe, mode, str(p)], capture_output=True, text=True)
            assert r.returncode == 1
            with pytest.raises(RuntimeError) as e:
                reader(p)
            assert r.stdout.strip() == str(e.value), name
