"""Harness, CLI, archive and bound formulas, against fixtures produced by
the real reference (tests/golden/make_golden_harness.py).  The reference's own tests
(tests/test_harness.py, tests/test_cli.py, tests/test_bounds.py) are the model: CPU tests
cover the host logic (formulas, grids, validation, CSV, archives, exit codes), GPU tests
run the sweeps / commands through libsklsq and compare the rows with the reference's."""

import csv
import hashlib
import json
import math
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_2603_16644_b200 as sq
from paper_2603_16644_b200 import bounds as B
from paper_2603_16644_b200 import errors as E
from paper_2603_16644_b200.cli import main
from paper_2603_16644_b200.harness import BENCH_COLUMNS, CSV_COLUMNS, write_csv

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "harness_golden.json")))
ARCHIVE = os.path.join(HERE, "golden", "archive_ref")


def _outcome(fn):
    try:
        return {"value": fn()}
    except Exception as ex:  # noqa: BLE001
        return {"raises": type(ex).__name__}


# ------------------------------------------------------------------ CPU -----
@pytest.mark.parametrize("case", sorted(GOLD["bounds"]))
def test_bound_formulas_match_reference(case):
    spec = GOLD["bounds"][case]
    bi = B.BoundInputs(**spec["inputs"])
    got = {
        "bound_ls": _outcome(lambda: B.bound_ls(bi)),
        "bound_ne_family": _outcome(lambda: B.bound_ne_family(bi)),
        "bound_ne_family_seminormal": _outcome(lambda: B.bound_ne_family(bi, "seminormal")),
        "bound_ne_family_bad": _outcome(lambda: B.bound_ne_family(bi, "other")),
        "bound_pne_old": _outcome(lambda: B.bound_pne(bi, "old")),
        "bound_pne_new": _outcome(lambda: B.bound_pne(bi, "new")),
        "bound_pne_bad": _outcome(lambda: B.bound_pne(bi, "x")),
        "bound_hpne_old": _outcome(lambda: B.bound_hpne(bi, "old")),
        "bound_hpne_new": _outcome(lambda: B.bound_hpne(bi, "new")),
        "bound_notnormal": _outcome(lambda: B.bound_notnormal(bi, 12.5, 1.1)),
        "eta1": _outcome(lambda: B.eta1(bi.kappa_rs, bi.u1) if bi.kappa_rs is not None else None),
    }
    assert got == spec["results"]     # bitwise: same formulas, same operation order


def test_rho_grid_and_sample_size_match_reference():
    for key, vals in GOLD["rho_grid"].items():
        lo, hi, pts = key.split(",")
        assert sq.rho_grid(float(lo), float(hi), int(pts)).tolist() == vals
    for key, val in GOLD["sample_size"].items():
        m, n, mu, eps, dl = key.split(",")
        assert sq.sample_size_lower_bound(sq.EmbeddingParams(int(m), int(n), float(mu), float(eps), float(dl))) == val
    with pytest.raises(ValueError):
        sq.rho_grid(1e-2, 1e-8, 3)
    with pytest.raises(ValueError):
        sq.rho_grid(1e-8, 1e-2, 0)
    with pytest.raises(ValueError):
        sq.EmbeddingParams(10, 20, 0.5, 0.5, 0.1)
    with pytest.raises(ValueError):
        sq.EmbeddingParams(100, 20, 0.1, 0.5, 0.1)   # mu below n/m


def _cfg(**overrides):
    base = dict(m=120, n=10, kappa=1e3, rho_grid=sq.rho_grid(1e-10, 1e-2, 3), methods=("qr", "pne", "hpne"),
                precision="double", trials_per_point=2, seed=17)
    base.update(overrides)
    return sq.SweepConfig(**base)


def test_sweep_config_validation():
    with pytest.raises(ValueError):
        _cfg(methods=("qr", "bogus"))
    with pytest.raises(ValueError):
        _cfg(precision="quad")
    with pytest.raises(ValueError):
        _cfg(trials_per_point=0)
    with pytest.raises(ValueError):
        _cfg(rho_grid=np.array([1e-2, 1e-8]))
    with pytest.raises(ValueError):
        _cfg(methods=())
    with pytest.raises(ValueError):
        _cfg(transform="fft")
    assert _cfg(precision="auto").precision == "auto"


def test_write_csv_roundtrip(tmp_path):
    rows = [dict({c: "" for c in CSV_COLUMNS}, method="qr", m=5, rel_error=0.1 + 0.2, seed=2 ** 63 + 5, trial=0),
            dict({c: "" for c in CSV_COLUMNS}, method="ne", error="NotPositiveDefinite: pivot 3")]
    path = tmp_path / "s.csv"
    write_csv(path, rows, CSV_COLUMNS)
    with open(path, newline="") as fh:
        got = list(csv.DictReader(fh))
    assert list(got[0].keys()) == CSV_COLUMNS
    assert float(got[0]["rel_error"]) == 0.1 + 0.2     # repr round trip is exact
    assert int(got[0]["seed"]) == 2 ** 63 + 5
    assert got[1]["error"].startswith("NotPositiveDefinite") and got[1]["rel_error"] == ""


def test_reference_archive_loads_bitwise():
    p = sq.load_problem(ARCHIVE)
    want = json.load(open(os.path.join(HERE, "golden", "archive_ref_sha.json")))
    for k in ("a", "b", "x_star"):
        assert hashlib.sha256(np.ascontiguousarray(getattr(p, k)).tobytes()).hexdigest() == want[k]
    assert (p.m, p.n, p.kappa, p.rho, p.seed) == (40, 6, 1e3, 1e-6, 5)


@pytest.mark.parametrize("mode", ["mtx", "npy", "both"])
def test_archive_roundtrip(tmp_path, mode):
    rs = np.random.default_rng(3)
    p = sq.LeastSquaresProblem(a=rs.standard_normal((30, 4)) * 10.0 ** rs.integers(-300, 300, (30, 4)),
                               b=rs.standard_normal(30), x_star=rs.standard_normal(4), rho=1e-6, kappa=1e3, seed=9)
    d = tmp_path / mode
    sq.save_problem(p, d, sidecar=mode != "mtx", mtx=mode != "npy")
    assert (d / "A.npy").exists() == (mode != "mtx")
    assert (d / "A.mtx").exists() == (mode != "npy")
    q = sq.load_problem(d)
    for k in ("a", "b", "x_star"):
        assert np.array_equal(np.asarray(getattr(q, k)), getattr(p, k))
    assert (q.kappa, q.rho, q.seed) == (p.kappa, p.rho, p.seed)
    meta = json.load(open(d / "meta.json"))
    assert meta["format_version"] == 1
    with pytest.raises(ValueError):
        sq.save_problem(p, tmp_path / "none", sidecar=False, mtx=False)


def test_archive_rejects_bad_version_and_shape(tmp_path):
    import shutil
    d = tmp_path / "arch"
    shutil.copytree(ARCHIVE, d)
    meta = json.load(open(d / "meta.json"))
    json.dump(dict(meta, m=41), open(d / "meta.json", "w"))
    with pytest.raises(ValueError):
        sq.load_problem(d)
    json.dump(dict(meta, format_version=2), open(d / "meta.json", "w"))
    with pytest.raises(ValueError):
        sq.load_problem(d)


def test_mmio_forms(tmp_path):
    from paper_2603_16644_b200.mmio import read_matrix, read_vector, write_matrix
    a = np.array([[1.5, -2.0], [0.0, 3.25], [4.0, 1e-8]])
    write_matrix(tmp_path / "a.mtx", a)
    assert np.array_equal(read_matrix(tmp_path / "a.mtx"), a)
    text = tmp_path / "ints.mtx"
    text.write_text("%%MatrixMarket matrix array real general\n2 2\n1\n2\n3e0\n-4.5e-1\n")
    assert np.array_equal(read_matrix(text), np.array([[1.0, 3.0], [2.0, -0.45]]))
    with pytest.raises(ValueError):
        read_vector(tmp_path / "a.mtx")
    with pytest.raises(ValueError):
        write_matrix(tmp_path / "c.mtx", np.zeros((2, 2, 2)))


def test_cli_argument_errors_exit_two(tmp_path):
    with pytest.raises(SystemExit) as exc:
        main(["solve", "--problem", "x", "--method", "cgls"])
    assert exc.value.code == 2
    assert main(["solve", "--problem", str(tmp_path / "missing")]) == 2
    assert main(["gen", "--m", "10", "--n", "20", "--out", str(tmp_path / "bad")]) == 2
    assert main(["--device", "cpu", "gen", "--m", "10", "--n", "2", "--out", str(tmp_path / "b2")]) == 2
    # nne without --b-matrix is rejected after loading the archive, before any device work
    assert main(["solve", "--problem", ARCHIVE, "--method", "nne"]) == 2


def test_cli_module_entry_and_version():
    root = os.path.dirname(HERE)
    r = subprocess.run([sys.executable, "-m", "paper_2603_16644_b200", "--version"], cwd=root, capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.strip() == sq.__version__


# ------------------------------------------------------------------ GPU -----
def _close(a, b, rel):
    return abs(a - b) <= rel * max(abs(a), abs(b))


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(GOLD["sweeps"]))
def test_sweep_rows_match_reference(name):
    spec = GOLD["sweeps"][name]
    cfg = dict(spec["config"])
    cfg["rho_grid"] = np.array(cfg["rho_grid"])
    cfg["methods"] = tuple(cfg["methods"])
    rows = sq.run_sweep(sq.SweepConfig(**cfg))
    ref = spec["rows"]
    assert len(rows) == len(ref)
    for got, want in zip(rows, ref):
        assert list(got.keys()) == CSV_COLUMNS
        for k in ("method", "m", "n", "kappa", "rho", "precision", "d", "seed", "trial"):
            assert got[k] == want[k], (k, got[k], want[k])
        # same outcome class (the exception name), empty exactly where the reference's is.
        # Exception: the normal equations past the binary64 frontier (kappa^2 u >> 1, the
        # "failure" sweep: kappa 1e9) break down on rounding noise (pivot ~ -u ||G||), so
        # whether a pivot lands below zero depends on the Gram's summation order; there
        # either outcome is the reference's behaviour up to rounding.
        frontier = got["method"] == "ne" and got["kappa"] ** 2 * 2.0 ** -53 > 1.0
        if frontier and (got["error"] == "") != (want["error"] == ""):
            assert got["error"] in ("",) or got["error"].startswith("NotPositiveDefinite"), got["error"]
            continue
        assert got["error"].split(":")[0] == want["error"].split(":")[0], (got["error"], want["error"])
        for k in CSV_COLUMNS:
            if k in ("wall_ms", "error"):
                continue
            assert (got[k] == "") == (want[k] == ""), (k, got[k], want[k])
        if want["error"]:
            continue
        assert got["wall_ms"] > 0.0
        assert got["rel_error"] <= max(10 * want["rel_error"], 1e-14), (got["method"], got["rel_error"], want["rel_error"])
        assert _close(got["rel_residual"], want["rel_residual"], 1e-3)
        for k in ("kappa_ap", "kappa_rs"):
            if want[k] != "":
                assert _close(got[k], want[k], 5e-2), (k, got[k], want[k])
        # bounds: same formulas on device-measured inputs (kappas, residual ratios)
        for k in ("bound_ls", "bound_ne", "bound_pne_old", "bound_pne_new", "bound_hpne_old", "bound_hpne_new"):
            if want[k] != "":
                assert got[k] > 0.0 and _close(got[k], want[k], 0.5), (k, got[k], want[k])


@pytest.mark.gpu
def test_sweep_deterministic_up_to_timing():
    strip = lambda rows: [{k: v for k, v in r.items() if k != "wall_ms"} for r in rows]  # noqa: E731
    cfg = _cfg(trials_per_point=1)
    assert strip(sq.run_sweep(cfg)) == strip(sq.run_sweep(cfg))


@pytest.mark.gpu
def test_benchmark_rows(tmp_path):
    spec = GOLD["benchmark"]
    path = tmp_path / "bench.csv"
    rows = sq.run_benchmark(**{**spec["args"], "n_list": tuple(spec["args"]["n_list"])}, output_path=path)
    assert len(rows) == len(spec["rows"])
    for got, want in zip(rows, spec["rows"]):
        assert list(got.keys()) == BENCH_COLUMNS
        for k in ("method", "m", "n", "kappa", "trials"):
            assert got[k] == want[k]
        assert got["median_wall_ms"] > 0 and got["speedup_vs_qr"] > 0
        assert got["rel_error"] <= max(10 * want["rel_error"], 1e-14)
    assert path.exists()


@pytest.mark.gpu
def test_cli_end_to_end(tmp_path, capsys):
    path = tmp_path / "prob"
    assert main(["gen", "--m", "200", "--n", "12", "--kappa", "1e3", "--rho", "1e-6", "--seed", "5",
                 "--out", str(path)]) == 0
    p = sq.load_problem(path)
    assert p.m == 200 and p.n == 12 and abs(np.linalg.norm(p.x_star) - 1.0) <= 1e-14
    for method in ("qr", "ne", "sne", "pne", "hpne"):
        assert main(["solve", "--problem", str(path), "--method", method]) == 0
    out = capsys.readouterr().out
    assert "rel error vs x*" in out and "bound (new form)" in out and "hpne" in out
    # the reference-written archive, auto precision and nne through both B forms
    assert main(["solve", "--problem", ARCHIVE, "--precision", "auto", "--method", "hpne"]) == 0
    bpath = tmp_path / "bmat.mtx"
    from paper_2603_16644_b200.mmio import write_matrix
    write_matrix(bpath, p.a)
    assert main(["solve", "--problem", str(path), "--method", "nne", "--b-matrix", str(bpath)]) == 0
    assert main(["solve", "--problem", str(path), "--method", "nne", "--b-matrix", str(path)]) == 0
    # numerical failure -> 3
    hard = tmp_path / "hard"   # kappa^2 u ~ 1e8: the Gram is indefinite far beyond rounding noise
    assert main(["gen", "--m", "400", "--n", "30", "--kappa", "1e12", "--rho", "1e-6", "--seed", "1",
                 "--out", str(hard)]) == 0
    assert main(["solve", "--problem", str(hard), "--method", "ne"]) == 3
    # sweep / bench CSVs
    out_csv = tmp_path / "sweep.csv"
    assert main(["sweep", "--m", "150", "--n", "10", "--kappa", "1e3", "--rho-min", "1e-8", "--rho-max", "1e-4",
                 "--rho-points", "2", "--methods", "qr,pne", "--trials", "1", "--seed", "2", "--csv",
                 str(out_csv)]) == 0
    with open(out_csv, newline="") as fh:
        rows = list(csv.DictReader(fh))
    assert list(rows[0].keys()) == CSV_COLUMNS and len(rows) == 4
    bench_csv = tmp_path / "bench.csv"
    assert main(["bench", "--m", "150", "--n-list", "8,10", "--kappa", "1e3", "--trials", "1", "--seed", "2",
                 "--csv", str(bench_csv)]) == 0
    with open(bench_csv, newline="") as fh:
        rows = list(csv.DictReader(fh))
    assert list(rows[0].keys()) == BENCH_COLUMNS and len(rows) == 6
    # .npy sidecar archive without text files
    big = tmp_path / "npy"
    assert main(["gen", "--m", "300", "--n", "16", "--seed", "3", "--npy", "--no-mtx", "--out", str(big)]) == 0
    assert not (big / "A.mtx").exists() and (big / "A.npy").exists()
    assert main(["solve", "--problem", str(big), "--method", "pne"]) == 0


@pytest.mark.gpu
def test_coherence_on_device():
    q = sq.random_orthogonal_columns(500, 8, 4)
    mu = sq.coherence(q)
    assert math.isclose(mu, float(np.einsum("ij,ij->i", q, q).max()), rel_tol=1e-12)
    with pytest.raises(E.NotOrthonormal):
        sq.coherence(q * 1.01)
