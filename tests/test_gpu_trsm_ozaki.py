"""Blocked TRSM with INT8 (Ozaki scheme II) off-diagonal updates (sk_trsm_ozaki_f64)
against the one-kernel FP64 DMMA solve (sk_trsm_right_upper_f64, itself checked
against the oracle in test_gpu_kernels.py).

The blocked solve is the standard right-looking split A_p[:, h:] = (A[:, h:] -
A_p[:, :h] R[:h, h:]) R[h:, h:]^-1; the update's only rounding is the t-bit scaling
(row scales for A_p, column scales for R), an FP64 GEMM's error size.  Asserted: the
backward residual ||A_p R - A|| / (||A_p|| ||R||) is within 4x of the DMMA solve's
(or 1e-15), and the two solutions agree to the conditioning of R."""
import numpy as np
import pytest

from oracle import restatement as R

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch as t
    return t


def _solve(torch, a, r, engine):
    from paper_2603_16644_b200.dense import _trsm
    return _trsm(a, r, engine=engine)


def _fell_back():
    from paper_2603_16644_b200 import _lib
    return _lib.lib().sk_trsm_ozaki_fell_back() == 1


def _backward(torch, a, r, ap):
    res = torch.linalg.matrix_norm(ap @ r - a)
    return float(res / (torch.linalg.matrix_norm(ap) * torch.linalg.matrix_norm(r)))


@pytest.mark.parametrize("m,n", [(5000, 2048), (70000, 1500), (3000, 2600), (1000, 1100), (257, 1300)])
def test_blocked_trsm_random(torch, m, n):
    g = R.philox(m + 3 * n, 17)
    a = torch.from_numpy(g.standard_normal((m, n))).cuda()
    r = torch.from_numpy(np.triu(g.standard_normal((n, n))) + 8 * np.eye(n)).cuda()
    ap_oz = _solve(torch, a, r, "ozaki")
    assert not _fell_back()
    ap_dm = _solve(torch, a, r, "dmma")
    b_oz, b_dm = _backward(torch, a, r, ap_oz), _backward(torch, a, r, ap_dm)
    assert b_oz <= max(4 * b_dm, 1e-15), (b_oz, b_dm)
    rel = float((ap_oz - ap_dm).abs().max() / ap_dm.abs().max())
    assert rel < 1e-12, rel


@pytest.mark.parametrize("kappa", [1e4, 1e10, 1e14])
def test_blocked_trsm_ill_conditioned(torch, kappa):
    """R of a graded, ill-conditioned matrix (what the sketch QR produces)."""
    m, n = 20000, 1280
    g = R.philox(int(np.log10(kappa)), 19)
    u, _ = np.linalg.qr(g.standard_normal((3 * n, n)))
    v, _ = np.linalg.qr(g.standard_normal((n, n)))
    s = np.logspace(0, -np.log10(kappa), n)
    rr = np.linalg.qr((u * s) @ v.T, mode="r")
    a = torch.from_numpy(g.standard_normal((m, n)) @ ((s[:, None] * v.T))).cuda()
    r = torch.from_numpy(np.ascontiguousarray(rr)).cuda()
    ap_oz = _solve(torch, a, r, "ozaki")
    assert not _fell_back()
    ap_dm = _solve(torch, a, r, "dmma")
    b_oz, b_dm = _backward(torch, a, r, ap_oz), _backward(torch, a, r, ap_dm)
    assert b_oz <= max(4 * b_dm, 1e-15), (b_oz, b_dm)
    # forward: both are kappa(R) u away from the exact A R^-1
    rel = float(torch.linalg.matrix_norm(ap_oz - ap_dm) / torch.linalg.matrix_norm(ap_dm))
    assert rel < 1e3 * kappa * 1.1e-16 + 1e-13, rel


def test_blocked_trsm_guard(torch):
    """A non-finite entry of A_p or of R's off-diagonal block re-runs the whole solve on
    the DMMA kernel: bitwise the DMMA result.  (The spikiness test max sqrt(h) > 64
    ||row|| cannot fire below h = 4096; a dominant entry only moves the scale, and the
    bound stays 2^-t max|row| sum|col| <= 2^-t ||row|| ||col||_1.)"""
    m, n = 4000, 1536
    g = R.philox(5, 23)
    a = g.standard_normal((m, n))
    a[123, 7] = 1e6
    r = np.triu(g.standard_normal((n, n))) + 8 * np.eye(n)
    at, rt = torch.from_numpy(a).cuda(), torch.from_numpy(r).cuda()
    ap_oz = _solve(torch, at, rt, "ozaki")
    assert not _fell_back()
    ap_dm = _solve(torch, at, rt, "dmma")
    assert _backward(torch, at, rt, ap_oz) <= max(4 * _backward(torch, at, rt, ap_dm), 1e-15)
    r2 = r.copy()
    r2[5, 1000] = np.inf
    r2t = torch.from_numpy(r2).cuda()
    ap_oz = _solve(torch, at, r2t, "ozaki")
    assert _fell_back()
    ap_dm = _solve(torch, at, r2t, "dmma")
    assert torch.equal(torch.isnan(ap_oz), torch.isnan(ap_dm))
    fin = torch.isfinite(ap_dm)
    assert torch.equal(ap_oz[fin], ap_dm[fin])
    a[123, 7] = np.nan
    at = torch.from_numpy(a).cuda()
    ap_oz = _solve(torch, at, rt, "ozaki")
    assert _fell_back()
    ap_dm = _solve(torch, at, rt, "dmma")
    assert torch.equal(torch.isnan(ap_oz), torch.isnan(ap_dm))
    fin = torch.isfinite(ap_dm)
    assert torch.equal(ap_oz[fin], ap_dm[fin])


def test_blocked_trsm_zero_diagonal(torch):
    import paper_2603_16644_b200 as sq
    n = 1300
    r = np.triu(np.random.default_rng(1).standard_normal((n, n))) + 8 * np.eye(n)
    r[1200, 1200] = 0.0
    a = torch.ones((2000, n), dtype=torch.float64, device="cuda")
    with pytest.raises(sq.SingularTriangular):
        _solve(torch, a, torch.from_numpy(r).cuda(), "ozaki")


@pytest.fixture
def int8_trsm(monkeypatch):
    from paper_2603_16644_b200 import dense
    monkeypatch.setattr(dense, "TRSM_ENGINE", "ozaki")
    return dense


@pytest.mark.parametrize("kappa", [1e1, 1e6, 1e12])
@pytest.mark.parametrize("method", ["pne", "hpne"])
def test_pipeline_on_blocked_trsm(int8_trsm, torch, kappa, method):
    """Algorithm 1 end to end with the blocked INT8 TRSM: same level and an error within
    2x (+1e-15) of the same pipeline on the DMMA TRSM."""
    import paper_2603_16644_b200 as sq
    from paper_2603_16644_b200.probgen import generate_problem_device
    a, b, xs = generate_problem_device(24000, 1280, kappa, 1e-6, R.mix64(7, int(np.log10(kappa))),
                                       torch.device("cuda"))
    oz = sq.algorithm1_pipeline(a, b, method, "auto", 3.0, "dct2", 0, xs, diagnostics=False)
    int8_trsm.TRSM_ENGINE = "dmma"
    dm = sq.algorithm1_pipeline(a, b, method, "auto", 3.0, "dct2", 0, xs, diagnostics=False)
    assert oz.preconditioner.computed_in == dm.preconditioner.computed_in
    assert oz.relative_error <= 2 * dm.relative_error + 1e-15, (oz.relative_error, dm.relative_error)
