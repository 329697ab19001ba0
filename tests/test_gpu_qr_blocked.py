"""Blocked (WY) level QR for binary32 / binary64 (64-column panels factored by the
dataflow kernel, trailing columns updated with V T^T V^T): R against the oracle's
restatement of householder_reduce in the level precision (src/dense.py:108-161; the
reference's order there is BLAS-defined, src/precision.py:181-187), against the
column-at-a-time kernel (SK_QR_BLOCKED=0), the reference's sign convention, Q, and
RankDeficient raised at the right column in a later panel."""
import numpy as np
import pytest

from oracle import restatement as R

pytestmark = pytest.mark.gpu

TOL = {"binary32": 2e-5, "binary64": 1e-13}


@pytest.fixture(scope="module")
def sq():
    import paper_2603_16644_b200 as mod
    return mod


@pytest.fixture(autouse=True, params=["cluster+lookahead", "cluster", "flow-panels"])
def blocked_everywhere(request, monkeypatch):
    """every panel path: cluster panels with the side-stream lookahead (default), cluster
    panels in order (SK_QR_LOOKAHEAD=0), dataflow-kernel panels (SK_QR_PANEL=flow)"""
    monkeypatch.setenv("SK_QR_BLOCKED", "1")
    if request.param == "cluster":
        monkeypatch.setenv("SK_QR_LOOKAHEAD", "0")
    elif request.param == "flow-panels":
        monkeypatch.setenv("SK_QR_PANEL", "flow")


@pytest.mark.parametrize("level", ["binary32", "binary64"])
@pytest.mark.parametrize("d,n", [(70, 65), (200, 129), (300, 100), (600, 200), (1500, 257), (3000, 1000)])
def test_blocked_r_matches_oracle(sq, level, d, n):
    a = R.philox(d + n, 11).standard_normal((d, n)) * np.logspace(0, -2, n)
    lev = getattr(sq, level.upper())
    got = sq.qr_in_precision(a, lev)
    dt = np.float32 if level == "binary32" else np.float64
    ref_r = R.householder_steps(a.astype(dt))[2].astype(np.float64)
    scale = np.abs(ref_r).max()
    assert np.abs(got.r - ref_r).max() <= TOL[level] * scale
    assert np.array_equal(np.sign(np.diagonal(got.r)), np.sign(np.diagonal(ref_r)))   # alpha = -sign(x0) |x|
    # Q: orthonormal columns, Q R = A to the level's roundoff
    q = got.q
    assert np.abs(q.T @ q - np.eye(n)).max() <= 50 * TOL[level]
    assert np.abs(q @ got.r - a).max() <= 50 * TOL[level] * np.abs(a).max()


@pytest.mark.parametrize("level", ["binary32", "binary64"])
def test_blocked_matches_unblocked_kernel(sq, monkeypatch, level):
    a = R.philox(7, 3).standard_normal((6144, 2048))
    lev = getattr(sq, level.upper())
    blocked = sq.qr_in_precision(a[:, :700], lev).r
    monkeypatch.setenv("SK_QR_BLOCKED", "0")
    plain = sq.qr_in_precision(a[:, :700], lev).r
    assert np.abs(blocked - plain).max() <= TOL[level] * np.abs(plain).max()


@pytest.mark.parametrize("level", ["binary32", "binary64"])
def test_blocked_rank_deficient_in_a_later_panel(sq, level):
    a = R.philox(9, 4).standard_normal((500, 150))
    a[:, 100] = 0.0            # stays exactly zero under every reflector: norm 0 at column 100
    with pytest.raises(sq.RankDeficient, match="100"):
        sq.qr_in_precision(a, getattr(sq, level.upper()))


@pytest.mark.parametrize("level", ["binary32", "binary64"])
def test_small_panels_rank_deficient_and_sign(sq, level):
    """config-1-sized sketches (every panel on the register-resident one-CTA kernel):
    RankDeficient at the right column of a later panel, the reference's signs."""
    a = R.philox(5, 6).standard_normal((300, 120))
    a[:, 70] = 0.0
    with pytest.raises(sq.RankDeficient, match="70"):
        sq.qr_in_precision(a, getattr(sq, level.upper()))
    a = R.philox(5, 7).standard_normal((330, 96)) * np.logspace(0, -3, 96)
    got = sq.qr_in_precision(a, getattr(sq, level.upper()))
    dt = np.float32 if level == "binary32" else np.float64
    ref_r = R.householder_steps(a.astype(dt))[2].astype(np.float64)
    assert np.abs(got.r - ref_r).max() <= TOL[level] * np.abs(ref_r).max()
    assert np.array_equal(np.sign(np.diagonal(got.r)), np.sign(np.diagonal(ref_r)))
