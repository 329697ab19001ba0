"""One-sided Jacobi singular values (the kappa diagnostics, src/dense.py:365-415): the
pair-per-CTA kernel (default for columns up to 2048 rows) against the warp-per-pair
kernel and the oracle's restatement, including the NoConvergence outcome."""
import numpy as np
import pytest

from oracle import restatement as R

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sq():
    import paper_2603_16644_b200 as mod
    return mod


@pytest.mark.parametrize("n,kappa", [(64, 1e3), (300, 1e6), (1000, 1e2), (2048, 1e4)])
def test_cta_kernel_matches_warp_kernel(sq, monkeypatch, n, kappa):
    rs = R.philox(n, 7)
    u, _ = np.linalg.qr(rs.standard_normal((n, n)))
    v, _ = np.linalg.qr(rs.standard_normal((n, n)))
    a = np.linalg.qr((u * np.logspace(0, -np.log10(kappa), n)) @ v.T)[1]   # upper, singular values as given
    monkeypatch.setenv("SK_JACOBI", "cta")
    s_cta = sq.jacobi_singular_values(a)
    monkeypatch.setenv("SK_JACOBI", "warp")
    s_warp = sq.jacobi_singular_values(a)
    assert np.abs(s_cta - s_warp).max() <= 1e-12 * s_warp[0]
    assert abs(s_cta[0] / s_cta[-1] / (s_warp[0] / s_warp[-1]) - 1) <= 1e-9
    if n <= 300:
        ref = R.jacobi_sv(a)
        assert np.abs(s_cta - ref).max() <= 1e-12 * ref[0]


def test_cta_kernel_no_convergence(sq, monkeypatch):
    from paper_2603_16644_b200.errors import NoConvergence
    monkeypatch.setenv("SK_JACOBI", "cta")
    with pytest.raises(NoConvergence):
        sq.jacobi_singular_values(R.philox(5, 3).standard_normal((64, 64)), max_sweeps=1, tol=1e-300)
