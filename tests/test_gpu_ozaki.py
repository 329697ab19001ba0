"""INT8 tensor-core (Ozaki scheme II) FP64 Gram against an extended-precision
reference and against the FP64 DMMA Gram.

Bound checked: the engine's only rounding is the per-column t-bit scaling, so
|G - X^T Y|_ij <= 2^-t (2^e_i sum|Y_j| + 2^f_j sum|X_i|) / 2 + one final rounding;
we assert the looser "no worse than 4x the DMMA GEMM's error, or 1e-15 of |X|^T|Y|"."""
import numpy as np
import pytest

from oracle import restatement as R

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch as t
    return t


def _exact(x, y):
    xl, yl = x.astype(np.longdouble), y.astype(np.longdouble)
    return xl.T @ yl


def _check(torch, x, y, syrk):
    from paper_2603_16644_b200.dense import _gram
    xt = torch.from_numpy(x).cuda()
    yt = xt if syrk else torch.from_numpy(y).cuda()
    g_oz = _gram(xt, None if syrk else yt, engine="ozaki").cpu().numpy()
    g_dm = _gram(xt, None if syrk else yt, engine="dmma").cpu().numpy()
    ex = _exact(x, x if syrk else y)
    absb = (np.abs(x).T @ np.abs(x if syrk else y))
    e_oz = float(np.max(np.abs(g_oz - ex) / np.maximum(absb, 1e-300)))
    e_dm = float(np.max(np.abs(g_dm - ex) / np.maximum(absb, 1e-300)))
    assert np.all(np.isfinite(g_oz))
    assert e_oz <= max(4 * e_dm, 1e-15), (e_oz, e_dm)
    if syrk:
        assert np.array_equal(g_oz, g_oz.T)
    return e_oz, e_dm


@pytest.mark.parametrize("m,n,syrk", [(1000, 128, True), (1000, 128, False), (5000, 300, True),
                                      (5000, 300, False), (6000, 520, False), (300000, 24, True),
                                      (300000, 20, False), (77, 256, False)])
def test_ozaki_gram_random(torch, m, n, syrk):
    g = R.philox(m + 7 * n, 3)
    x = g.standard_normal((m, n))
    y = g.standard_normal((m, n))
    _check(torch, x, y, syrk)


def _fell_back():
    from paper_2603_16644_b200 import _lib
    return _lib.lib().sk_gram_ozaki_fell_back() == 1


def test_ozaki_gram_scaled_columns_and_rows(torch):
    g = R.philox(11, 3)
    m, n = 40000, 200
    x = g.standard_normal((m, n)) * (10.0 ** g.uniform(-8, 8, n))[None, :]
    y = g.standard_normal((m, n)) * (10.0 ** g.uniform(-8, 8, n))[None, :]
    _check(torch, x, x, True)          # column scales: per-column exponents absorb them
    assert not _fell_back()
    _check(torch, x, y, False)
    assert not _fell_back()
    xr = x * (10.0 ** g.uniform(-3, 3, m))[:, None]
    _check(torch, xr, xr, True)        # rows spanning 1e6: the top decade carries the norm,
    assert not _fell_back()            # max sqrt(m) / ||x|| ~ 15 < 64: stays on INT8, accurate
    xs = x * np.where(np.arange(m) % 1000 == 0, 1e4, 1.0)[:, None]
    _check(torch, xs, xs, True)        # 40 rows 1e4 above the rest: spiky -> FP64 fallback
    assert _fell_back()


def test_ozaki_guard_spiky_and_non_finite(torch):
    from paper_2603_16644_b200.dense import _gram
    g = R.philox(12, 3)
    m, n = 20000, 130
    x = g.standard_normal((m, n))
    xt = torch.from_numpy(x).cuda()
    _gram(xt, engine="ozaki")
    assert not _fell_back()
    x[17, 3] = 1e6                      # one outlier: max sqrt(m) >> ||x||
    xt = torch.from_numpy(x).cuda()
    got = _gram(xt, engine="ozaki")
    assert _fell_back()
    assert torch.equal(got, _gram(xt, engine="dmma"))
    x[17, 3] = np.nan
    got = _gram(torch.from_numpy(x).cuda(), engine="ozaki").cpu().numpy()
    assert _fell_back() and np.isnan(got[3, 3])


@pytest.fixture
def int8_gram(monkeypatch):
    """Every Gram of the solvers on the INT8 engine, whatever its size."""
    from paper_2603_16644_b200 import dense
    monkeypatch.setattr(dense, "GRAM_ENGINE", "ozaki")


def _golden_keys():
    from tests.golden_data import META
    return sorted(META["runs"])


@pytest.mark.parametrize("key", _golden_keys())
def test_pipeline_golden_runs_on_int8_gram(int8_gram, key):
    """The reference's golden pipeline runs (level, escalation, error, kappa0) hold with
    the kappa0 SYRK and the PNE / HPNE Grams on the INT8 engine."""
    import paper_2603_16644_b200 as sq
    from tests.test_gpu_pipeline import test_pipeline_vs_reference_runs
    test_pipeline_vs_reference_runs(sq, key)


@pytest.mark.parametrize("kappa", [1e2, 1e6, 1e10, 1e14])
@pytest.mark.parametrize("rho", [1e-14, 1e-6, 1e-1])
def test_config5_grid_on_int8_gram(int8_gram, kappa, rho):
    import paper_2603_16644_b200 as sq
    from tests.test_gpu_configs import test_config5_grid_scaled
    test_config5_grid_scaled(sq, kappa, rho)


def test_ozaki_gram_special_values(torch):
    from paper_2603_16644_b200.dense import _gram
    m, n = 3000, 130
    x = np.zeros((m, n))
    x[:, 5] = 1.0                      # constant column
    x[7, 9] = -3.5                     # a single entry
    x[:, 20] = R.philox(1, 3).standard_normal(m)
    g_oz = _gram(torch.from_numpy(x).cuda(), engine="ozaki").cpu().numpy()
    ref = x.T @ x
    exact = np.ones((n, n), dtype=bool)
    exact[20, :] = exact[:, 20] = False
    assert np.array_equal(g_oz[exact], ref[exact])   # zeros, small integers, single products
    assert abs(g_oz[20, 20] - ref[20, 20]) <= 1e-15 * ref[20, 20]
    assert abs(g_oz[5, 20] - ref[5, 20]) <= 1e-15 * np.abs(x[:, 20]).sum()


@pytest.mark.parametrize("syrk", [True, False])
def test_ozaki_gram_fewest_moduli(torch, syrk):
    """m >= 2^21 rows: gram_moduli picks 15 moduli, t = 47 (worst case 2^-40 ||X_i||
    ||Y_j||, 2^8 under the FP64 GEMM's gamma_K).  Against the DMMA Gram the difference
    stays at the FP64 GEMM's own error level, far inside that bound."""
    from paper_2603_16644_b200.dense import _gram
    m, n = (1 << 21) + 3, 200
    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    x = torch.randn(m, n, dtype=torch.float64, device="cuda", generator=g)
    x[:, 7] *= 1e-6                      # a scaled column (its own scale)
    y = x if syrk else torch.randn(m, n, dtype=torch.float64, device="cuda", generator=g)
    g_oz = _gram(x, None if syrk else y, engine="ozaki")
    g_dm = _gram(x, None if syrk else y, engine="dmma")
    nx, ny = x.norm(dim=0), y.norm(dim=0)
    rel = ((g_oz - g_dm).abs() / (nx[:, None] * ny[None, :])).max().item()
    assert rel <= 2.0 ** -40, rel
    if syrk:
        assert torch.equal(g_oz, g_oz.T)


def test_pipeline_fewest_moduli_matches_dmma(torch, monkeypatch):
    """Algorithm 1 at 2^21 rows (15-modulus Grams) against the same pipeline with every
    Gram on FP64 DMMA: same level, error within 2x (+1e-15)."""
    import paper_2603_16644_b200 as sq
    from paper_2603_16644_b200 import dense
    from paper_2603_16644_b200.probgen import generate_problem_device
    for kappa in (1e1, 1e6):
        a, b, xs = generate_problem_device((1 << 21) + 64, 256, kappa, 1e-6, R.mix64(9, int(np.log10(kappa))),
                                           torch.device("cuda"))
        monkeypatch.setattr(dense, "GRAM_ENGINE", "ozaki")
        oz = sq.algorithm1_pipeline(a, b, "hpne", "auto", 3.0, "dct2", 0, xs, diagnostics=False)
        monkeypatch.setattr(dense, "GRAM_ENGINE", "dmma")
        dm = sq.algorithm1_pipeline(a, b, "hpne", "auto", 3.0, "dct2", 0, xs, diagnostics=False)
        assert oz.preconditioner.computed_in == dm.preconditioner.computed_in
        assert oz.relative_error <= 2 * dm.relative_error + 1e-15, (kappa, oz.relative_error, dm.relative_error)
        del a, b, xs
