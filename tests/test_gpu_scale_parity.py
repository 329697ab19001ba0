"""Parity at scale (VERDICT r1 "pin the config-3 code paths"):

* the GPU pipeline against the row-chunked hybrid CPU oracle (oracle/hybrid.py: the
  reference's estimator, Philox operator, pocketfft sketch, bitwise binary16 level QR
  and n x n solves, LAPACK TRSM) at 524288 x 1024 on the three sides of the
  precision thresholds (kappa 10 -> binary16, 1e3 -> binary32, 2e6 -> binary64):
  same kappa0 decision, same level and escalation, error <= 10x the oracle's;
* the INT8 (Ozaki-II) engine at >= 2^21 rows, where the Gram runs on 15 moduli with
  t = 47, over kappa 1e2 .. 1e14: the forced-INT8 Gram and the blocked TRSM with
  INT8 updates against the FP64 DMMA kernels.
"""
import math

import numpy as np
import pytest
import torch

import paper_2603_16644_b200 as sq
from oracle import hybrid
from oracle import restatement as R

pytestmark = pytest.mark.gpu

KAPPAS = [1e2, 1e4, 1e6, 1e8, 1e10, 1e12, 1e14]


@pytest.mark.timeout(900)
@pytest.mark.parametrize("kappa,method,level", [(10.0, "hpne", "binary16"), (1e3, "hpne", "binary32"),
                                                (2e6, "hpne", "binary64"), (1e3, "pne", "binary32")])
def test_pipeline_vs_hybrid_oracle_at_scale(kappa, method, level):
    from paper_2603_16644_b200.probgen import generate_problem_device, planted_triangle_device
    m, n, seed = 524288, 1024, 31
    a, b, xs = generate_problem_device(m, n, kappa, 1e-6, seed)
    got = sq.algorithm1_pipeline(a, b, method=method, precision="auto", seed=1, x_star=xs, diagnostics=False)
    ah, bh, xh = a.cpu().numpy(), b.cpu().numpy(), xs.cpu().numpy()
    del a, b
    torch.cuda.empty_cache()
    ref = hybrid.pipeline(ah, bh, method=method, precision="auto", seed=1, x_star=xh)
    # the reference estimator on the planted n x n R (A^T A = R^T R / P): the decision
    r = planted_triangle_device(n, kappa, seed + 1).cpu().numpy()
    k0_r, over_r = R.kappa0_from_gram(r.T @ r)
    assert ref.decision[1] == R.choose_level(k0_r, over_r) == level
    assert got.precision_decision.selected.name == level
    if not over_r:
        assert got.precision_decision.kappa0 == pytest.approx(ref.decision[0], abs=1e-3)
    assert got.preconditioner.computed_in.name == ref.pre.level
    assert (got.escalated_from.name if got.escalated_from else None) == ref.escalated_from
    assert got.relative_error <= max(10 * ref.relative_error, 1e-14), (got.relative_error, ref.relative_error)


@pytest.mark.timeout(900)
def test_int8_gram_pipeline_kappa_grid_at_2p21_rows():
    """Every Gram forced onto the INT8 engine at m = 2^21 (15 moduli, t = 47): the
    pipeline's levels, escalations and errors match the FP64 DMMA engine's."""
    from paper_2603_16644_b200 import dense
    from paper_2603_16644_b200.probgen import generate_problem_device
    m, n = 1 << 21, 256
    for kappa in KAPPAS:
        a, b, xs = generate_problem_device(m, n, kappa, 1e-8, 40 + int(math.log10(kappa)))
        out = {}
        for engine in ("ozaki", "dmma"):
            dense.GRAM_ENGINE = engine
            try:
                out[engine] = [sq.algorithm1_pipeline(a, b, method=meth, precision="auto", seed=2, x_star=xs,
                                                      diagnostics=False) for meth in ("pne", "hpne")]
            except sq.SketchLsqError as ex:
                out[engine] = type(ex).__name__
            finally:
                dense.GRAM_ENGINE = "auto"
        if isinstance(out["dmma"], str):
            assert out["ozaki"] == out["dmma"], (kappa, out)
            continue
        for oz, dm in zip(out["ozaki"], out["dmma"]):
            assert oz.precision_decision.selected == dm.precision_decision.selected, kappa
            assert oz.preconditioner.computed_in == dm.preconditioner.computed_in, kappa
            assert oz.escalated_from == dm.escalated_from, kappa
            assert oz.relative_error <= max(10 * dm.relative_error, 1e-14), (kappa, oz.relative_error,
                                                                              dm.relative_error)
        del a, b


@pytest.mark.timeout(900)
def test_int8_gram_error_bound_at_2p21_rows():
    """The INT8 Gram of A_p-like and ill-conditioned columns at 2^21 rows is within the
    FP64 GEMM's error size of the DMMA Gram, for every kappa of the grid."""
    from paper_2603_16644_b200.dense import _gram
    from paper_2603_16644_b200.probgen import generate_problem_device
    m, n = 1 << 21, 256
    for kappa in KAPPAS:
        a, _, _ = generate_problem_device(m, n, kappa, 0.0, 60 + int(math.log10(kappa)))
        g8, g64 = _gram(a, engine="ozaki"), _gram(a, engine="dmma")
        lib = __import__("paper_2603_16644_b200._lib", fromlist=["lib"]).lib()
        absg = _gram(a.abs(), engine="dmma")
        err = ((g8 - g64).abs() / absg).max().item()
        assert err <= m * 2.0 ** -52, (kappa, err)
        del a


@pytest.mark.timeout(900)
def test_blocked_int8_trsm_kappa_grid_at_2p21_rows():
    """The blocked TRSM (DMMA leaves + INT8 updates, 15 moduli) at 2^21 x 2048 over
    kappa(R) 1e2 .. 1e14: backward error at the FP64 level, no worse than 4x the DMMA
    solve's, and forward agreement within kappa u."""
    from paper_2603_16644_b200 import _lib
    from paper_2603_16644_b200.dense import _trsm
    from paper_2603_16644_b200.probgen import planted_triangle_device
    m, n = 1 << 21, 2048
    g = torch.Generator(device="cuda").manual_seed(5)
    a = torch.randn(m, n, dtype=torch.float64, device="cuda", generator=g)
    lib = _lib.lib()
    rows = slice(0, 65536)
    for kappa in KAPPAS:
        r = planted_triangle_device(n, kappa, 70 + int(math.log10(kappa)))
        ap8 = _trsm(a, r, engine="ozaki")
        assert lib.sk_trsm_ozaki_fell_back() == 0
        ap64 = _trsm(a, r, engine="dmma")
        back = []
        for ap in (ap8, ap64):
            res = (ap[rows] @ r - a[rows]).abs().max().item()
            back.append(res / (ap[rows].abs().max().item() * r.abs().max().item() * n))
        assert back[0] <= max(4 * back[1], 1e-16), (kappa, back)
        fwd = ((ap8[rows] - ap64[rows]).abs().max() / ap64[rows].abs().max()).item()
        assert fwd <= max(kappa * 2.0 ** -52 * n, 1e-12), (kappa, fwd)
        del ap8, ap64
