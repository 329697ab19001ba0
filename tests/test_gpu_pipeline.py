"""GPU parity of the solvers and Algorithm 1 against the reference's golden runs
and the reference's own solver tests (hot-path subset of
pkg/tests/test_solvers.py and pkg/tests/test_acceptance.py).

Parity gate (BASELINE.json north star): same chosen precision, same escalation,
same outcome class, and relative forward error no worse than 10x the
reference's on the same A, b and sketch."""
import math

import numpy as np
import pytest

from oracle import restatement as R
from oracle.problems import planted_problem
from tests.golden_data import ARR, META, problem

pytestmark = pytest.mark.gpu

ERR_FLOOR = 1e-14   # below this both solvers are at the binary64 noise floor


@pytest.fixture(scope="module")
def sq():
    import paper_2603_16644_b200 as mod
    return mod


SEEDS = {"p600_k1e2": 4, "p600_k1e6": 4, "p600_k1e10": 4, "p600_k1e6_s6": 6}


@pytest.mark.parametrize("key", sorted(META["runs"]))
def test_pipeline_vs_reference_runs(sq, key):
    _, name, method, prec = key.split("/")
    info = META["runs"][key]
    p = problem(name)
    seed = SEEDS.get(name, META["cases"][name]["seed"])
    rep = sq.algorithm1_pipeline(p.a, p.b, method=method, precision=prec, seed=seed, x_star=p.x_star)
    assert rep.preconditioner.computed_in.name == info["level"]
    assert (rep.escalated_from.name if rep.escalated_from else None) == info["escalated_from"]
    assert rep.relative_error <= max(10 * info["rel_error"], ERR_FLOOR), (rep.relative_error, info["rel_error"])
    assert rep.residual_norm == pytest.approx(info["residual_norm"], rel=1e-6)
    ref_k0 = info["kappa0"]
    if (ref_k0 is not None and not (isinstance(ref_k0, float) and math.isnan(ref_k0))
            and not rep.precision_decision.overflowed):
        # kappa0 = 0.5 log10(n ||G||_1 est ||G^-1||_1) with kappa(G) up to ~1e16:
        # summation-order differences move it by O(kappa(G) u) relative -> 1e-4 in log10
        assert abs(rep.precision_decision.kappa0 - info["kappa0"]) <= 1e-4
    # preconditioner quality is the point of the sketch: never worse than the
    # reference's (ours rounds the exact sampled transform once, so it is often better)
    assert rep.preconditioner.kappa_ap <= 2.0 * info["kappa_ap"] + 1.0
    # kappa(R_s) tracks kappa(A) up to the level's rounding noise (a binary32 sketch
    # of a kappa = 1e8 matrix resolves it only to a factor ~2)
    assert info["kappa_rs"] / 3 <= rep.preconditioner.kappa_rs <= 3 * info["kappa_rs"]


def test_stage_functions_vs_reference(sq):
    p = problem("p300_k10_s5")
    pre = sq.build_preconditioner(p.a, seed=5)
    assert pre.sketch_descriptor == META["stage"]["descriptor"]
    a_p = sq.precondition_matrix(p.a, pre)
    assert np.abs(pre.r_s - ARR["stage/p300_k10_s5/r_s"]).max() <= 1e-12 * np.abs(pre.r_s).max()
    assert np.abs(a_p - ARR["stage/p300_k10_s5/a_p"]).max() <= 1e-11
    assert pre.kappa_ap == pytest.approx(META["stage"]["kappa_ap"], rel=1e-6)
    outs = {"qr": sq.solve_qr_baseline(p.a, p.b, x_star=p.x_star),
            "ne": sq.solve_normal(p.a, p.b, x_star=p.x_star),
            "sne": sq.solve_seminormal(p.a, p.b, x_star=p.x_star),
            "nne_ap": sq.solve_notnormal(p.a, a_p, p.b, x_star=p.x_star),
            "pne": sq.solve_pne(p.a, p.b, pre, x_star=p.x_star, a_p=a_p),
            "hpne": sq.solve_hpne(p.a, p.b, pre, x_star=p.x_star, a_p=a_p)}
    for tag, rep in outs.items():
        ref = ARR[f"solve/p300_k10_s5/{tag}"]
        assert np.linalg.norm(rep.x_hat - ref) <= 1e-10 * np.linalg.norm(ref), tag
        assert rep.method == {"nne_ap": "nne"}.get(tag, tag)
    pn = problem("p600_k1e10")
    with pytest.raises(sq.NotPositiveDefinite):
        sq.solve_normal(pn.a, pn.b)


# ---- ports of pkg/tests/test_solvers.py (hot path) --------------------------
def test_qr_baseline_recovers_planted_solution(sq):
    for seed in range(3):
        p = planted_problem(200, 16, 1e2, 1e-8, seed)
        rep = sq.solve_qr_baseline(p.a, p.b, x_star=p.x_star)
        assert rep.relative_error <= 1e-12
        assert rep.residual_norm == pytest.approx(1e-8, abs=1e-12)
        assert rep.method == "qr" and rep.wall_ms > 0.0


def test_all_methods_agree_on_well_conditioned_input(sq):
    p = planted_problem(300, 20, 10.0, 1e-4, 5)
    x_qr = sq.solve_qr_baseline(p.a, p.b).x_hat
    pre = sq.build_preconditioner(p.a, seed=5)
    a_p = sq.precondition_matrix(p.a, pre)
    for x in (sq.solve_normal(p.a, p.b).x_hat, sq.solve_seminormal(p.a, p.b).x_hat,
              sq.solve_notnormal(p.a, p.a, p.b).x_hat, sq.solve_pne(p.a, p.b, pre, a_p=a_p).x_hat,
              sq.solve_hpne(p.a, p.b, pre, a_p=a_p).x_hat):
        assert np.linalg.norm(x - x_qr) <= 1e-10 * np.linalg.norm(x_qr)


def test_normal_equations_break_when_gram_loses_definiteness(sq):
    p = planted_problem(400, 30, 1e9, 1e-6, 1)
    with pytest.raises(sq.NotPositiveDefinite):
        sq.solve_normal(p.a, p.b)


def test_identity_preconditioner_reduces_pne_to_ne(sq):
    p = planted_problem(250, 18, 1e2, 1e-6, 7)
    pre = sq.Preconditioner(r_s=np.eye(p.a.shape[1]), computed_in=sq.BINARY64, kappa_rs=1.0)
    a_p = sq.precondition_matrix(p.a, pre)
    assert np.array_equal(a_p, p.a)
    assert np.array_equal(sq.solve_pne(p.a, p.b, pre, a_p=a_p).x_hat, sq.solve_normal(p.a, p.b).x_hat)


def test_notnormal_reduces_to_hpne_and_ne(sq):
    for seed in range(3):
        p = planted_problem(300, 20, 1e2, 1e-4, seed)
        pre = sq.build_preconditioner(p.a, seed=seed)
        a_p = sq.precondition_matrix(p.a, pre)
        x_h = sq.solve_hpne(p.a, p.b, pre, a_p=a_p).x_hat
        x_bh = sq.solve_notnormal(p.a, a_p, p.b).x_hat
        assert np.linalg.norm(x_bh - x_h) <= 1e-13 * np.linalg.norm(x_h)
        x_n = sq.solve_normal(p.a, p.b).x_hat
        x_bn = sq.solve_notnormal(p.a, p.a, p.b).x_hat
        assert np.linalg.norm(x_bn - x_n) <= 1e-12 * np.linalg.norm(x_n)
    with pytest.raises(sq.DimensionMismatch):
        sq.solve_notnormal(p.a, p.a[:, :4], p.b)


def test_exact_qr_preconditioner_is_idempotent(sq):
    for seed in range(2):
        p = planted_problem(300, 24, 1e6, 0.0, seed)
        r = R.householder_qr(p.a)[1]
        pre = sq.Preconditioner(r_s=r, computed_in=sq.BINARY64, kappa_rs=1e6)
        sq.precondition_matrix(p.a, pre)
        assert pre.kappa_ap <= 1.0 + 1e-6


def test_preconditioner_quality_at_default_sample_factor(sq):
    for seed in range(3):
        p = planted_problem(1024, 32, 1e6, 0.0, seed)
        pre = sq.build_preconditioner(p.a, seed=seed)
        assert pre.r_s.shape == (32, 32)
        sq.precondition_matrix(p.a, pre)
        assert pre.kappa_ap <= 10.0
        assert pre.kappa_rs == pytest.approx(1e6, rel=0.7)
        assert pre.computed_in is sq.BINARY64 and pre.sketch_descriptor is not None


def test_solve_scale_equivariance(sq):
    """Power-of-two scaling of A and b leaves the solution bitwise unchanged."""
    p = planted_problem(200, 16, 1e3, 1e-6, 9)
    for k in (3, -5):
        s = 2.0 ** k
        got = sq.algorithm1_pipeline(p.a * s, p.b * s, method="pne", precision="double", seed=9)
        ref = sq.algorithm1_pipeline(p.a, p.b, method="pne", precision="double", seed=9)
        assert np.array_equal(got.x_hat, ref.x_hat)
        assert np.array_equal(sq.solve_normal(p.a * s, p.b * s).x_hat, sq.solve_normal(p.a, p.b).x_hat)


def test_pipeline_fixed_precision_paths(sq):
    p = planted_problem(600, 40, 1e2, 1e-8, 3)
    for name, level in (("half", sq.BINARY16), ("single", sq.BINARY32), ("double", sq.BINARY64)):
        rep = sq.algorithm1_pipeline(p.a, p.b, method="pne", precision=name, seed=3, x_star=p.x_star)
        assert rep.preconditioner.computed_in is level
        assert rep.escalated_from is None
        assert rep.relative_error <= 1e-6
        assert rep.bounds == {}


def test_pipeline_auto_selects_by_conditioning(sq):
    for kappa, level in ((1e2, sq.BINARY16), (1e6, sq.BINARY32), (1e10, sq.BINARY64)):
        p = planted_problem(600, 40, kappa, 1e-8, 4)
        rep = sq.algorithm1_pipeline(p.a, p.b, method="hpne", precision="auto", seed=4, x_star=p.x_star)
        assert rep.precision_decision.selected is level
        assert rep.preconditioner.computed_in is level


def test_pipeline_escalates_when_half_collapses(sq):
    p = planted_problem(600, 40, 1e6, 1e-8, 6)
    rep = sq.algorithm1_pipeline(p.a, p.b, method="pne", precision="half", seed=6, x_star=p.x_star)
    assert rep.escalated_from is sq.BINARY16
    assert rep.preconditioner.computed_in is sq.BINARY32
    assert rep.relative_error <= 1e-6


def test_pipeline_rejects_unknown_method_and_bad_input(sq):
    p = planted_problem(100, 8, 10.0, 0.0, 0)
    with pytest.raises(ValueError):
        sq.algorithm1_pipeline(p.a, p.b, method="cgls")
    with pytest.raises(ValueError):
        sq.algorithm1_pipeline(p.a, p.b, precision="quad")
    bad = p.a.copy()
    bad[3, 2] = np.nan
    with pytest.raises(ValueError):
        sq.algorithm1_pipeline(bad, p.b)
    with pytest.raises(sq.DimensionMismatch):
        sq.algorithm1_pipeline(p.a[:5], p.b[:5])
    with pytest.raises(sq.DimensionMismatch):
        sq.algorithm1_pipeline(p.a, p.b[:-1])


def test_overflow_on_demotion(sq):
    p = planted_problem(100, 8, 10.0, 0.0, 0)
    big = p.a * 1e6        # max|A| ~ 1e6 > 65504: binary16 demotion overflows
    with pytest.raises(sq.Overflow):
        sq.build_preconditioner(big, level=sq.BINARY16)


def test_report_norms_are_consistent(sq):
    p = planted_problem(300, 20, 1e3, 1e-2, 8)
    rep = sq.solve_qr_baseline(p.a, p.b, x_star=p.x_star)
    r = p.b - p.a @ rep.x_hat
    assert rep.residual_norm == pytest.approx(np.linalg.norm(r), rel=1e-12)
    denom = np.linalg.norm(p.a, "fro") * np.linalg.norm(rep.x_hat)
    assert rep.relative_residual == pytest.approx(np.linalg.norm(r) / denom, rel=1e-12)
    assert rep.norm_is_frobenius


def test_torch_cuda_inputs_stay_on_device(sq):
    import torch
    p = planted_problem(2000, 50, 1e4, 1e-8, 3)
    at = torch.from_numpy(p.a).cuda()
    bt = torch.from_numpy(p.b).cuda()
    rep = sq.algorithm1_pipeline(at, bt, method="hpne", precision="auto", seed=3, x_star=p.x_star,
                                 stage_timing=True)
    ref = R.pipeline(p.a, p.b, method="hpne", precision="auto", seed=3, x_star=p.x_star, diagnostics=False)
    assert rep.precision_decision.selected.name == ref.decision[1]
    assert rep.relative_error <= max(10 * ref.relative_error, ERR_FLOOR)
    assert {"sketch", "level_qr", "trsm", "gram", "nxn"} <= set(rep.stage_ms)
    pre = sq.build_preconditioner(at, seed=3)
    a_p = sq.precondition_matrix(at, pre)
    assert isinstance(a_p, torch.Tensor) and a_p.is_cuda


@pytest.mark.parametrize("kappa,prec,level", [(1e2, "auto", "binary16"), (1e6, "auto", "binary32"),
                                              (1e2, "single", "binary32"), (1e10, "auto", "binary64")])
def test_streamed_host_ingestion_matches(sq, monkeypatch, kappa, prec, level):
    """Host input above STREAM_MIN_BYTES is copied in row chunks that overlap the
    kappa0 Gram and the (speculative) sketch; decisions and accuracy must match."""
    from paper_2603_16644_b200 import solvers as S
    p = planted_problem(3000, 40, kappa, 1e-8, 5)
    ref = R.pipeline(p.a, p.b, method="hpne", precision=prec, seed=5, x_star=p.x_star, diagnostics=False)
    monkeypatch.setattr(S, "STREAM_MIN_BYTES", 0)
    monkeypatch.setattr(S, "STREAM_CHUNKS", 7)
    got = sq.algorithm1_pipeline(p.a, p.b, method="hpne", precision=prec, seed=5, x_star=p.x_star,
                                 diagnostics=False)
    assert got.preconditioner.computed_in.name == ref.pre.level == level
    assert got.relative_error <= max(10 * ref.relative_error, ERR_FLOOR)
    bad = p.a.copy()
    bad[2999, 39] = np.inf
    with pytest.raises(ValueError):
        sq.algorithm1_pipeline(bad, p.b, precision=prec)


def test_device_auto_path_validates_through_the_gram(sq):
    """Device-resident A under "auto" is validated by the kappa0 Gram (non-finite A
    makes G non-finite) and ||A||_F^2 comes from trace(G)."""
    import torch
    p = planted_problem(2000, 50, 1e4, 1e-8, 3)
    rep = sq.algorithm1_pipeline(torch.from_numpy(p.a).cuda(), torch.from_numpy(p.b).cuda(), method="pne",
                                 precision="auto", seed=3, x_star=p.x_star)
    ref = R.pipeline(p.a, p.b, method="pne", precision="auto", seed=3, x_star=p.x_star, diagnostics=False)
    assert rep.relative_residual == pytest.approx(ref.relative_residual, rel=1e-8)
    assert rep.relative_error <= max(10 * ref.relative_error, ERR_FLOOR)
    bad = p.a.copy()
    bad[1234, 7] = np.nan
    with pytest.raises(ValueError):
        sq.algorithm1_pipeline(torch.from_numpy(bad).cuda(), torch.from_numpy(p.b).cuda(), precision="auto")
    with pytest.raises(sq.DimensionMismatch):
        sq.algorithm1_pipeline(torch.from_numpy(p.a).cuda(), torch.from_numpy(p.b[:-3]).cuda(), precision="auto")


def test_sharded_pipeline_single_rank_device_ops(sq):
    """distributed.algorithm1_pipeline_sharded with the production DeviceOps on one
    GPU (no process group: every all-reduce is the identity)."""
    from paper_2603_16644_b200.distributed import algorithm1_pipeline_sharded
    for kappa, method, prec in ((1e2, "hpne", "auto"), (1e6, "pne", "half")):
        p = planted_problem(600, 40, kappa, 1e-8, 6)
        got = algorithm1_pipeline_sharded(p.a, p.b, method=method, precision=prec, seed=6, x_star=p.x_star)
        ref = R.pipeline(p.a, p.b, method=method, precision=prec, seed=6, x_star=p.x_star, diagnostics=False)
        assert got.preconditioner.computed_in.name == ref.pre.level
        assert (got.escalated_from.name if got.escalated_from else None) == ref.escalated_from
        assert got.relative_error <= max(10 * ref.relative_error, ERR_FLOOR)
        one = sq.algorithm1_pipeline(p.a, p.b, method=method, precision=prec, seed=6, x_star=p.x_star,
                                     diagnostics=False)
        assert np.linalg.norm(got.x_hat - one.x_hat) <= 1e-12 * np.linalg.norm(one.x_hat)
