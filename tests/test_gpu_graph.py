"""PipelinePlan: the whole config-1-class solve as one CUDA graph with deferred verdicts
(sk_defer_verdicts).  Results must equal the eager algorithm1_pipeline bit for bit,
failures must raise what the eager call raises, and a replay with new inputs must not
see the previous ones."""
import numpy as np
import pytest
import torch

import paper_2603_16644_b200 as sq
from paper_2603_16644_b200 import _lib
from paper_2603_16644_b200.graph import PipelinePlan
from oracle import restatement as R
from oracle.problems import planted_problem

pytestmark = pytest.mark.gpu


def _eager(a, b, method, prec, xs, seed=1):
    return sq.algorithm1_pipeline(a, b, method=method, precision=prec, seed=seed, x_star=xs, diagnostics=False)


def _same(rep, ref):
    assert np.array_equal(rep.x_hat, ref.x_hat)
    assert rep.residual_norm == ref.residual_norm
    assert rep.relative_residual == ref.relative_residual
    assert rep.relative_error == ref.relative_error
    assert rep.preconditioner.computed_in.name == ref.preconditioner.computed_in.name
    assert torch.equal(rep.preconditioner.r_device(), ref.preconditioner.r_device())


@pytest.mark.parametrize("method", ["pne", "hpne"])
@pytest.mark.parametrize("prec", ["single", "double", "auto"])
def test_plan_equals_eager_config1(method, prec):
    p = planted_problem(1000, 100, 1e8, 1e-6, 11)
    a, b = torch.from_numpy(p.a).cuda(), torch.from_numpy(p.b).cuda()
    plan = PipelinePlan(1000, 100, method=method, precision=prec, seed=1)
    ref = _eager(a, b, method, prec, p.x_star)
    for _ in range(3):                       # replays are idempotent
        rep = plan.solve(a, b, p.x_star)
        _same(rep, ref)
    if prec == "auto":
        assert rep.precision_decision.selected.name == ref.precision_decision.selected.name
        assert rep.precision_decision.kappa0 == ref.precision_decision.kappa0
    # and the oracle's level / error class (config-1 gate)
    o = R.pipeline(p.a, p.b, method=method, precision=prec, seed=1, x_star=p.x_star, diagnostics=False)
    assert rep.preconditioner.computed_in.name == o.pre.level
    assert rep.relative_error <= max(10 * o.relative_error, 1e-14)


def test_plan_new_inputs_each_replay_and_host_inputs():
    plan = PipelinePlan(700, 60, method="hpne", precision="single", seed=5)
    for seed in (1, 2, 3):
        p = planted_problem(700, 60, 1e4, 1e-8, seed)
        ref = _eager(p.a, p.b, "hpne", "single", p.x_star, seed=5)
        _same(plan.solve(p.a, p.b, p.x_star), ref)       # numpy inputs
    # in-place inputs: fill plan.a / plan.b on the device, solve() without arguments
    p = planted_problem(700, 60, 1e4, 1e-8, 9)
    plan.a.copy_(torch.from_numpy(p.a))
    plan.b.copy_(torch.from_numpy(p.b))
    _same(plan.solve(x_star=p.x_star), _eager(p.a, p.b, "hpne", "single", p.x_star, seed=5))


def test_plan_binary16_level_and_escalation():
    """binary16 at kappa 1e8 collapses in the level QR: the recorded RankDeficient
    re-runs eagerly, which escalates to binary32 exactly like algorithm1_pipeline."""
    for kappa in (1e2, 1e8):
        p = planted_problem(1200, 80, kappa, 1e-6, 4)
        ref = _eager(p.a, p.b, "pne", "half", p.x_star)
        rep = PipelinePlan(1200, 80, method="pne", precision="half", seed=1).solve(p.a, p.b, p.x_star)
        _same(rep, ref)
        assert (rep.escalated_from.name if rep.escalated_from else None) == \
               (ref.escalated_from.name if ref.escalated_from else None)


def _raises_same(fn_eager, fn_plan):
    with pytest.raises(Exception) as e1:
        fn_eager()
    with pytest.raises(Exception) as e2:
        fn_plan()
    assert type(e1.value) is type(e2.value)
    return e2.value


def test_plan_failures_raise_like_eager():
    p = planted_problem(500, 40, 1e3, 1e-6, 2)
    plan = PipelinePlan(500, 40, method="pne", precision="single", seed=1)
    bad = p.a.copy()
    bad[17, 3] = np.nan
    err = _raises_same(lambda: _eager(bad, p.b, "pne", "single", None), lambda: plan.solve(bad, p.b))
    assert isinstance(err, ValueError)
    big = p.a * 1e300                          # overflows binary32 in the sketch's demotion
    err = _raises_same(lambda: _eager(big, p.b, "pne", "single", None), lambda: plan.solve(big, p.b))
    assert isinstance(err, sq.Overflow)
    zero = p.a.copy()
    zero[:, 5] = 0.0                           # exactly rank deficient
    plan64 = PipelinePlan(500, 40, method="hpne", precision="double", seed=1)
    _raises_same(lambda: _eager(zero, p.b, "hpne", "double", None), lambda: plan64.solve(zero, p.b))
    # the plan recovers on the next good input
    _same(plan.solve(p.a, p.b, p.x_star), _eager(p.a, p.b, "pne", "single", p.x_star))


def test_plan_refuses_bad_methods():
    with pytest.raises(ValueError):
        PipelinePlan(100, 10, method="sne")


@pytest.mark.parametrize("m,n,method,prec", [(140000, 256, "hpne", "single"),   # INT8 Gram (GEMM-TN)
                                             (140000, 256, "pne", "double"),    # INT8 Gram (SYRK)
                                             (9000, 1100, "pne", "single"),     # + INT8 TRSM
                                             (9000, 1100, "hpne", "auto")])
def test_plan_with_the_int8_engines_equals_eager(m, n, method, prec):
    """Shapes on the INT8 Ozaki-II Gram / TRSM: their guard flags stay on the device and
    the DMMA fallbacks run gated on them, so the graph is bitwise the eager solve."""
    p = planted_problem(m, n, 1e3, 1e-6, 31)
    a, b = torch.from_numpy(p.a).cuda(), torch.from_numpy(p.b).cuda()
    plan = PipelinePlan(m, n, method=method, precision=prec, seed=3)
    ref = _eager(a, b, method, prec, p.x_star, seed=3)
    for _ in range(2):
        _same(plan.solve(a, b, p.x_star), ref)


def test_plan_int8_gram_guard_fallback_equals_eager():
    """A spiky column (one entry dominating its column norm) trips the INT8 Gram's guard:
    eager falls back to the DMMA Gram on the host's read of the flag, the graph runs the
    gated DMMA Gram on the device flag; the results are the same bits."""
    from paper_2603_16644_b200 import dense as D
    p = planted_problem(140000, 256, 1e3, 1e-6, 32)
    a = p.a.copy()
    a[77, 5] *= 1e6
    a_d, b_d = torch.from_numpy(a).cuda(), torch.from_numpy(p.b).cuda()
    plan = PipelinePlan(140000, 256, method="hpne", precision="double", seed=3)
    ref = _eager(a_d, b_d, "hpne", "double", None, seed=3)
    assert _lib.lib().sk_gram_ozaki_fell_back() == 1        # the eager Gram did fall back
    _same(plan.solve(a_d, b_d), ref)


@pytest.mark.parametrize("prec", ["half", "single", "double"])
def test_plan_with_the_fft_sketch_equals_eager(prec):
    """m % 2048 == 0 takes the FFT sketch, whose pass-B request lists are planned on the
    device: the whole solve still captures, bitwise the eager result."""
    p = planted_problem(4096, 64, 1e3, 1e-6, 21)
    plan = PipelinePlan(4096, 64, method="hpne", precision=prec, seed=2)
    ref = _eager(p.a, p.b, "hpne", prec, p.x_star, seed=2)
    for _ in range(2):
        _same(plan.solve(p.a, p.b, p.x_star), ref)


def test_deferred_verdicts_refuse_host_value_entry_points():
    """While verdicts are deferred an entry point that returns a host value fails
    loudly instead of synchronising."""
    import ctypes as C
    lib = _lib.lib()
    st = torch.zeros(4, dtype=torch.float64, device="cuda")
    g = torch.eye(8, dtype=torch.float64, device="cuda")
    ws = torch.empty(1 << 16, dtype=torch.uint8, device="cuda")
    out = (C.c_double * 2)()
    assert lib.sk_defer_verdicts(st.data_ptr()) == 0
    try:
        rc = lib.sk_gram_check(g.data_ptr(), 8, out, ws.data_ptr(), ws.numel(),
                               torch.cuda.current_stream().cuda_stream)
    finally:
        lib.sk_defer_verdicts(None)
    assert rc == -2 and b"sk_defer_verdicts" in lib.sk_last_error()


def test_plans_on_two_host_threads():
    """The deferred-verdict record is per host thread and each plan owns its buffers and
    streams: two threads replaying their own plans concurrently get the eager results."""
    import threading
    probs = [planted_problem(800, 70, 1e4, 1e-6, s) for s in (41, 42)]
    refs = [_eager(p.a, p.b, "hpne", "single", p.x_star, seed=7) for p in probs]
    plans = [PipelinePlan(800, 70, method="hpne", precision="single", seed=7) for _ in probs]
    errors = []

    def work(i):
        try:
            for _ in range(20):
                _same(plans[i].solve(probs[i].a, probs[i].b, probs[i].x_star), refs[i])
        except Exception as ex:  # noqa: BLE001
            errors.append(ex)

    threads = [threading.Thread(target=work, args=(i,)) for i in range(2)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
