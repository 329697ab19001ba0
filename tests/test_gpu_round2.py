"""Chunked A_p pipeline, wide blocked TRSM, the production-engine §8(b) exports,
wall_ms semantics and the device problem generator under the reference names."""
import ctypes as C
import math

import numpy as np
import pytest
import torch

import paper_2603_16644_b200 as sq
from oracle import restatement as R
from oracle.problems import planted_problem

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("method,prec,rows", [("hpne", "auto", 1000), ("pne", "single", 777),
                                              ("pne", "half", 1500)])
def test_chunked_ap_pipeline_matches_unchunked_and_oracle(method, prec, rows):
    """A_p produced row chunk by row chunk and consumed by the Gram (never
    materialised) gives the reference's level / escalation and error <= 10x."""
    from paper_2603_16644_b200 import solvers
    kappa = 1e6 if prec == "half" else 1e3
    p = planted_problem(6000, 120, kappa, 1e-6, 17)
    ref = R.pipeline(p.a, p.b, method=method, precision=prec, seed=3, x_star=p.x_star, diagnostics=False)
    full = sq.algorithm1_pipeline(p.a, p.b, method=method, precision=prec, seed=3, x_star=p.x_star,
                                  diagnostics=False)
    solvers.AP_CHUNK_ROWS = rows
    try:
        got = sq.algorithm1_pipeline(p.a, p.b, method=method, precision=prec, seed=3, x_star=p.x_star,
                                     diagnostics=True)
    finally:
        solvers.AP_CHUNK_ROWS = None
    assert got.preconditioner.computed_in.name == ref.pre.level == full.preconditioner.computed_in.name
    assert (got.escalated_from.name if got.escalated_from else None) == ref.escalated_from
    assert got.relative_error <= max(10 * ref.relative_error, 1e-14)
    assert np.linalg.norm(got.x_hat - full.x_hat) <= 1e-6 * np.linalg.norm(full.x_hat)
    if method == "pne":      # kappa(A_p) from the chunked Gram's Cholesky factor
        assert 1.0 <= got.preconditioner.kappa_ap < 20
    assert "trsm_gram" not in got.stage_ms or got.stage_ms["trsm_gram"] >= 0


def test_chunked_ozaki_gram_accumulates_in_fp64():
    """sk_gram_ozaki_acc_f64 with accumulate=1 sums per-chunk FP64 Grams: equal to the
    one-shot Gram within the INT8 engine's error bound."""
    from paper_2603_16644_b200.dense import _gram
    g = torch.Generator(device="cuda").manual_seed(1)
    x = torch.randn(3 * 65536, 256, dtype=torch.float64, device="cuda", generator=g)
    y = torch.randn(3 * 65536, 256, dtype=torch.float64, device="cuda", generator=g)
    whole = _gram(x, y, engine="ozaki")
    acc = torch.empty(256, 256, dtype=torch.float64, device="cuda")
    for i, r0 in enumerate(range(0, x.shape[0], 65536)):
        _gram(x[r0:r0 + 65536], y[r0:r0 + 65536], out=acc, accumulate=i > 0, engine="ozaki")
    exact = (x.cpu().numpy().T @ y.cpu().numpy())
    bound = 1e-12 * np.abs(x.cpu().numpy()).T @ np.abs(y.cpu().numpy())
    assert np.all(np.abs(acc.cpu().numpy() - exact) <= bound)
    assert np.all(np.abs(whole.cpu().numpy() - exact) <= bound)


@pytest.mark.parametrize("n", [4352, 5000])
def test_blocked_trsm_wide(n):
    """n >= 4098 used to divide by zero in the row-residue launch (update depth h > 2048);
    h is now capped at 2048 and the right part recurses."""
    from paper_2603_16644_b200.dense import _trsm
    m = 65536
    g = torch.Generator(device="cuda").manual_seed(n)
    a = torch.randn(m, n, dtype=torch.float64, device="cuda", generator=g)
    r = torch.triu(torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g)) / math.sqrt(n)
    r += torch.diag(1.0 + torch.rand(n, dtype=torch.float64, device="cuda", generator=g))
    ap = _trsm(a, r, engine="ozaki")
    lib = __import__("paper_2603_16644_b200._lib", fromlist=["lib"]).lib()
    assert lib.sk_trsm_ozaki_fell_back() == 0
    ref = _trsm(a, r, engine="dmma")
    back = (ap @ r - a).abs().max().item()
    assert back <= 1e-12 * a.abs().max().item() * math.sqrt(n)
    assert (ap - ref).abs().max().item() <= 1e-10 * ref.abs().max().item()


def test_contract_exports_use_production_engine():
    """sk_gemm_tn_f64 / sk_syrk_f64 / sk_kappa0_f64 take the INT8 engine at scale
    (sk_gram_ozaki_fell_back() reports the INT8 path ran without falling back) and
    agree with the DMMA Gram."""
    from paper_2603_16644_b200 import _lib
    from paper_2603_16644_b200.dense import _gram
    lib = _lib.lib()
    m, n = 262144, 256     # m n^2 = 2^34 >= 2^33
    g = torch.Generator(device="cuda").manual_seed(2)
    a = torch.randn(m, n, dtype=torch.float64, device="cuda", generator=g)
    y = torch.randn(m, n, dtype=torch.float64, device="cuda", generator=g)
    v = torch.randn(m, dtype=torch.float64, device="cuda", generator=g)
    ws = torch.empty(max(lib.sk_gemm_tn_workspace(m, n), lib.sk_kappa0_workspace(m, n)), dtype=torch.uint8,
                     device="cuda")
    gg = torch.empty(n, n, dtype=torch.float64, device="cuda")
    rhs = torch.empty(n, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    assert lib.sk_gemm_tn_f64(a.data_ptr(), n, y.data_ptr(), n, m, n, v.data_ptr(), gg.data_ptr(), n,
                              rhs.data_ptr(), ws.data_ptr(), ws.numel(), st) == 0
    torch.cuda.synchronize()
    assert lib.sk_gram_ozaki_fell_back() == 0
    ref = _gram(a, y, engine="dmma")
    assert (gg - ref).abs().max().item() <= 1e-12 * (a.abs().t() @ y.abs()).max().item()
    assert torch.allclose(rhs, a.t() @ v, rtol=1e-12, atol=1e-9)
    assert lib.sk_syrk_f64(a.data_ptr(), n, m, n, gg.data_ptr(), n, ws.data_ptr(), ws.numel(), st) == 0
    torch.cuda.synchronize()
    assert torch.equal(gg, gg.t())
    k0, over = C.c_double(), C.c_int()
    assert lib.sk_kappa0_f64(a.data_ptr(), n, m, n, C.byref(k0), C.byref(over), ws.data_ptr(), ws.numel(),
                             st) == 0
    assert over.value == 0 and 0.0 < k0.value < 4.0


def test_wall_ms_covers_kappa0_estimate():
    """wall_ms includes the kappa0 estimate (src/solvers.py:300-306) for device input."""
    p = planted_problem(20000, 200, 1e2, 1e-6, 5)
    a = torch.from_numpy(p.a).cuda()
    b = torch.from_numpy(p.b).cuda()
    rep = sq.algorithm1_pipeline(a, b, method="hpne", precision="auto", diagnostics=False, stage_timing=True)
    stages = sum(rep.stage_ms.values())
    assert rep.wall_ms >= 0.9 * stages


def test_generate_problem_contracts():
    """Port of tests/test_probgen.py:18-99 (reference contracts) for the device generator."""
    for seed in range(6):
        rho = (0.0, 1e-8, 1e-2, 1.0)[seed % 4]
        kappa = (1.0, 1e2, 1e4)[seed % 3]
        p = sq.generate_problem(300, 24, kappa, rho, seed=seed)
        assert abs(np.linalg.norm(p.x_star) - 1.0) <= 1e-14
        r = p.b - p.a @ p.x_star
        assert abs(np.linalg.norm(r) - rho) <= 1e-12 * rho + 1e-14
        assert np.linalg.norm(p.a.T @ r) <= 1e-12 * rho + 1e-13
        assert p.m == 300 and p.n == 24
    for seed in range(3):
        for kappa in (1.0, 1e2, 1e6):
            p = sq.generate_problem(200, 16, kappa, 0.0, seed=seed)
            assert sq.condition_diagnostics(p.a).two_norm_condition == pytest.approx(kappa, rel=0.01)
    p, q = sq.generate_problem(120, 10, 1e3, 1e-4, seed=42), sq.generate_problem(120, 10, 1e3, 1e-4, seed=42)
    assert np.array_equal(p.a, q.a) and np.array_equal(p.b, q.b) and np.array_equal(p.x_star, q.x_star)
    assert not np.array_equal(p.a, sq.generate_problem(120, 10, 1e3, 1e-4, seed=43).a)
    p = sq.generate_problem(90, 8, 1e2, 0.0, seed=3)
    np.testing.assert_allclose(p.b, p.a @ p.x_star, rtol=1e-14, atol=1e-15)
    for args in ((10, 20, 1e2, 0.0), (100, 10, 0.5, 0.0), (100, 10, 1e2, -1.0)):
        with pytest.raises(ValueError):
            sq.generate_problem(*args, seed=0)
    r = sq.triangular_with_condition(12, 1e4, seed=7)
    assert np.all(r[np.tril_indices(12, -1)] == 0.0)
    assert sq.condition_diagnostics(r).two_norm_condition == pytest.approx(1e4, rel=1e-6)
    with pytest.raises(ValueError):
        sq.triangular_with_condition(1, 1e2, seed=0)
    q = sq.random_orthogonal_columns(50, 7, seed=5)
    assert q.shape == (50, 7) and np.linalg.norm(q.T @ q - np.eye(7)) <= 1e-13
    # same random streams as the reference: x* is bitwise the oracle generator's
    assert np.array_equal(sq.generate_problem(300, 24, 1e2, 1e-6, seed=9).x_star,
                          planted_problem(300, 24, 1e2, 1e-6, 9).x_star)


def test_sharded_device_generator_is_one_global_problem():
    """Two row shards of generate_problem_device(rank=g, world=2) stack into one
    problem with kappa(A) = kappa(R), ||e|| = rho, e orthogonal to range(A)."""
    from paper_2603_16644_b200.probgen import generate_problem_device
    parts = [generate_problem_device(4096, 64, 1e4, 1e-3, 11, rank=g, world=2) for g in range(2)]
    assert torch.equal(parts[0][2], parts[1][2])           # same x*
    a = torch.cat([p[0] for p in parts]).cpu().numpy()
    b = torch.cat([p[1] for p in parts]).cpu().numpy()
    x = parts[0][2].cpu().numpy()
    sv = np.linalg.svd(a, compute_uv=False)
    assert sv[0] / sv[-1] == pytest.approx(1e4, rel=0.01)
    e = b - a @ x
    assert np.linalg.norm(e) == pytest.approx(1e-3, rel=1e-10)
    assert np.linalg.norm(a.T @ e) <= 1e-12


def test_measure_bound_inputs_matches_oracle_diagnostics():
    """measure_bound_inputs (src/bounds.py:202-255) on the device against the same
    quantities from the oracle's Jacobi diagnostics (restatement.condition_number)."""
    p = planted_problem(600, 40, 1e4, 1e-6, 8)
    rep = sq.algorithm1_pipeline(p.a, p.b, method="pne", precision="single", seed=2, x_star=p.x_star,
                                 diagnostics=False)
    pre = rep.preconditioner
    bi = sq.measure_bound_inputs(p, rep, pre)
    r_s = pre.r_s
    a_p = np.linalg.solve(r_s.T, p.a.T).T
    ka = R.condition_number(p.a)[1]
    krs = R.condition_number(r_s)[1]
    kap = R.condition_number(a_p)[1]
    kapta = R.condition_number(a_p.T @ p.a)[1]
    assert bi.kappa_a == pytest.approx(ka, rel=1e-8)
    assert bi.kappa_rs == pytest.approx(krs, rel=1e-8)
    assert bi.kappa_ap == pytest.approx(kap, rel=1e-8)
    assert bi.kappa_apta == pytest.approx(kapta, rel=1e-6)
    assert bi.u1 == 2.0 ** -23 and bi.u2 == 2.0 ** -52 and bi.eps_b is None
    x = rep.x_hat
    na = R.condition_number(p.a)[0]
    assert bi.res_ratio_a == pytest.approx(np.linalg.norm(p.a @ x - p.b) / (na * np.linalg.norm(x)), rel=1e-6)
    y = r_s @ x
    assert bi.nu_pne == pytest.approx(np.linalg.norm(y) / (R.condition_number(r_s)[0] * np.linalg.norm(x)), rel=1e-8)
    nap, napta = R.condition_number(a_p)[0], R.condition_number(a_p.T @ p.a)[0]
    assert bi.nu_hpne == pytest.approx(nap * na / napta, rel=1e-6)


def test_pageable_host_input_staged_bitwise(monkeypatch):
    """Pageable numpy input above STREAM_MIN_BYTES goes through the pinned staging ring
    (several pieces per chunk, slots reused); the result is bitwise that of pinned
    input, which the copy engine reads directly."""
    from paper_2603_16644_b200 import solvers as S
    monkeypatch.setattr(S, "STREAM_MIN_BYTES", 0)
    monkeypatch.setattr(S._PinnedRing, "PIECE_BYTES", 96 * 1024)       # many pieces, slot reuse
    S._PINNED.release()
    p = planted_problem(20000, 48, 1e3, 1e-6, 3)
    a_np = np.ascontiguousarray(p.a)
    pageable = sq.algorithm1_pipeline(a_np, p.b, method="hpne", precision="auto", seed=3, x_star=p.x_star,
                                      diagnostics=False)
    pinned = sq.algorithm1_pipeline(torch.from_numpy(a_np).pin_memory(), p.b, method="hpne", precision="auto",
                                    seed=3, x_star=p.x_star, diagnostics=False)
    assert np.array_equal(pageable.x_hat, pinned.x_hat)
    assert pageable.precision_decision.selected == pinned.precision_decision.selected
    S._PINNED.release()
