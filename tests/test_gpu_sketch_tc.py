"""tcgen05 binary16 sketch vs the FP64 DMMA sketch and the closed-form operator,
plus the row-shard decomposition that the multi-GPU path relies on."""
import numpy as np
import pytest

from oracle import restatement as R

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch
    import paper_2603_16644_b200 as sq
    from paper_2603_16644_b200 import sketch as S
    return torch, sq, S


def _sum(env, op, a, algo, row_offset=0, out=None, accumulate=False):
    torch, sq, S = env
    dsk = S.DeviceSketch(op)
    total, flag = S._sketch_sum(dsk, a, 16, row_offset=row_offset, out=out, accumulate=accumulate, algo=algo)
    torch.cuda.synchronize()
    return total, int(flag.item())


@pytest.mark.parametrize("m,n,d,transform", [(3000, 40, 120, "dct2"), (70001, 300, 900, "dct2"),
                                             (40000, 257, 771, "wht"), (262144, 512, 1536, "dct2")])
def test_tc_matches_dmma(env, m, n, d, transform):
    torch, sq, S = env
    g = R.philox(m + n, 3)
    a = torch.from_numpy(g.standard_normal((m, n))).cuda()
    op = sq.make_sketch(m, d, transform, seed=5)
    tc, f1 = _sum(env, op, a, "tc")
    dm, f2 = _sum(env, op, a, "dmma")
    assert f1 == 0 and f2 == 0
    tc, dm = tc.cpu().numpy(), dm.cpu().numpy()
    # both contract the same fp16-rounded A; the TC operator is rounded to fp16
    # (relative 2^-11 per entry, random signs -> ~2^-11/sqrt(...) in the sums)
    err = np.abs(tc - dm).max() / np.abs(dm).max()
    assert err <= 2e-3, err
    if transform == "wht":     # +-1 operator is exact in fp16: only fp32 accumulation order differs
        assert err <= 1e-5, err


@pytest.mark.parametrize("transform,tol", [("wht", 1e-5), ("dct2", 2e-3)])
def test_tc_row_shards_sum_to_full(env, transform, tol):
    # WHT: the +-1 operator is exact, so shards match to fp32 accumulation order.
    # DCT: the fp32 phase recurrence restarts at each shard's 32-column chunks,
    # so a few operator entries round to the neighbouring fp16 value.
    torch, sq, S = env
    m, n, d = 50000, 130, 390
    a = torch.from_numpy(R.philox(9, 3).standard_normal((m, n))).cuda()
    op = sq.make_sketch(m, d, transform, seed=2)
    full, _ = _sum(env, op, a, "tc")
    cut = [0, 12345, 30000, m]
    acc = None
    for lo, hi in zip(cut[:-1], cut[1:]):
        acc, _ = _sum(env, op, a[lo:hi].contiguous(), "tc", row_offset=lo, out=acc, accumulate=acc is not None)
    full, acc = full.cpu().numpy(), acc.cpu().numpy()
    assert np.abs(full - acc).max() <= tol * np.abs(full).max()


def test_tc_overflow_flag(env):
    torch, sq, S = env
    a = torch.ones((1000, 20), dtype=torch.float64, device="cuda")
    a[17, 3] = 1e6     # > 65504: binary16 demotion overflows
    op = sq.make_sketch(1000, 60, "dct2", seed=1)
    _, flag = _sum(env, op, a, "tc")
    assert flag == 1


def test_tc_pipeline_half_level_matches_oracle(env):
    torch, sq, S = env
    from oracle.problems import planted_problem
    p = planted_problem(20000, 64, 10.0, 1e-6, 3)
    rep = sq.algorithm1_pipeline(p.a, p.b, method="hpne", precision="half", seed=3, x_star=p.x_star)
    ref = R.pipeline(p.a, p.b, method="hpne", precision="half", seed=3, x_star=p.x_star, diagnostics=False)
    assert rep.preconditioner.computed_in.name == "binary16" and ref.pre.level == "binary16"
    assert rep.relative_error <= max(10 * ref.relative_error, 1e-14)
    assert rep.preconditioner.kappa_ap <= 10
