"""FP64 fast (FFT, Makhoul + pruned four-step) sampled DCT-II sketch vs the dense
FP64 DMMA sketch and the oracle's pocketfft sketch."""
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


def _sum(env, op, a, level, algo, row_offset=0, out=None, accumulate=False):
    torch, sq, S = env
    total, flag = S._sketch_sum(S.DeviceSketch(op), a, level, row_offset=row_offset, out=out,
                                accumulate=accumulate, algo=algo)
    torch.cuda.synchronize()
    return total, int(flag.item())


@pytest.fixture(params=["tf32", "fft", "mma", "simt"])
def passb(request, monkeypatch):
    """pass-B engine of the FFT sketch (libsklsq reads SK_FFT_PASSB per call): "tf32" the
    default (3xTF32 tensor cores for the binary32 transform, DMMA for binary64), "fft" the
    length-M1 FFT over j1 (power-of-two M1 in [16, 4096]; the DMMA sum otherwise), "mma"
    the DMMA direct sum, "simt" the SIMT direct sum"""
    monkeypatch.setenv("SK_FFT_PASSB", request.param)
    return request.param


@pytest.mark.parametrize("m,n,d", [(4096, 20, 60), (8192, 37, 111), (65536, 130, 390), (1 << 20, 64, 192)])
def test_fft_matches_dense_fp64(env, passb, m, n, d):
    torch, sq, S = env
    a = torch.from_numpy(R.philox(m + n, 3).standard_normal((m, n))).cuda()
    op = sq.make_sketch(m, d, "dct2", seed=3)
    fft, f1 = _sum(env, op, a, 64, "fft")
    dm, f2 = _sum(env, op, a, 64, "dmma")
    assert f1 == 0 and f2 == 0
    fft, dm = fft.cpu().numpy(), dm.cpu().numpy()
    # both FP64: transform vs direct summation, errors ~ u log M vs u sqrt(M)
    assert np.abs(fft - dm).max() <= 1e-12 * np.abs(dm).max()


def test_fft_matches_reference_pocketfft(env):
    torch, sq, S = env
    from oracle.problems import planted_problem
    p = planted_problem(8192, 24, 1e3, 1e-6, 2)
    op = sq.make_sketch(8192, 72, "dct2", seed=9)
    ref = R.sketch_apply(R.draw_sketch(8192, 72, "dct2", seed=9), p.a)
    for level, tol in (("binary64", 1e-13), ("binary32", 3e-6)):
        data = p.a.astype(R.LEVEL_DTYPE[level])
        got = sq.apply_sketch(op, data)            # auto engine -> FFT for M % 4096 == 0
        ref_l = R.sketch_apply(R.draw_sketch(8192, 72, "dct2", seed=9), data)
        assert np.abs(got - ref_l).max() <= tol * np.abs(ref_l).max(), level
    assert np.abs(sq.apply_sketch(op, p.a) - ref).max() <= 1e-13 * np.abs(ref).max()


def test_fft_row_shards_sum_to_full(env):
    torch, sq, S = env
    m, n, d = 16384, 40, 120
    a = torch.from_numpy(R.philox(4, 3).standard_normal((m, n))).cuda()
    op = sq.make_sketch(m, d, "dct2", seed=1)
    full, _ = _sum(env, op, a, 64, "fft")
    acc = None
    cut = [0, 5000, 12000, m]
    for lo, hi in zip(cut[:-1], cut[1:]):
        acc, _ = _sum(env, op, a[lo:hi].contiguous(), 64, "fft", row_offset=lo, out=acc, accumulate=acc is not None)
    full, acc = full.cpu().numpy(), acc.cpu().numpy()
    assert np.abs(full - acc).max() <= 1e-12 * np.abs(full).max()


def test_fft_binary32_overflow_flag(env):
    torch, sq, S = env
    a = torch.ones((4096, 8), dtype=torch.float64, device="cuda")
    a[100, 3] = 1e300
    op = sq.make_sketch(4096, 24, "dct2", seed=1)
    _, flag = _sum(env, op, a, 32, "fft")
    assert flag == 1


@pytest.mark.parametrize("kappa,prec", [(1e10, "auto"), (1e6, "auto"), (1e3, "double")])
def test_pipeline_fft_levels_vs_oracle(env, kappa, prec):
    torch, sq, S = env
    from oracle.problems import planted_problem
    p = planted_problem(8192, 48, kappa, 1e-8, 7)
    got = sq.algorithm1_pipeline(p.a, p.b, method="pne", precision=prec, seed=7, x_star=p.x_star)
    ref = R.pipeline(p.a, p.b, method="pne", precision=prec, seed=7, x_star=p.x_star, diagnostics=False)
    assert got.preconditioner.computed_in.name == ref.pre.level
    assert got.relative_error <= max(10 * ref.relative_error, 1e-14)
    assert got.preconditioner.kappa_ap <= 10


@pytest.mark.parametrize("level", [16, 32])
def test_fft_low_levels_match_dense(env, passb, level):
    """binary16 / binary32: the FFT path demotes A on load exactly like the dense
    DMMA path (same level rounding and overflow flag), then transforms in binary32 like
    the reference (src/sketch.py:163-167: pocketfft on float32 data; pass B sums in
    FP64), so it agrees with the FP64 dense sum to binary32 transform roundoff."""
    torch, sq, S = env
    m, n, d = 1 << 16, 48, 144
    a = torch.from_numpy(R.philox(level, 3).standard_normal((m, n)) * 3.0).cuda()
    op = sq.make_sketch(m, d, "dct2", seed=5)
    fft, f1 = _sum(env, op, a, level, "fft")
    dm, f2 = _sum(env, op, a, level, "dmma")
    assert f1 == f2 == 0
    fft, dm = fft.cpu().numpy(), dm.cpu().numpy()
    assert np.abs(fft - dm).max() <= 4e-6 * np.abs(dm).max()
    big = a.clone()
    big[7, 3] = 1e6 if level == 16 else 1e300
    assert _sum(env, op, big, level, "fft")[1] == 1


def test_fft_tall_m1_beyond_pass_b_table(env):
    """M1 = M / 1024 = 16384 (config 4's 16M rows): no shared-memory twiddle table limit."""
    torch, sq, S = env
    m, n, d = 1 << 24, 8, 24
    g = torch.Generator(device="cuda").manual_seed(3)
    a = torch.randn(m, n, dtype=torch.float64, device="cuda", generator=g)
    op = sq.make_sketch(m, d, "dct2", seed=2)
    fft, f1 = _sum(env, op, a, 64, "fft")
    dm, f2 = _sum(env, op, a, 64, "dmma")
    fft, dm = fft.cpu().numpy(), dm.cpu().numpy()
    assert np.abs(fft - dm).max() <= 1e-11 * np.abs(dm).max()


@pytest.mark.parametrize("m,n,d,level", [(4096, 20, 60, 64), (65536, 130, 390, 32), (1 << 20, 64, 6144, 16)])
def test_device_request_planning_equals_host(env, monkeypatch, m, n, d, level):
    """pass-B request lists built on the device (plan_requests, no host round trip) give
    the same sketch, bit for bit, as the host construction (SK_FFT_HOST_PLAN=1)."""
    torch, sq, S = env
    a = torch.from_numpy(R.philox(m + d, 5).standard_normal((m, n))).cuda()
    op = sq.make_sketch(m, d, "dct2", seed=4)
    dev, _ = _sum(env, op, a, level, "fft")
    monkeypatch.setenv("SK_FFT_HOST_PLAN", "1")
    host, _ = _sum(env, op, a, level, "fft")
    assert torch.equal(dev, host)
