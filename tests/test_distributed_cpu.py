"""Multi-process (world_size 2, gloo, CPU) test of the row-sharded Algorithm-1
orchestration in paper_2603_16644_b200.distributed.

The GPU kernels are replaced by oracle arithmetic (OracleOps) so the sharding
logic itself -- global row offsets for the sketch operator, all-reduce of the
kappa0 Gram, of the sketch partials (rounded to the level after the sum), of
the Gram+rhs and of the residual/Frobenius scalars, replicated n x n decisions
and escalation -- is exercised here without a GPU."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import restatement as R
from oracle.problems import planted_problem


class OracleOps:
    def validate(self, a):
        t = torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64))
        if not torch.isfinite(t).all():
            raise ValueError("a contains non-finite entries")      # src/dense.py:63-64
        return t, float((t * t).sum())

    def vector(self, b, m):
        import paper_2603_16644_b200 as sq
        t = torch.as_tensor(np.asarray(b, dtype=np.float64))
        if t.shape[0] != m:
            raise sq.DimensionMismatch(f"b length {t.shape[0]} != rows {m}")
        return t

    def gram(self, x, y=None):
        y = x if y is None else y
        return torch.from_numpy(x.numpy().T @ y.numpy())

    def gemv_t(self, x, v):
        return torch.from_numpy(x.numpy().T @ v.numpy())

    def sketch_partial(self, op, a_local, level, row_offset):
        sk = R.Sketch(op.m, op.d, op.transform, op.seed, op.signs, op.sampled_rows)
        omega = R.sketch_matrix(sk) / math.sqrt(sk.m_pad / sk.d)          # unscaled S F D
        m_local = a_local.shape[0]
        data, over = R.demote(a_local.numpy(), level.name)
        part = omega[:, row_offset:row_offset + m_local] @ data.astype(np.float64)   # d x n
        return torch.from_numpy(np.ascontiguousarray(part.T)), torch.tensor([float(over)], dtype=torch.float64)

    def sketch_level_qr(self, total, op, level):
        import paper_2603_16644_b200 as sq
        s = total.numpy().T                                     # d x n, exact sampled transform
        scale = math.sqrt(op.m_pad / op.d)
        if level.name == "binary16":
            a_s = s.astype(np.float32).astype(np.float16) * np.float16(scale)
        elif level.name == "binary32":
            a_s = s.astype(np.float32) * np.float32(scale)
        else:
            a_s = s * scale
        try:
            return torch.from_numpy(R.qr_at_level(a_s, level.name)[1])
        except R.RankDeficient as ex:
            raise sq.RankDeficient(str(ex)) from None

    def trsm(self, a, r):
        return torch.from_numpy(np.ascontiguousarray(R.tri_solve(r.numpy(), a.numpy().T, transposed=True).T))

    def chol_solve(self, g, rhs):
        import paper_2603_16644_b200 as sq
        try:
            return torch.from_numpy(R.spd_solve(g.numpy(), rhs.numpy()))
        except R.NotPositiveDefinite as ex:
            raise sq.NotPositiveDefinite(str(ex)) from None

    def lu_solve(self, g, rhs):
        return torch.from_numpy(R.lu_pivoted_solve(g.numpy(), rhs.numpy()))

    def trsv(self, r, y):
        return torch.from_numpy(R.tri_solve(r.numpy(), y.numpy()))

    def kappa0_from_gram(self, g):
        return R.kappa0_from_gram(g.numpy())

    def residual_sq(self, a, x, b):
        r = a.numpy() @ x.numpy() - b.numpy()
        return float(r @ r), float(x.numpy() @ x.numpy())


CASES = [  # (m, n, kappa, rho, seed, method, precision)
    (600, 40, 1e2, 1e-8, 4, "hpne", "auto"),
    (600, 40, 1e6, 1e-8, 4, "pne", "auto"),
    (600, 40, 1e6, 1e-8, 6, "pne", "half"),      # binary16 collapses -> escalation to binary32
    (601, 33, 1e10, 1e-6, 2, "hpne", "auto"),    # overflowed kappa0 -> binary64, odd shard split
]


def _worker(rank, world, port, cuts, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2603_16644_b200.distributed import algorithm1_pipeline_sharded
    out = []
    for (m, n, kappa, rho, seed, method, prec) in CASES:
        p = planted_problem(m, n, kappa, rho, seed)
        lo, hi = cuts(m)[rank], cuts(m)[rank + 1]
        rep = algorithm1_pipeline_sharded(p.a[lo:hi], p.b[lo:hi], method=method, precision=prec, seed=seed,
                                          x_star=p.x_star, ops=OracleOps())
        out.append((rep.x_hat, rep.preconditioner.computed_in.name,
                    rep.escalated_from.name if rep.escalated_from else None, rep.relative_error,
                    rep.residual_norm, rep.preconditioner.sketch_descriptor))
    q.put((rank, out))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _uneven(m):
    return [0, m // 3, m]


@pytest.mark.timeout(300)
def test_two_rank_gloo_matches_single_process_and_oracle():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, _uneven, q)) for r in range(2)]
    for p_ in procs:
        p_.start()
    results = dict(q.get(timeout=240) for _ in procs)
    for p_ in procs:
        p_.join(timeout=60)
        assert p_.exitcode == 0
    from paper_2603_16644_b200.distributed import algorithm1_pipeline_sharded
    for i, (m, n, kappa, rho, seed, method, prec) in enumerate(CASES):
        r0, r1 = results[0][i], results[1][i]
        assert np.array_equal(r0[0], r1[0])                  # replicated n x n work: identical x on every rank
        assert r0[1:3] == r1[1:3]
        p = planted_problem(m, n, kappa, rho, seed)
        single = algorithm1_pipeline_sharded(p.a, p.b, method=method, precision=prec, seed=seed, x_star=p.x_star,
                                             ops=OracleOps())
        ref = R.pipeline(p.a, p.b, method=method, precision=prec, seed=seed, x_star=p.x_star, diagnostics=False)
        assert r0[1] == single.preconditioner.computed_in.name == ref.pre.level
        assert r0[2] == (single.escalated_from.name if single.escalated_from else None) == ref.escalated_from
        assert r0[3] <= max(10 * ref.relative_error, 1e-14)
        assert np.linalg.norm(r0[0] - single.x_hat) <= max(1e-6, 50 * ref.relative_error) * np.linalg.norm(single.x_hat)
        assert r0[4] == pytest.approx(ref.residual_norm, rel=1e-6)
        assert r0[5] == {"m": m, "d": int(math.ceil(3.0 * n)), "transform": "dct2", "seed": seed}


def _fail_worker(rank, world, port, q):
    """Rank-local validation failures must raise on EVERY rank (no rank may be left
    waiting in the next all-reduce): NaN in rank 1's shard, a short b on rank 0, a bad
    method name."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2603_16644_b200 as sq
    from paper_2603_16644_b200.distributed import algorithm1_pipeline_sharded
    p = planted_problem(300, 20, 1e2, 1e-8, 3)
    lo, hi = (0, 150) if rank == 0 else (150, 300)
    out = []
    a = p.a[lo:hi].copy()
    if rank == 1:
        a[7, 3] = np.nan
    for args, kw in (((a, p.b[lo:hi]), {}),
                     ((p.a[lo:hi], p.b[lo:hi - 1] if rank == 0 else p.b[lo:hi]), {}),
                     ((p.a[lo:hi], p.b[lo:hi]), {"method": "qr"})):
        try:
            algorithm1_pipeline_sharded(*args, ops=OracleOps(), **kw)
            out.append(None)
        except (ValueError, sq.SketchLsqError) as ex:
            out.append(type(ex).__name__)
    # the group still works afterwards: a good solve on both ranks
    rep = algorithm1_pipeline_sharded(p.a[lo:hi], p.b[lo:hi], method="pne", seed=3, x_star=p.x_star, ops=OracleOps())
    out.append(rep.relative_error < 1e-8)
    q.put((rank, out))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(180)
def test_two_rank_local_errors_raise_on_every_rank():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_fail_worker, args=(r, 2, port, q)) for r in range(2)]
    for p_ in procs:
        p_.start()
    results = dict(q.get(timeout=150) for _ in procs)
    for p_ in procs:
        p_.join(timeout=60)
        assert p_.exitcode == 0
    assert results[0][0] == "ValueError" and results[1][0] == "ValueError"             # NaN on rank 1
    assert results[0][1] == "DimensionMismatch" and results[1][1] == "DimensionMismatch"   # short b on rank 0
    assert results[0][2] == results[1][2] == "ValueError"                                # bad method
    assert results[0][3] and results[1][3]
