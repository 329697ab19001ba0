"""Two ranks of the row-sharded pipeline with the PRODUCTION arithmetic (DeviceOps:
libsklsq kernels) on one GPU.

Both processes drive cuda:0 and all-reduce through gloo (device tensors staged via
the host), so the device-side pieces that only the sharded path exercises run for
real: global row offsets in the tcgen05 (binary16) and FFT (binary32) sketches, the
all-reduced kappa0 Gram on the INT8 engine, the chunked TRSM -> Gram, and the
cross-rank agreement on a rank-local failure.  The kernels of the two ranks never
wait on each other (the exchange is host-side), so sharing one GPU is safe; NCCL
itself needs one GPU per rank and is exercised by bench.py --gpus N.

Reference semantics per rank: src/solvers.py:282-324.
"""
import math
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import restatement as R
from oracle.problems import planted_problem

pytestmark = pytest.mark.gpu

CASES = [  # (m, n, kappa, rho, seed, method, precision, gram engine, A_p chunk rows)
    (8192, 256, 10.0, 1e-6, 5, "hpne", "auto", "auto", 0),      # binary16: tcgen05 sketch, row offsets
    (8192, 256, 1e4, 1e-6, 6, "pne", "auto", "ozaki", 0),       # binary32: FFT sketch, INT8 Grams
    (8192, 256, 1e2, 1e-6, 7, "hpne", "single", "ozaki", 1024),  # chunked TRSM -> INT8 Gram
    (6000, 200, 1e6, 1e-6, 8, "pne", "half", "auto", 700),       # escalation + chunked, odd chunks
]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2603_16644_b200 as sq
    from paper_2603_16644_b200 import dense, solvers
    from paper_2603_16644_b200.distributed import algorithm1_pipeline_sharded
    out = []
    for (m, n, kappa, rho, seed, method, prec, engine, chunk) in CASES:
        p = planted_problem(m, n, kappa, rho, seed)
        cut = [0, m // 3, m]
        lo, hi = cut[rank], cut[rank + 1]
        dense.GRAM_ENGINE = engine
        solvers.AP_CHUNK_ROWS = chunk or None
        try:
            a = torch.from_numpy(p.a[lo:hi].copy()).cuda()
            b = torch.from_numpy(p.b[lo:hi].copy()).cuda()
            rep = algorithm1_pipeline_sharded(a, b, method=method, precision=prec, seed=seed, x_star=p.x_star)
            out.append((rep.x_hat, rep.preconditioner.computed_in.name,
                        rep.escalated_from.name if rep.escalated_from else None, rep.relative_error,
                        rep.residual_norm))
        finally:
            dense.GRAM_ENGINE = "auto"
            solvers.AP_CHUNK_ROWS = None
    # a non-finite entry in rank 1's shard raises on both ranks
    p = planted_problem(4096, 64, 1e2, 1e-6, 9)
    lo, hi = (0, 2048) if rank == 0 else (2048, 4096)
    a = p.a[lo:hi].copy()
    if rank == 1:
        a[5, 5] = np.inf
    try:
        algorithm1_pipeline_sharded(torch.from_numpy(a).cuda(), torch.from_numpy(p.b[lo:hi].copy()).cuda())
        out.append("no error")
    except ValueError:
        out.append("ValueError")
    torch.cuda.synchronize()
    q.put((rank, out))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(900)
def test_two_ranks_device_ops_match_single_gpu_and_oracle():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p_ in procs:
        p_.start()
    results = dict(q.get(timeout=800) for _ in procs)
    for p_ in procs:
        p_.join(timeout=120)
        assert p_.exitcode == 0
    import paper_2603_16644_b200 as sq
    for i, (m, n, kappa, rho, seed, method, prec, engine, chunk) in enumerate(CASES):
        r0, r1 = results[0][i], results[1][i]
        assert np.array_equal(r0[0], r1[0]), "replicated n x n work must give identical x on every rank"
        assert r0[1:3] == r1[1:3]
        p = planted_problem(m, n, kappa, rho, seed)
        ref = R.pipeline(p.a, p.b, method=method, precision=prec, seed=seed, x_star=p.x_star, diagnostics=False)
        single = sq.algorithm1_pipeline(p.a, p.b, method=method, precision=prec, seed=seed, x_star=p.x_star,
                                        diagnostics=False)
        assert r0[1] == ref.pre.level == single.preconditioner.computed_in.name, (i, r0[1], ref.pre.level)
        assert r0[2] == ref.escalated_from
        assert r0[3] <= max(10 * ref.relative_error, 1e-14), (i, r0[3], ref.relative_error)
        assert r0[4] == pytest.approx(ref.residual_norm, rel=1e-6)
        assert np.linalg.norm(r0[0] - single.x_hat) <= max(1e-9, 50 * ref.relative_error) * np.linalg.norm(p.x_star)
    assert results[0][-1] == results[1][-1] == "ValueError"
