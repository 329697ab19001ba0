"""Row-sharded Algorithm 1 over torch.distributed (one process per GPU).

A and b are split into contiguous row blocks; rank g holds rows
[offset_g, offset_g + m_g) and uses GLOBAL row indices for the sketch operator
(signs, DCT phases), so partial results are exact pieces of the global ones.
Every m-sized pass is local; the only exchanges are all-reduces of small
results:

  ||A||_F^2, ||r||^2            sum of 2 scalars
  kappa0 Gram   A_g^T A_g       n x n   f64
  sketch        Omega_g A_g     d x n   f64   (rounded to the level AFTER the sum)
  demotion overflow flag        max
  Gram + rhs    A_p,g^T [A_g|b_g] or A_p,g^T [A_p,g|b_g]   n x (n+1) f64

The n x n work (kappa0 Cholesky/Hager, level QR of the sketch, LU/Cholesky) is
replicated: every rank holds bit-identical inputs after the all-reduce, so all
ranks take the same decisions (precision level, escalation, Cholesky->LU
fallback) without further communication.

The arithmetic is behind a small `ops` object so that the orchestration can be
exercised on CPU with the gloo backend in the tests (with oracle arithmetic);
production uses `DeviceOps` (libsklsq kernels + NCCL over NVLink).
"""

from __future__ import annotations

import math
import time

import numpy as np
import torch
import torch.distributed as dist

from .errors import DimensionMismatch, NotPositiveDefinite, RankDeficient
from .precision import BINARY64, PrecisionDecision, PrecisionLevel, level_from_name, next_higher, select_precision
from .sketch import DCT2, make_sketch
from .solvers import Preconditioner, SolveReport, _Stages


class DeviceOps:
    """libsklsq kernels on this rank's GPU."""

    def validate(self, a):
        from .device import as_dmat
        d = as_dmat(a)
        return d.t, d.frob2

    def vector(self, b, m):
        from .device import as_dvec
        return as_dvec(b, m)

    def _dmat(self, t):
        """t as a DMat carrying cached column statistics (the INT8 Gram engine scans a
        matrix used by two Grams once: A in the kappa0 SYRK and in A_p^T A)."""
        from .dense import _colstats, _gram_engine
        from .device import DMat
        key = (t.data_ptr(), tuple(t.shape), t.stride(0))
        cache = getattr(self, "_cs", None)
        if cache is not None and cache[0] == key:
            return DMat(t, None, "torch", cache[1])
        m, n = t.shape
        cs = _colstats(t) if _gram_engine(m, n, False, None) == "ozaki" else None
        self._cs = (key, cs)
        return DMat(t, None, "torch", cs)

    def gram(self, x, y=None):
        from .dense import _gram
        return _gram(self._dmat(x), None if y is None else self._dmat(y))

    def gram_and_rhs(self, x, y, b):
        """(X^T Y or X^T X, X^T b) with the memory-bound GEMV on a side stream."""
        from .solvers import _gram_and_rhs
        return _gram_and_rhs(x, None if y is None else self._dmat(y), b)

    def gemv_t(self, x, v):
        from .dense import _gemv_t
        return _gemv_t(x, v)

    def make_operator(self, m, d, transform, seed):
        # signs drawn on the device (bitwise make_sketch's), rows on the host
        from .sketch import _make_sketch_dev
        op, self._dsk = _make_sketch_dev(m, d, transform, seed)
        return op

    def sketch_partial(self, op, a_local, level, row_offset):
        from .sketch import DeviceSketch, _sketch_sum
        dsk = getattr(self, "_dsk", None)
        if dsk is None or dsk.op is not op:
            dsk = DeviceSketch(op)
        total, flag = _sketch_sum(dsk, a_local, level.code, row_offset=row_offset)
        return total, flag.to(torch.float64)

    def sketch_level_qr(self, total, op, level):
        from .precision import _qr_level_dev
        from .sketch import _sketch_finalize
        a_s, _ = _sketch_finalize(total, op, level)
        return _qr_level_dev(a_s, level, op.d, total.shape[0])

    def chunk_rows(self, m, n, device):
        from .solvers import _ap_chunk_rows
        return _ap_chunk_rows(m, n, device)

    def trsm_gram(self, a, r, b, method, rows):
        """TRSM -> Gram per row chunk (A_p never materialised; config 4 at P = 2)."""
        from .solvers import _trsm_gram_chunked
        from .device import DMat
        return _trsm_gram_chunked(self._dmat(a) if method != "pne" else DMat(a, None, "torch"), r, b, method, rows)

    def trsm(self, a, r):
        # A_p in the per-device scratch buffer of algorithm1_pipeline (no 64 GB
        # allocation per solve); handed back by release()
        from .dense import _trsm
        from .solvers import _AP_SCRATCH
        self._ap = _AP_SCRATCH.take(a.shape[0], a.shape[1], a.device)
        return _trsm(a, r, out=self._ap[1])

    def release(self):
        from .solvers import _AP_SCRATCH
        ap = getattr(self, "_ap", None)
        if ap is not None:
            _AP_SCRATCH.give(*ap)
            self._ap = None
        self._cs = None

    def chol_solve(self, g, rhs):
        from .dense import _chol_solve
        return _chol_solve(g, rhs)

    def lu_solve(self, g, rhs):
        from .dense import _lu_solve
        return _lu_solve(g, rhs)

    def trsv(self, r, y):
        from .dense import _trsv
        return _trsv(r, y)

    def kappa0_from_gram(self, g):
        from .precision import _kappa0_from_gram
        return _kappa0_from_gram(g)

    def residual_sq(self, a, x, b):
        """(||A_g x - b_g||^2, ||x||^2) by the sk_residual streaming kernel."""
        import ctypes as C
        from . import _lib
        from .device import WORKSPACE, call, stream_handle
        m, n = a.shape
        out = (C.c_double * 2)()
        wp, wn = WORKSPACE.get(_lib.lib().sk_matrix_stats_workspace(m, n))
        call("sk_residual", a.data_ptr(), m, n, a.stride(0), x.data_ptr(), b.data_ptr(), None, out, wp, wn,
             stream_handle())
        return float(out[0]), float(out[1])


def _world() -> int:
    return dist.get_world_size() if (dist.is_available() and dist.is_initialized()) else 1


def _allreduce(t: torch.Tensor, op=None) -> torch.Tensor:
    """In-place all-reduce (SUM by default).  NCCL reduces device tensors over NVLink;
    under gloo (CPU tests, or ranks sharing one GPU in the device tests) a CUDA tensor
    is staged through host memory."""
    if _world() > 1:
        op = op or dist.ReduceOp.SUM
        if t.is_cuda and dist.get_backend() == "gloo":
            h = t.cpu()
            dist.all_reduce(h, op=op)
            t.copy_(h)
        else:
            dist.all_reduce(t, op=op)
    return t


_ERR_CLASSES = None


def _agree(fn, *args, **kw):
    """Run a rank-local step and agree on its outcome before anyone enters the next
    collective: if any rank raised, every rank raises (the failing rank its own
    exception, the others the same class naming the failing rank), so one bad shard
    cannot leave the other ranks waiting in an all-reduce."""
    global _ERR_CLASSES
    from . import errors as E
    if _ERR_CLASSES is None:
        _ERR_CLASSES = [ValueError, E.DimensionMismatch, E.Overflow, E.RankDeficient, E.SingularTriangular,
                        E.NumericallySingular, E.NotPositiveDefinite, E.NoConvergence, E.SketchLsqError, RuntimeError]
    exc, code = None, 0
    try:
        out = fn(*args, **kw)
    except Exception as ex:  # noqa: BLE001
        exc, out = ex, None
        code = next((i + 1 for i, c in enumerate(_ERR_CLASSES) if isinstance(ex, c)), len(_ERR_CLASSES))
    if _world() > 1:
        dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else "cpu"
        flag = torch.tensor([code, dist.get_rank() if code else -1], dtype=torch.int64, device=dev)
        _allreduce(flag, dist.ReduceOp.MAX)
        code, who = int(flag[0]), int(flag[1])
        if code and exc is None:
            raise _ERR_CLASSES[min(code, len(_ERR_CLASSES)) - 1](f"rank {who} failed this step")
    if exc is not None:
        raise exc
    return out


def _row_layout(m_local: int, device) -> tuple[int, int]:
    """-> (global m, this rank's row offset) from the shard sizes."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return m_local, 0
    world, rank = dist.get_world_size(), dist.get_rank()
    sizes = torch.zeros(world, dtype=torch.int64, device=device)
    sizes[rank] = m_local
    dist.all_reduce(sizes)
    sizes = sizes.cpu().tolist()
    return int(sum(sizes)), int(sum(sizes[:rank]))


def algorithm1_pipeline_sharded(a_local, b_local, method="pne", precision="auto", d_factor=3.0, transform=DCT2,
                                seed=0, x_star=None, *, ops=None, diagnostics=False, stage_timing=False):
    """Algorithm 1 (src/solvers.py:282-324) on row shards; returns the same
    SolveReport on every rank.  `diagnostics` is accepted for signature parity;
    the sharded path does not compute kappa_rs / kappa_ap (NaN)."""
    ops = ops or DeviceOps()
    stages = _Stages(stage_timing and torch.cuda.is_available())
    stages.mark("check")

    def check():
        if method not in ("pne", "hpne"):
            raise ValueError(f"pipeline method must be pne or hpne, got {method!r}")
        if not isinstance(precision, PrecisionLevel) and precision != "auto":
            level_from_name(precision)
        a_, frob2_ = ops.validate(a_local)
        return a_, frob2_, ops.vector(b_local, a_.shape[0])

    a, frob2_local, b = _agree(check)      # a bad shard raises on every rank
    m_local, n = a.shape
    m, offset = _row_layout(m_local, a.device)
    if m < n:
        raise DimensionMismatch(f"need rows >= cols, got {(m, n)}")
    t0 = time.perf_counter()
    decision = None
    if isinstance(precision, PrecisionLevel):
        level = precision
    elif precision == "auto":
        stages.mark("kappa0")
        g = _allreduce(ops.gram(a))
        k0, over = ops.kappa0_from_gram(g)
        decision = PrecisionDecision(kappa0=k0, selected=select_precision(k0, over), overflowed=over)
        level = decision.selected
    else:
        level = level_from_name(precision)
    d = int(math.ceil(d_factor * n))
    if d < n:
        raise ValueError(f"d_factor {d_factor} gives d={d} < n={n}")
    mk = getattr(ops, "make_operator", None)
    op = mk(m, d, transform, seed) if mk is not None else make_sketch(m, d, transform, seed)
    escalated_from = None
    while True:
        try:
            stages.mark("sketch")
            total, flag = ops.sketch_partial(op, a, level, offset)
            _allreduce(total)
            _allreduce(flag, dist.ReduceOp.MAX if dist.is_available() and dist.is_initialized() else None)
            if float(flag.reshape(-1)[0]) > 0:
                from .errors import Overflow
                raise Overflow(f"input exceeds the {level.name} range")
            stages.mark("level_qr")
            r_s = ops.sketch_level_qr(total, op, level)
            if bool((torch.diagonal(r_s) == 0).any()):
                raise RankDeficient("sketched factor has a zero diagonal entry")
            break
        except RankDeficient:
            wider = next_higher(level)
            if escalated_from is not None or wider is None:
                raise
            escalated_from, level = level, wider
    def local_gram():
        rows = ops.chunk_rows(m_local, n, a.device) if hasattr(ops, "chunk_rows") else 0
        if rows:
            stages.mark("trsm_gram")
            return ops.trsm_gram(a, r_s, b, method, rows)
        stages.mark("trsm")
        a_p = ops.trsm(a, r_s)
        stages.mark("gram")
        if hasattr(ops, "gram_and_rhs"):
            return ops.gram_and_rhs(a_p, None if method == "pne" else a, b)
        return (ops.gram(a_p) if method == "pne" else ops.gram(a_p, a)), ops.gemv_t(a_p, b)

    try:
        g, rhs = _agree(local_gram)
        g, rhs = _allreduce(g), _allreduce(rhs)
    finally:
        if hasattr(ops, "release"):
            ops.release()
    stages.mark("nxn")
    if method == "pne":
        try:
            y = ops.chol_solve(g, rhs)
        except NotPositiveDefinite:
            y = ops.lu_solve(g, rhs)
        x = ops.trsv(r_s, y)
    else:
        x = ops.lu_solve(g, rhs)
    stages.mark("report")
    rr, xx = ops.residual_sq(a, x, b)
    sums = _allreduce(torch.tensor([rr, frob2_local], dtype=torch.float64, device=a.device))
    stages.mark("end")
    rr, frob2 = float(sums[0]), float(sums[1])
    x_hat = x.detach().cpu().numpy()
    res = math.sqrt(rr)
    denom = math.sqrt(frob2) * math.sqrt(xx)
    rel_err = None
    if x_star is not None:
        xs = np.asarray(x_star.detach().cpu() if isinstance(x_star, torch.Tensor) else x_star, dtype=np.float64)
        rel_err = float(np.linalg.norm(x_hat - xs) / np.linalg.norm(xs))
    pre = Preconditioner(r_s=r_s if r_s.is_cuda else r_s.detach().cpu().numpy(), computed_in=level,
                         kappa_rs=math.nan, kappa_ap=math.nan, sketch_descriptor=op.descriptor())
    rep = SolveReport(method=method, x_hat=x_hat, residual_norm=res,
                      relative_residual=res / denom if denom > 0 else math.inf, relative_error=rel_err,
                      wall_ms=(time.perf_counter() - t0) * 1e3, preconditioner=pre,
                      precision_decision=decision, escalated_from=escalated_from, stage_ms=stages.result())
    return rep
