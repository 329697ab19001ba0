"""Row-chunked hybrid CPU oracle for sizes the op-for-op restatement cannot reach
(SURVEY §8(c) "Restatement needed at scale").  TEST INFRASTRUCTURE (see
oracle/__init__.py): used by tests/, tools/config3_parity.py and bench.py's CPU
legs, never by the product.

Follows Algorithm 1 line by line (src/solvers.py:168-324, src/precision.py:153-276)
with the reference's own arithmetic wherever it is feasible at config-3 size, and a
LAPACK/BLAS step with the same mathematics where the reference's Python loops are
not (m-sized substitution):

  _check_system        restatement.checked_system (src/solvers.py:87-96)
  kappa0               G = A^T A (numpy BLAS, as src/precision.py:230, row-chunked),
                       then the reference's Cholesky + Hager on G (restatement)
  demotion + sketch    restatement.demote / draw_sketch / sketch_apply: the reference's
                       Philox operator and pocketfft DCT-II (binary16 input transformed
                       in binary32), sampled and scaled in the level; pocketfft runs with
                       `workers` threads, which transforms each column independently
                       (bitwise the single-worker result)
  level QR             binary16: the C restatement of the emulated Householder
                       (oracle/fast.py, bitwise the reference's R); binary32/64: the
                       restatement's native Householder (R only; Q is never used)
  A_p = A R^-1         scipy.linalg.solve_triangular (LAPACK dtrsm) per row chunk
                       instead of the reference's column loop (src/dense.py:231-236)
  Gram + rhs           sum over row chunks of A_p,c^T A_c (HPNE) / A_p,c^T A_p,c (PNE)
                       and A_p,c^T b_c (numpy BLAS; A_p never materialised)
  n x n                the reference's LU / Cholesky (+ LU fallback) / substitution
                       (restatement.lu_pivoted_solve, spd_solve, tri_solve)
  report               r = A x - b, norms (src/solvers.py:99-117)

Diagnostics (kappa(R_s), kappa(A_p)) are not computed.
"""

from __future__ import annotations

import math
import time

import numpy as np
import scipy.linalg

from . import restatement as R

CHUNK = 1 << 17


def _gram_chunked(a, chunk=CHUNK):
    n = a.shape[1]
    g = np.zeros((n, n))
    for r0 in range(0, a.shape[0], chunk):
        c = a[r0:r0 + chunk]
        g += c.T @ c
    return g


def kappa0(a, chunk=CHUNK):
    """estimate_log10_condition (src/precision.py:205-251) -> (kappa0, overflowed)."""
    with np.errstate(over="ignore", invalid="ignore", under="ignore"):
        g = _gram_chunked(a, chunk)
    return R.kappa0_from_gram(g)


COLBLOCK = 128


def checked_system(a, b, chunk=CHUNK):
    """src/solvers.py:87-96 without the full-size copies (f64 C-order input is used
    in place; the finiteness scan runs per row chunk)."""
    a = np.asarray(a)
    if a.ndim != 2:
        raise ValueError(f"a must be 2-D, got ndim={a.ndim}")
    if a.dtype != np.float64 or not a.flags.c_contiguous:
        return R.checked_system(a, b)
    for r0 in range(0, a.shape[0], chunk):
        if not np.isfinite(a[r0:r0 + chunk]).all():
            raise ValueError("a contains non-finite entries")
    b = np.asarray(b, dtype=np.float64)
    if b.ndim != 1:
        raise ValueError(f"b must be 1-D, got ndim={b.ndim}")
    if a.shape[0] < a.shape[1]:
        raise R.DimensionMismatch(f"need rows >= cols, got {a.shape}")
    if b.shape[0] != a.shape[0]:
        raise R.DimensionMismatch(f"b length {b.shape[0]} != rows {a.shape[0]}")
    return a, b


def sketch(a, level, d_factor=3.0, transform="dct2", seed=0, workers=-1, colblock=COLBLOCK):
    """build_preconditioner's demotion + apply_sketch (src/solvers.py:188-195), in
    blocks of columns: demotion, sign flip, transform, row sampling and scaling act on
    each column independently, so the blocked result is bitwise the whole-matrix one
    (and a 4M-row A needs no full-size temporaries)."""
    m, n = a.shape
    d = int(math.ceil(d_factor * n))
    op = R.draw_sketch(m, d, transform, seed)
    out = None
    import scipy.fft
    with scipy.fft.set_workers(workers):
        for c0 in range(0, n, colblock):
            data, over = R.demote(np.ascontiguousarray(a[:, c0:c0 + colblock]), level)
            if over:
                raise R.Overflow(f"input exceeds the {level} range")
            blk = R.sketch_apply(op, data)
            if out is None:
                out = np.empty((d, n), dtype=blk.dtype)
            out[:, c0:c0 + colblock] = blk
    return out, op


def level_r(a_s, level):
    """qr_in_precision(a_s, level).r (src/precision.py:153-202)."""
    if level == "binary16":
        from .fast import qr_at_level16
        return qr_at_level16(a_s)
    data = a_s.astype(np.float64) if level == "binary64" else R.demote(a_s, level)[0]
    if level == "binary32" and R.demote(a_s, level)[1]:
        raise R.Overflow("input exceeds the binary32 range")
    return R.householder_steps(data)[2].astype(np.float64)


def trsm_gram(a, b, r_s, method, chunk=CHUNK):
    """precondition_matrix + the PNE / HPNE Gram and rhs, per row chunk."""
    n = a.shape[1]
    g, rhs = np.zeros((n, n)), np.zeros(n)
    zeros = np.nonzero(np.diagonal(r_s) == 0)[0]
    if zeros.size:
        raise R.SingularTriangular(f"zero diagonal entry at index {zeros[0]}")
    for r0 in range(0, a.shape[0], chunk):
        ac = a[r0:r0 + chunk]
        apc = scipy.linalg.solve_triangular(r_s, ac.T, trans="T", lower=False, check_finite=False).T
        g += apc.T @ (apc if method == "pne" else ac)
        rhs += apc.T @ b[r0:r0 + chunk]
    return g, rhs


def pipeline(a, b, method="pne", precision="auto", d_factor=3.0, transform="dct2", seed=0, x_star=None,
             chunk=CHUNK, workers=-1, timings=None):
    """algorithm1_pipeline (src/solvers.py:282-324) at scale -> restatement.Report."""
    tm = timings if timings is not None else {}
    a, b = checked_system(a, b, chunk)
    if method not in ("pne", "hpne"):
        raise ValueError(f"pipeline method must be pne or hpne, got {method!r}")
    t0 = time.perf_counter()
    decision = None
    if precision == "auto":
        t = time.perf_counter()
        k0, over = kappa0(a, chunk)
        decision = (k0, R.choose_level(k0, over), over)
        level = decision[1]
        tm["kappa0"] = time.perf_counter() - t
    else:
        level = R.canonical_level(precision)
    failed = None
    while True:                                  # src/solvers.py:255-279: one escalation
        try:
            t = time.perf_counter()
            a_s, op = sketch(a, level, d_factor, transform, seed, workers)
            tm["sketch"] = tm.get("sketch", 0.0) + time.perf_counter() - t
            t = time.perf_counter()
            r_s = level_r(a_s, level)
            tm["level_qr"] = tm.get("level_qr", 0.0) + time.perf_counter() - t
            if (np.diagonal(r_s) == 0).any():
                raise R.RankDeficient("sketched factor has a zero diagonal entry")
            break
        except R.RankDeficient:
            wider = R.WIDER.get(level)
            if failed is not None or wider is None:
                raise
            failed, level = level, wider
    t = time.perf_counter()
    g, rhs = trsm_gram(a, b, r_s, method, chunk)
    tm["trsm_gram"] = time.perf_counter() - t
    t = time.perf_counter()
    if method == "pne":
        try:
            y = R.spd_solve(g, rhs)
        except R.NotPositiveDefinite:
            y = R.lu_pivoted_solve(g, rhs)
        x = R.tri_solve(r_s, y)
    else:
        x = R.lu_pivoted_solve(g, rhs)
    tm["nxn"] = time.perf_counter() - t
    pre = R.Pre(r_s, level, math.nan, math.nan, {"m": a.shape[0], "d": op.d, "transform": transform, "seed": seed})
    rep = R.report(method, a, b, x, t0, x_star, pre)
    rep.decision = decision
    rep.escalated_from = failed
    rep.wall_ms = (time.perf_counter() - t0) * 1e3
    rep.timings = tm
    return rep
