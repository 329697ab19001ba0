"""Dense kernels on the device, mirroring src/dense.py of the reference.

Public functions keep the reference names and argument conventions
(`triangular_solve`, `lu_solve`, `cholesky_solve`, `cholesky_factor`,
`householder_qr`, `householder_reduce`, `jacobi_singular_values`,
`condition_diagnostics`, `hager_one_norm_inverse_estimate`) and accept numpy
arrays or torch tensors.  Underscored helpers take validated device matrices and
are what the solvers call, so a pipeline never leaves the GPU.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .device import WORKSPACE, DMat, as_dmat, as_dvec, call, device, like_input, stream_handle, to_host
from .errors import DimensionMismatch, RankDeficient


@dataclass(frozen=True)
class QRFactors:
    """Thin QR factors (src/dense.py:29-34)."""

    q: np.ndarray | None
    r: np.ndarray


@dataclass(frozen=True)
class ConditionDiagnostics:
    """Spectral summary (src/dense.py:37-54)."""

    two_norm: float
    two_norm_condition: float
    singular_values: np.ndarray


# --------------------------------------------------------------- device ops --
def _rm(t: torch.Tensor) -> torch.Tensor:
    """Row-major view with unit column stride (what the C ABI expects)."""
    if t.dim() == 2 and (t.stride(1) != 1 or t.stride(0) < t.shape[1]):
        return t.contiguous()
    return t


GRAM_ENGINE = "auto"       # "dmma" (FP64 DMMA), "ozaki" (INT8 tensor cores), "auto"
OZAKI_MIN_WORK = 1 << 33   # m * n^2 above which "auto" takes the INT8 engine


def _gram_engine(m: int, n: int, accumulate: bool, engine: str | None) -> str:
    """Engine for an m x n Gram (accumulating calls sum per-call FP64 results on either
    engine, so row chunks of A_p / A take the same engine as the whole would)."""
    e = engine or GRAM_ENGINE
    if e == "auto":
        e = "ozaki" if (n >= 128 and m * n * n >= OZAKI_MIN_WORK) else "dmma"
    return e


TRSM_ENGINE = "auto"       # "dmma" (one left-looking DMMA kernel), "ozaki" (blocked, INT8 updates)
TRSM_OZAKI_MIN_N = 1025    # the blocked solve splits only above its 1024-column leaves


def _trsm_engine(m: int, n: int, inplace: bool, engine: str | None) -> str:
    e = engine or TRSM_ENGINE
    if e == "auto":
        e = "ozaki" if (n >= TRSM_OZAKI_MIN_N and m * n * n >= OZAKI_MIN_WORK) else "dmma"
    return "dmma" if inplace else e


def _colstats(t: torch.Tensor, v: torch.Tensor | None = None) -> torch.Tensor:
    """[max_k |T[k, j]| for j] + [sum_k T[k, j]^2 for j] (+ [T^T v] if v is given)
    (device, f64, 2n or 3n)."""
    t = _rm(t)
    m, n = t.shape
    out = torch.empty((3 if v is not None else 2) * n, dtype=torch.float64, device=t.device)
    lib = _lib.lib()
    wp, wn = WORKSPACE.get(lib.sk_colstats_workspace(n))
    call("sk_colstats_f64", t.data_ptr(), t.stride(0), m, n, v.data_ptr() if v is not None else None,
         out.data_ptr(), wp, wn, stream_handle())
    return out


def _gram(x: DMat | torch.Tensor, y: DMat | torch.Tensor | None = None, out: torch.Tensor | None = None,
          accumulate: bool = False, engine: str | None = None) -> torch.Tensor:
    """G = X^T Y (SYRK when y is None or y is x): FP64 DMMA, or the INT8 tensor-core
    Ozaki engine (sk_gram_ozaki_ex_f64) for large products.  A DMat operand whose
    `colstats` is set (the pipeline scans A once) passes its column statistics along.
    The INT8 engine falls back to DMMA by itself on spiky or non-finite columns."""
    xt = _rm(x.t if isinstance(x, DMat) else x)
    yt = xt if y is None else _rm(y.t if isinstance(y, DMat) else y)
    m, n = xt.shape
    if yt.shape != xt.shape:
        raise DimensionMismatch(f"gram operands {tuple(xt.shape)} vs {tuple(yt.shape)}")
    if out is None:
        out = torch.empty((n, n), dtype=torch.float64, device=xt.device)
    lib = _lib.lib()
    if _gram_engine(m, n, accumulate, engine) == "ozaki":
        syrk = xt.data_ptr() == yt.data_ptr() and xt.stride(0) == yt.stride(0)
        xmax = x.colstats if isinstance(x, DMat) else None
        ymax = (y.colstats if isinstance(y, DMat) else None) if y is not None else xmax
        wp, wn = WORKSPACE.get(max(lib.sk_gram_ozaki_workspace(m, n, int(syrk)), lib.sk_gram_workspace(m, n)))
        call("sk_gram_ozaki_acc_f64", xt.data_ptr(), xt.stride(0), yt.data_ptr(), yt.stride(0), m, n,
             xmax.data_ptr() if xmax is not None else None, ymax.data_ptr() if ymax is not None else None,
             out.data_ptr(), out.stride(0), int(accumulate), wp, wn, stream_handle())
        return out
    wsb = lib.sk_gram_workspace(m, n)
    wp, wn = WORKSPACE.get(wsb)
    call("sk_gram_f64", xt.data_ptr(), xt.stride(0), yt.data_ptr(), yt.stride(0), m, n,
         out.data_ptr(), out.stride(0), int(accumulate), wp, wn, stream_handle())
    return out


def _gemv_t(x: DMat | torch.Tensor, v: torch.Tensor, out: torch.Tensor | None = None,
            accumulate: bool = False) -> torch.Tensor:
    """out = X^T v (memory-bound)."""
    xt = _rm(x.t if isinstance(x, DMat) else x)
    m, n = xt.shape
    if out is None:
        out = torch.empty(n, dtype=torch.float64, device=xt.device)
    lib = _lib.lib()
    wp, wn = WORKSPACE.get(lib.sk_gemv_t_workspace(m, n))
    call("sk_gemv_t_f64", xt.data_ptr(), xt.stride(0), m, n, v.data_ptr(), out.data_ptr(),
         int(accumulate), wp, wn, stream_handle())
    return out


APITCH_PAD = 8   # doubles of row padding for A_p (64 bytes)


def _new_ap(m: int, n: int, device) -> torch.Tensor:
    """An m x n f64 output for the TRSM, row pitch padded off a power of two (the
    TRSM re-reads A_p panels of many CTAs at once; 2^k-byte row strides map them
    onto the same memory channels)."""
    pad = APITCH_PAD if (n * 8) % 4096 == 0 and m > 4096 else 0
    return torch.empty((m, n + pad), dtype=torch.float64, device=device)[:, :n]


def _trsm(a: DMat | torch.Tensor, r: torch.Tensor, out: torch.Tensor | None = None,
          engine: str | None = None) -> torch.Tensor:
    """A_p = A R^{-1} (R upper, device f64).  Large solves take the blocked path whose
    off-diagonal updates run on the INT8 tensor cores (sk_trsm_ozaki_f64)."""
    at = _rm(a.t if isinstance(a, DMat) else a)
    r = _rm(r)
    m, n = at.shape
    if out is None:
        out = _new_ap(m, n, at.device)
    st = _lib.SkStatus()
    if _trsm_engine(m, n, out.data_ptr() == at.data_ptr(), engine) == "ozaki":
        wp, wn = WORKSPACE.get(_lib.lib().sk_trsm_ozaki_workspace(m, n))
        call("sk_trsm_ozaki_f64", at.data_ptr(), at.stride(0), m, n, r.data_ptr(), r.stride(0),
             out.data_ptr(), out.stride(0), C.byref(st), wp, wn, stream_handle())
    else:
        call("sk_trsm_right_upper_f64", at.data_ptr(), at.stride(0), m, n, r.data_ptr(), r.stride(0),
             out.data_ptr(), out.stride(0), C.byref(st), stream_handle())
    return out


def _trsv(r: torch.Tensor, rhs: torch.Tensor, transposed: bool = False) -> torch.Tensor:
    r, rhs = _rm(r), rhs.contiguous()
    n = r.shape[0]
    out = torch.empty(n, dtype=torch.float64, device=r.device)
    wp, wn = WORKSPACE.get(2 * 8 * n + 1024)
    st = _lib.SkStatus()
    call("sk_trsv_f64", r.data_ptr(), r.stride(0), n, int(transposed), rhs.data_ptr(), out.data_ptr(),
         C.byref(st), wp, wn, stream_handle())
    return out


def _chol_solve(s: torch.Tensor, rhs: torch.Tensor) -> torch.Tensor:
    s, rhs = s.contiguous(), rhs.contiguous()
    n = s.shape[0]
    out = torch.empty(n, dtype=torch.float64, device=s.device)
    wp, wn = WORKSPACE.get(_lib.lib().sk_nxn_workspace(n))
    st = _lib.SkStatus()
    call("sk_chol_solve_f64", s.data_ptr(), n, rhs.data_ptr(), out.data_ptr(), C.byref(st), wp, wn,
         stream_handle())
    return out


def _lu_solve(g: torch.Tensor, rhs: torch.Tensor) -> torch.Tensor:
    g, rhs = g.contiguous(), rhs.contiguous()
    n = g.shape[0]
    out = torch.empty(n, dtype=torch.float64, device=g.device)
    wp, wn = WORKSPACE.get(_lib.lib().sk_nxn_workspace(n))
    st = _lib.SkStatus()
    call("sk_lu_solve_f64", g.data_ptr(), n, rhs.data_ptr(), out.data_ptr(), C.byref(st), wp, wn,
         stream_handle())
    return out


def _qr_r(a_s_level: torch.Tensor, level_code: int, d: int, n: int) -> torch.Tensor:
    """R of a column-major d x n level-dtype buffer (overwritten)."""
    r = torch.empty((n, n), dtype=torch.float64, device=a_s_level.device)
    wp, wn = WORKSPACE.get(_lib.lib().sk_qr_workspace(level_code, d, n))
    st = _lib.SkStatus()
    call("sk_qr_r", level_code, a_s_level.data_ptr(), d, n, r.data_ptr(), r.stride(0), C.byref(st), wp, wn,
         stream_handle())
    return r


def _householder_r64(at: torch.Tensor) -> torch.Tensor:
    """householder_reduce(a)[2] for a device f64 row-major m x n (m >= n).

    Up to TALL_QR_MAX_ROWS rows this is the column Householder kernel (the
    reference's algorithm and sign convention).  Taller matrices use TSQR: the R
    factors of row blocks are stacked and reduced again (a tree of Householder
    QRs).  R is unique up to the signs of its rows; every caller (seminormal
    equations, the Q^T b column of the QR baseline, singular values) is invariant
    to those signs."""
    m, n = at.shape
    if m < n:
        raise DimensionMismatch(f"need rows >= cols, got {m} x {n}")
    if m <= TALL_QR_MAX_ROWS:
        colmajor = at.t().contiguous()          # n x m row-major == m x n column-major
        return _qr_r(colmajor, 64, m, n)
    rows = max(n, TALL_QR_MAX_ROWS // 2)
    rs = [_householder_r64(at[r0:min(m, r0 + rows)]) for r0 in range(0, m, rows)
          if min(m, r0 + rows) - r0 >= n]
    tail = m % rows
    if tail and tail < n:                       # a short last block joins the stack as rows
        rs.append(at[m - tail:].contiguous())
    return _householder_r64(torch.cat(rs, dim=0))


def _jacobi_sv(at: torch.Tensor, max_sweeps: int = 30, tol: float = 1e-14) -> np.ndarray:
    at = _rm(at)
    rows, n = at.shape
    sv = (C.c_double * n)()
    wp, wn = WORKSPACE.get(_lib.lib().sk_jacobi_workspace(rows, n))
    call("sk_jacobi_sv_f64", at.data_ptr(), rows, n, at.stride(0), int(max_sweeps), float(tol), sv, wp, wn,
         stream_handle())
    return np.array(sv[:], dtype=np.float64)


TALL_QR_MAX_ROWS = 262144     # the column Householder kernel's chunk-tree limit
GRAM_DIAGNOSTICS = True       # tall kappa diagnostics via the Gram (fast); False: via TSQR (robust)


def _chol_factor(s: torch.Tensor) -> torch.Tensor:
    """Upper R with R^T R = (S + S^T)/2 (NotPositiveDefinite on breakdown)."""
    s = s.contiguous()
    n = s.shape[0]
    r = torch.empty((n, n), dtype=torch.float64, device=s.device)
    wp, wn = WORKSPACE.get(_lib.lib().sk_nxn_workspace(n))
    st = _lib.SkStatus()
    call("sk_chol_factor_f64", s.data_ptr(), n, r.data_ptr(), C.byref(st), wp, wn, stream_handle())
    return r


def _diagnostics_dev(at: torch.Tensor) -> ConditionDiagnostics:
    """condition_diagnostics on a device matrix (src/dense.py:418-448).

    The reference reduces a tall matrix to its n x n Householder R before Jacobi.
    Beyond TALL_QR_MAX_ROWS rows (e.g. A_p at m = 4M) the R factor is taken from the
    Cholesky factor of the Gram A^T A (same singular values in exact arithmetic);
    that is accurate while kappa(A) << 1e8, which holds for the preconditioned A_p
    this is used on (kappa(A_p) = O(1))."""
    if at.shape[0] < at.shape[1]:
        at = at.t().contiguous()
    m, n = at.shape
    w = at
    if m > TALL_QR_MAX_ROWS and GRAM_DIAGNOSTICS:
        try:
            w = _chol_factor(_gram(at))
        except Exception:   # noqa: BLE001  (breakdown: kappa out of the Gram route's range)
            sv = np.full(n, np.nan)
            return ConditionDiagnostics(two_norm=math.nan, two_norm_condition=math.nan, singular_values=sv)
    elif m > n:
        try:
            w = _householder_r64(at)
        except RankDeficient:
            w = at
    sv = _jacobi_sv(w)
    cond = float(sv[0] / sv[-1]) if sv[-1] > 0 else float("inf")
    return ConditionDiagnostics(two_norm=float(sv[0]), two_norm_condition=cond, singular_values=sv)


# ----------------------------------------------------------------- public ---
def _square_dev(a, name):
    d = as_dmat(a, name)
    if d.shape[0] != d.shape[1]:
        raise ValueError(f"{name} must be square, got shape {d.shape}")
    return d


def triangular_solve(r, rhs, transposed=False):
    """Solve r x = rhs (or r^T x = rhs): src/dense.py:204-242."""
    rd = as_dmat(r, "r") if not isinstance(r, np.ndarray) or r.ndim == 2 else None
    if rd is None or rd.shape[0] != rd.shape[1]:
        raise ValueError(f"r must be square, got shape {np.shape(r)}")
    n = rd.shape[0]
    rhs_np = rhs.detach().cpu().numpy() if isinstance(rhs, torch.Tensor) else np.asarray(rhs)
    if rhs_np.shape[0] != n:
        raise DimensionMismatch(f"rhs length {rhs_np.shape[0]} != n = {n}")
    cols = [rhs_np] if rhs_np.ndim == 1 else [rhs_np[:, k] for k in range(rhs_np.shape[1])]
    outs = [to_host(_trsv(rd.t, as_dvec(c), transposed)) for c in cols]
    x = outs[0] if rhs_np.ndim == 1 else np.stack(outs, axis=1)
    return like_input(torch.from_numpy(x), "numpy" if not isinstance(rhs, torch.Tensor) else "torch")


def lu_solve(a, rhs):
    """LU with partial pivoting: src/dense.py:245-286."""
    ad = _square_dev(a, "a")
    n = ad.shape[0]
    rhs_np = np.asarray(rhs.detach().cpu() if isinstance(rhs, torch.Tensor) else rhs)
    if rhs_np.shape[0] != n:
        raise DimensionMismatch(f"rhs length {rhs_np.shape[0]} != n = {n}")
    cols = [rhs_np] if rhs_np.ndim == 1 else [rhs_np[:, k] for k in range(rhs_np.shape[1])]
    outs = [to_host(_lu_solve(ad.t, as_dvec(c))) for c in cols]
    return outs[0] if rhs_np.ndim == 1 else np.stack(outs, axis=1)


def cholesky_solve(s, rhs):
    """SPD solve with the 10-eps symmetry gate: src/dense.py:314-342."""
    sd = _square_dev(s, "s")
    n = sd.shape[0]
    rhs_np = np.asarray(rhs.detach().cpu() if isinstance(rhs, torch.Tensor) else rhs)
    if rhs_np.shape[0] != n:
        raise DimensionMismatch(f"rhs length {rhs_np.shape[0]} != n = {n}")
    cols = [rhs_np] if rhs_np.ndim == 1 else [rhs_np[:, k] for k in range(rhs_np.shape[1])]
    outs = [to_host(_chol_solve(sd.t, as_dvec(c))) for c in cols]
    return outs[0] if rhs_np.ndim == 1 else np.stack(outs, axis=1)


def _qr_factors_dev(at: torch.Tensor, level_code: int, want_q: bool):
    """(R, Q or None) of a device f64 row-major d x n matrix at the given level:
    sk_qr_in_precision_f64 (demotion and binary16 prescale on the f64 values, Q
    accumulated from the reflectors in the level arithmetic)."""
    at = _rm(at)
    d, n = at.shape
    r = torch.empty((n, n), dtype=torch.float64, device=at.device)
    q = torch.empty((d, n), dtype=torch.float64, device=at.device) if want_q else None
    wp, wn = WORKSPACE.get(_lib.lib().sk_qr_factors_workspace(level_code, d, n))
    st = _lib.SkStatus()
    call("sk_qr_in_precision_f64", level_code, at.data_ptr(), at.stride(0), d, n, r.data_ptr(), n,
         q.data_ptr() if q is not None else None, n, C.byref(st), wp, wn, stream_handle())
    return r, q


def householder_reduce(a, ops=None):
    """householder_reduce (src/dense.py:108-161) in binary64 on the device:
    (reflectors, taus, R) with reflector j of length m - j (unnormalised, first
    entry x_0 - alpha) and tau_j = 2 / v_j.v_j, the reference's sign convention.
    `ops` is accepted for signature parity; only the native arithmetic exists
    (binary16 emulation is reached through qr_in_precision).  Above
    TALL_QR_MAX_ROWS rows R comes from TSQR and the reflectors are not formed
    (returns (None, None, R))."""
    if ops is not None and getattr(ops, "name", "native") != "native":
        raise ValueError("householder_reduce: only the native arithmetic is available; use qr_in_precision")
    ad = as_dmat(a)
    m, n = ad.shape
    if m < n:
        raise DimensionMismatch(f"need rows >= cols, got {m} x {n}")
    if m > TALL_QR_MAX_ROWS:
        return None, None, to_host(_householder_r64(ad.t))
    r = torch.empty((n, n), dtype=torch.float64, device=ad.t.device)
    v = torch.empty((m, n), dtype=torch.float64, device=ad.t.device)
    taus = torch.empty(n, dtype=torch.float64, device=ad.t.device)
    wp, wn = WORKSPACE.get(_lib.lib().sk_qr_factors_workspace(64, m, n))
    st = _lib.SkStatus()
    call("sk_householder_f64", ad.ptr, ad.ld, m, n, r.data_ptr(), n, v.data_ptr(), n, taus.data_ptr(),
         C.byref(st), wp, wn, stream_handle())
    vh, th = to_host(v), to_host(taus)
    reflectors = [vh[j:, j].copy() for j in range(n)]
    return reflectors, [np.float64(t) for t in th], to_host(r)


_LEVEL_OF_DTYPE = {np.dtype(np.float16): (16, torch.float16), np.dtype(np.float32): (32, torch.float32),
                   np.dtype(np.float64): (64, torch.float64)}


def accumulate_thin_q(reflectors, taus, m, n, ops=None, dtype=np.float64):
    """accumulate_thin_q (src/dense.py:164-172): the thin Q formed by applying the
    reflectors backward to eye(m, n) in `dtype` arithmetic (float16: every scalar op
    rounded to binary16 and pairwise-tree sums, the reference's HALF_OPS; float32 /
    float64: native), on the device (sk_accumulate_q).  `ops` is accepted for
    signature parity: the arithmetic follows `dtype`."""
    dt = np.dtype(dtype)
    if dt not in _LEVEL_OF_DTYPE:
        raise ValueError(f"unsupported dtype {dt}")
    if len(reflectors) != n or len(taus) != n:
        raise DimensionMismatch(f"need {n} reflectors and taus, got {len(reflectors)} / {len(taus)}")
    code, tdt = _LEVEL_OF_DTYPE[dt]
    vpack = np.zeros((n, m), dtype=dt)          # row j = column j of the column-major m x n pack
    for j, vj in enumerate(reflectors):
        vj = np.asarray(vj)
        if vj.shape != (m - j,):
            raise DimensionMismatch(f"reflector {j} has shape {vj.shape}, expected {(m - j,)}")
        vpack[j, j:] = vj.astype(dt)
    dev = device()
    vd = torch.from_numpy(vpack).to(dev)
    td = torch.from_numpy(np.asarray(taus, dtype=dt)).to(dev)
    qd = torch.empty((n, m), dtype=tdt, device=dev)
    call("sk_accumulate_q", code, vd.data_ptr(), m, td.data_ptr(), m, n, qd.data_ptr(), m, stream_handle())
    return np.asfortranarray(to_host(qd).T)


def householder_qr(a):
    """Thin QR (src/dense.py:175-201): R and Q = H_0 ... H_{n-1} eye(m, n) from the
    device Householder factorisation (binary64, the reference's sign convention).
    Above TALL_QR_MAX_ROWS rows R comes from TSQR and Q is formed as A R^-1."""
    ad = as_dmat(a)
    m, n = ad.shape
    if m < n:
        raise DimensionMismatch(f"need rows >= cols, got {m} x {n}")
    if m > TALL_QR_MAX_ROWS:
        r = _householder_r64(ad.t)
        return QRFactors(q=to_host(_trsm(ad, r)), r=to_host(r))
    r, q = _qr_factors_dev(ad.t, 64, True)
    return QRFactors(q=to_host(q), r=to_host(r))


def jacobi_singular_values(a, max_sweeps=30, tol=1e-14):
    """One-sided Jacobi singular values: src/dense.py:365-415."""
    ad = as_dmat(a)
    return _jacobi_sv(ad.t, max_sweeps, tol)


def condition_diagnostics(a):
    """src/dense.py:418-448."""
    return _diagnostics_dev(as_dmat(a).t)


def hager_one_norm_inverse_estimate(solve, n):
    """Hager's estimator around a caller-supplied solve (src/dense.py:451-480).
    The callable is the caller's; the pipeline's own estimate runs entirely on
    the device inside sk_kappa0_from_gram."""
    if n < 1:
        raise ValueError(f"n must be >= 1, got {n}")
    x = np.full(n, 1.0 / n)
    best = 0.0
    for _ in range(5):
        y = np.asarray(solve(x, False), dtype=np.float64)
        best = max(best, float(np.abs(y).sum()))
        z = np.asarray(solve(np.where(y >= 0, 1.0, -1.0), True), dtype=np.float64)
        j = int(np.argmax(np.abs(z)))
        if abs(z[j]) <= float(z @ x):
            break
        x = np.zeros(n)
        x[j] = 1.0
    return best
