"""Operation-for-operation numpy restatement of the reference hot path.

TEST INFRASTRUCTURE (see oracle/__init__.py): the checker and the CPU
baseline, never the product.

Reference: `sketchlsq` 0.1.0, `/root/reference/pkg/src/sketchlsq/` (abbreviated
`src/` below).  Every routine names the reference lines it follows.  The goal
is bit-identical output to the reference in the same numpy/scipy/OpenBLAS
environment, so the numpy primitives (which BLAS call, which memory order,
which dtype each scalar lives in) are chosen to be the ones the reference
issues.  The code layout is our own: one module, plain functions, a small
arithmetic table for the binary16 emulation.
"""

from __future__ import annotations

import hashlib
import math
import time
from dataclasses import dataclass, field

import numpy as np
from scipy.fft import dct as _scipy_dct


# --------------------------------------------------------------------------
# Failure classes.  Same names as src/errors.py:10-55 so outcome classes can be
# compared by name against the product package.
# --------------------------------------------------------------------------
class OracleNumericalError(Exception):
    """Base of the oracle's numerical failures (mirrors SketchLsqError)."""


def _mk(name):
    return type(name, (OracleNumericalError,), {})


RankDeficient = _mk("RankDeficient")
SingularTriangular = _mk("SingularTriangular")
NumericallySingular = _mk("NumericallySingular")
NotPositiveDefinite = _mk("NotPositiveDefinite")
NoConvergence = _mk("NoConvergence")
DimensionMismatch = _mk("DimensionMismatch")
Overflow = _mk("Overflow")


# --------------------------------------------------------------------------
# Precision levels (src/precision.py:32-65)
# --------------------------------------------------------------------------
LEVEL_DTYPE = {"binary16": np.float16, "binary32": np.float32, "binary64": np.float64}
LEVEL_ALIASES = {"half": "binary16", "single": "binary32", "double": "binary64",
                 "binary16": "binary16", "binary32": "binary32", "binary64": "binary64"}
WIDER = {"binary16": "binary32", "binary32": "binary64"}
UNIT_ROUNDOFF = {"binary16": 2.0 ** -11, "binary32": 2.0 ** -24, "binary64": 2.0 ** -53}


def canonical_level(name: str) -> str:
    """src/precision.py:55-60 — alias lookup, ValueError on unknown names."""
    if name not in LEVEL_ALIASES:
        raise ValueError(f"unknown precision name {name!r}")
    return LEVEL_ALIASES[name]


def choose_level(kappa0: float, overflowed: bool) -> str:
    """src/precision.py:254-266 — thresholds <4 half, <=8 single, else double."""
    if overflowed or not math.isfinite(kappa0):
        return "binary64"
    if kappa0 < 4:
        return "binary16"
    return "binary32" if kappa0 <= 8 else "binary64"


# --------------------------------------------------------------------------
# Random streams (src/rng.py:23-46)
# --------------------------------------------------------------------------
_M64 = (1 << 64) - 1


def philox(seed: int, lane: int = 0) -> np.random.Generator:
    """src/rng.py:23-34: Philox keyed by (seed mod 2^64) | (lane << 64)."""
    return np.random.Generator(np.random.Philox(
        key=(int(seed) & _M64) | ((int(lane) & _M64) << 64)))


def mix64(*parts) -> int:
    """src/rng.py:37-46: blake2b-8 over 16-byte little-endian signed words."""
    digest = hashlib.blake2b(digest_size=8)
    for part in parts:
        digest.update(int(part).to_bytes(16, "little", signed=True))
    return int.from_bytes(digest.digest(), "little")


LANE_SIGNS, LANE_ROWS, LANE_GAUSS = 1, 2, 3   # src/rng.py:18-20


# --------------------------------------------------------------------------
# Input validation (src/dense.py:57-65, src/solvers.py:87-96)
# --------------------------------------------------------------------------
def as_float_matrix(a, name="a"):
    arr = np.asarray(a)
    if arr.ndim != 2:
        raise ValueError(f"{name} must be 2-D, got ndim={arr.ndim}")
    if arr.dtype not in (np.float16, np.float32, np.float64):
        arr = arr.astype(np.float64)
    if not np.isfinite(arr).all():
        raise ValueError(f"{name} contains non-finite entries")
    return arr


def checked_system(a, b):
    a = as_float_matrix(a)
    b = np.asarray(b, dtype=np.float64)
    if b.ndim != 1:
        raise ValueError(f"b must be 1-D, got ndim={b.ndim}")
    rows, cols = a.shape
    if rows < cols:
        raise DimensionMismatch(f"need rows >= cols, got {a.shape}")
    if b.shape[0] != rows:
        raise DimensionMismatch(f"b length {b.shape[0]} != rows {rows}")
    return a.astype(np.float64), b


# --------------------------------------------------------------------------
# Demotion (src/precision.py:90-103)
# --------------------------------------------------------------------------
def demote(a, level: str):
    """Returns (rounded array, overflowed flag)."""
    src = np.asarray(a)
    with np.errstate(over="ignore"):
        out = src.astype(LEVEL_DTYPE[level])
    return out, bool((np.isinf(out) & np.isfinite(src)).any())


# --------------------------------------------------------------------------
# Arithmetic tables for the Householder kernels.
# NATIVE follows src/dense.py:68-105 (BLAS in the array dtype); HALF follows
# src/precision.py:106-150 (every scalar op rounded to float16, pairwise trees).
# --------------------------------------------------------------------------
def tree_sum(x):
    """src/precision.py:106-115: level-by-level adjacent pairing along axis 0,
    an odd trailing element carried to the end of the next level."""
    while x.shape[0] > 1:
        pairs = x.shape[0] // 2
        nxt = x[0:2 * pairs:2] + x[1:2 * pairs:2]
        if x.shape[0] & 1:
            nxt = np.concatenate([nxt, x[2 * pairs:]], axis=0)
        x = nxt
    return x[0]


class _Native:
    dot = staticmethod(lambda u, v: u @ v)
    vec_mat = staticmethod(lambda v, m: v @ m)
    scale = staticmethod(lambda t, v: t * v)
    sqrt = staticmethod(np.sqrt)
    div = staticmethod(lambda p, q: p / q)
    sub = staticmethod(lambda p, q: p - q)

    @staticmethod
    def rank1_sub(m, v, w):
        m -= np.outer(v, w)


class _Half(_Native):
    dot = staticmethod(lambda u, v: tree_sum(u * v))
    vec_mat = staticmethod(lambda v, m: tree_sum(v[:, None] * m))

    @staticmethod
    def rank1_sub(m, v, w):
        m -= v[:, None] * w[None, :]


NATIVE, HALF = _Native(), _Half()


# --------------------------------------------------------------------------
# Householder QR (src/dense.py:108-201)
# --------------------------------------------------------------------------
def householder_steps(a, ar=NATIVE):
    """src/dense.py:108-161.  Returns (reflectors, taus, R)."""
    rows, cols = a.shape
    w = np.array(a, order="F", copy=True)
    two = w.dtype.type(2)
    vs, taus = [], []
    for j in range(cols):
        x = w[j:, j].copy()
        nrm = ar.sqrt(ar.dot(x, x))
        if nrm == 0:
            raise RankDeficient(f"pivot column {j} is zero at working precision")
        alpha = -nrm if x[0] >= 0 else nrm
        x[0] = ar.sub(x[0], alpha)          # x now holds the reflector v
        vtv = ar.dot(x, x)
        if vtv == 0:
            raise RankDeficient(f"reflector {j} vanished at working precision")
        tau = ar.div(two, vtv)
        if not np.isfinite(tau):
            raise RankDeficient(f"reflector {j} norm underflowed at working precision")
        if j + 1 < cols:
            trail = w[j:, j + 1:]
            ar.rank1_sub(trail, x, ar.scale(tau, ar.vec_mat(x, trail)))
        w[j, j] = alpha
        w[j + 1:, j] = 0
        vs.append(x)
        taus.append(tau)
    return vs, taus, np.array(w[:cols, :], copy=True)


def thin_q(vs, taus, rows, cols, ar=NATIVE, dtype=np.float64):
    """src/dense.py:164-172: backward accumulation onto eye(rows, cols)."""
    q = np.zeros((rows, cols), dtype=dtype, order="F")
    q[np.arange(cols), np.arange(cols)] = 1
    for j in range(cols - 1, -1, -1):
        blk = q[j:, :]
        ar.rank1_sub(blk, vs[j], ar.scale(taus[j], ar.vec_mat(vs[j], blk)))
    return q


def householder_qr(a):
    """src/dense.py:175-201 -> (Q, R) in the dtype of a."""
    a = as_float_matrix(a)
    rows, cols = a.shape
    if rows < cols:
        raise DimensionMismatch(f"need rows >= cols, got {rows} x {cols}")
    vs, taus, r = householder_steps(a)
    return thin_q(vs, taus, rows, cols, dtype=a.dtype), r


def qr_at_level(a, level: str):
    """src/precision.py:153-202 -> (Q, R) promoted to float64."""
    a = as_float_matrix(a)
    rows, cols = a.shape
    if rows < cols:
        raise DimensionMismatch(f"need rows >= cols, got {rows} x {cols}")
    if level == "binary64":
        return householder_qr(a.astype(np.float64))
    if level == "binary32":
        data, over = demote(a, "binary32")
        if over:
            raise Overflow("input exceeds the binary32 range")
        vs, taus, r = householder_steps(data)
        q = thin_q(vs, taus, rows, cols, dtype=np.float32)
        return q.astype(np.float64), r.astype(np.float64)
    # binary16: power-of-two prescale so max|a| lands in [0.5, 1)
    work = a.astype(np.float64)
    peak = float(np.abs(work).max())
    if peak == 0:
        raise RankDeficient("zero matrix")
    scale = 2.0 ** -math.frexp(peak)[1]
    data, _ = demote(work * scale, "binary16")
    with np.errstate(over="ignore", invalid="ignore", under="ignore"):
        vs, taus, r16 = householder_steps(data, HALF)
        q16 = thin_q(vs, taus, rows, cols, ar=HALF, dtype=np.float16)
    if not (np.isfinite(q16).all() and np.isfinite(r16).all()):
        raise Overflow("binary16 computation produced non-finite values")
    return q16.astype(np.float64), r16.astype(np.float64) / scale


# --------------------------------------------------------------------------
# Substitution, LU, Cholesky (src/dense.py:204-342)
# --------------------------------------------------------------------------
def tri_solve(r, rhs, transposed=False):
    """src/dense.py:204-242: R x = rhs (backward) or R^T x = rhs (forward)."""
    r = np.asarray(r)
    if r.ndim != 2 or r.shape[0] != r.shape[1]:
        raise ValueError(f"r must be square, got shape {r.shape}")
    n = r.shape[0]
    rhs = np.asarray(rhs)
    if rhs.shape[0] != n:
        raise DimensionMismatch(f"rhs length {rhs.shape[0]} != n = {n}")
    zeros = np.nonzero(np.diagonal(r) == 0)[0]
    if zeros.size:
        raise SingularTriangular(f"zero diagonal entry at index {zeros[0]}")
    x = np.array(rhs, dtype=np.result_type(r, rhs), copy=True)
    xs = x if x.ndim == 2 else x[:, None]
    order = range(n) if transposed else range(n - 1, -1, -1)
    for i in order:
        if transposed and i:
            xs[i] -= r[:i, i] @ xs[:i]
        elif not transposed and i + 1 < n:
            xs[i] -= r[i, i + 1:] @ xs[i + 1:]
        xs[i] /= r[i, i]
    return x


def lu_pivoted_solve(a, rhs):
    """src/dense.py:245-286: partial pivoting, lowest index on ties,
    NumericallySingular below n*eps*max|a|."""
    a = as_float_matrix(a)
    if a.shape[0] != a.shape[1]:
        raise ValueError(f"a must be square, got shape {a.shape}")
    n = a.shape[0]
    rhs = np.asarray(rhs)
    if rhs.shape[0] != n:
        raise DimensionMismatch(f"rhs length {rhs.shape[0]} != n = {n}")
    f = np.array(a, order="F", copy=True)
    perm = np.arange(n)
    floor = n * np.finfo(f.dtype).eps * np.abs(f).max()
    for k in range(n):
        p = k + int(np.argmax(np.abs(f[k:, k])))
        mag = abs(f[p, k])
        if mag < floor or mag == 0:
            raise NumericallySingular(
                f"pivot {k} magnitude {mag:.3e} below threshold {floor:.3e}")
        if p != k:
            f[[k, p], :] = f[[p, k], :]
            perm[[k, p]] = perm[[p, k]]
        f[k + 1:, k] /= f[k, k]
        f[k + 1:, k + 1:] -= np.outer(f[k + 1:, k], f[k, k + 1:])
    x = np.array(rhs[perm], dtype=np.result_type(f, rhs), copy=True)
    xs = x if x.ndim == 2 else x[:, None]
    for i in range(1, n):
        xs[i] -= f[i, :i] @ xs[:i]
    for i in range(n - 1, -1, -1):
        if i + 1 < n:
            xs[i] -= f[i, i + 1:] @ xs[i + 1:]
        xs[i] /= f[i, i]
    return x


def cholesky_lower(s):
    """src/dense.py:289-311: left-looking, on (s + s^T)/2."""
    s = np.asarray(s)
    n = s.shape[0]
    sym = (s + s.T) / s.dtype.type(2)
    ell = np.zeros((n, n), dtype=sym.dtype, order="F")
    for j in range(n):
        col = sym[j:, j] - ell[j:, :j] @ ell[j, :j]
        if not (col[0] > 0) or not np.isfinite(col[0]):
            raise NotPositiveDefinite(f"pivot {j} is {col[0]}")
        piv = np.sqrt(col[0])
        ell[j, j] = piv
        ell[j + 1:, j] = col[1:] / piv
    return ell


def spd_solve(s, rhs):
    """src/dense.py:314-342: symmetry gate 10*eps*max|s|, Cholesky, two solves."""
    s = as_float_matrix(s, "s")
    if s.shape[0] != s.shape[1]:
        raise ValueError(f"s must be square, got shape {s.shape}")
    if np.abs(s - s.T).max() > 10 * np.finfo(s.dtype).eps * np.abs(s).max():
        raise ValueError("s is not symmetric within 10*eps relative tolerance")
    rhs = np.asarray(rhs)
    if rhs.shape[0] != s.shape[0]:
        raise DimensionMismatch(f"rhs length {rhs.shape[0]} != n = {s.shape[0]}")
    up = np.asfortranarray(cholesky_lower(s).T)
    return tri_solve(up, tri_solve(up, rhs, transposed=True), transposed=False)


# --------------------------------------------------------------------------
# One-sided Jacobi and diagnostics (src/dense.py:345-448)
# --------------------------------------------------------------------------
_ROUNDS = {}


def circle_rounds(n):
    """src/dense.py:345-362: circle-method round-robin pairing."""
    if n in _ROUNDS:
        return _ROUNDS[n]
    seats = list(range(n)) + ([-1] if n % 2 else [])
    k = len(seats)
    out = []
    for _ in range(max(k - 1, 0)):
        pr = [(min(seats[i], seats[k - 1 - i]), max(seats[i], seats[k - 1 - i]))
              for i in range(k // 2)]
        pr = [(p, q) for p, q in pr if p != -1 and q != -1]
        if pr:
            out.append((np.array([p for p, _ in pr]), np.array([q for _, q in pr])))
        seats = [seats[0], seats[-1]] + seats[1:-1]
    _ROUNDS[n] = tuple(out)
    return _ROUNDS[n]


def jacobi_sv(a, max_sweeps=30, tol=1e-14):
    """src/dense.py:365-415: descending singular values or NoConvergence."""
    w = np.array(a, dtype=np.float64, order="F", copy=True)
    n = w.shape[1]
    gate = math.sqrt(w.shape[0]) * 2.0 ** -52
    done = n < 2
    for _ in range(max_sweeps):
        if done:
            break
        worst = 0.0
        for ps, qs in circle_rounds(n):
            cp, cq = w[:, ps], w[:, qs]
            pp = np.einsum("ij,ij->j", cp, cp)
            qq = np.einsum("ij,ij->j", cq, cq)
            pq = np.einsum("ij,ij->j", cp, cq)
            live = np.abs(pq) > gate * np.sqrt(pp) * np.sqrt(qq)
            with np.errstate(divide="ignore", invalid="ignore"):
                zeta = np.where(live, (qq - pp) / (2 * pq), 0.0)
            sg = np.where(zeta >= 0, 1.0, -1.0)
            t = np.where(live, sg / (np.abs(zeta) + np.hypot(1.0, zeta)), 0.0)
            c = 1.0 / np.sqrt(1.0 + t * t)
            s = t * c
            w[:, ps] = c * cp - s * cq
            w[:, qs] = s * cp + c * cq
            if t.size:
                worst = max(worst, float(np.abs(t).max()))
        done = worst < tol
    if not done:
        raise NoConvergence(f"Jacobi did not converge in {max_sweeps} sweeps")
    return np.sort(np.sqrt(np.einsum("ij,ij->j", w, w)))[::-1]


def condition_number(a):
    """src/dense.py:418-448 -> (two_norm, condition, singular values)."""
    a = as_float_matrix(a)
    if a.shape[0] < a.shape[1]:
        a = a.T
    rows, cols = a.shape
    w = a
    if rows > cols:
        try:
            w = householder_steps(a.astype(np.float64))[2]
        except RankDeficient:
            w = a
    sv = jacobi_sv(w)
    with np.errstate(divide="ignore", invalid="ignore"):
        cond = float(sv[0] / sv[-1]) if sv[-1] > 0 else float("inf")
    return float(sv[0]), cond, sv


# --------------------------------------------------------------------------
# Hager 1-norm inverse estimate (src/dense.py:451-480)
# --------------------------------------------------------------------------
def hager(solve, n):
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


# --------------------------------------------------------------------------
# kappa0 estimate and the level decision (src/precision.py:205-276)
# --------------------------------------------------------------------------
def kappa0_estimate(a):
    """-> (kappa0, overflowed).  Everything binary64 on the full A."""
    a = as_float_matrix(a)
    w = a.astype(np.float64)
    with np.errstate(over="ignore", invalid="ignore", under="ignore"):
        g = w.T @ w
    return kappa0_from_gram(g)


def kappa0_from_gram(g):
    """src/precision.py:231-251: the estimate given G = A^T A (row shards sum
    their partial Grams first)."""
    n = g.shape[0]
    with np.errstate(over="ignore", invalid="ignore", under="ignore"):
        if not np.isfinite(g).all():
            return math.nan, True
        n1 = float(np.abs(g).sum(axis=0).max())
        if n1 == 0 or not math.isfinite(n1):
            return math.nan, True
        try:
            up = np.asfortranarray(cholesky_lower(g).T)
        except NotPositiveDefinite:
            return math.nan, True
        est = hager(lambda rhs, tr: tri_solve(up, tri_solve(up, rhs, transposed=True)), n)
    value = n * n1 * est
    if not math.isfinite(value) or value <= 0:
        return math.nan, True
    return 0.5 * math.log10(value), False


def decide(a):
    """src/precision.py:269-276 -> (kappa0, level, overflowed)."""
    k0, over = kappa0_estimate(a)
    return k0, choose_level(k0, over), over


# --------------------------------------------------------------------------
# SRTT sketch (src/sketch.py:85-169)
# --------------------------------------------------------------------------
def padded_height(m, transform):
    if transform != "wht":
        return m
    return 1 << max(m - 1, 0).bit_length() if m > 1 else 1


@dataclass
class Sketch:
    m: int
    d: int
    transform: str
    seed: int
    signs: np.ndarray
    rows: np.ndarray

    @property
    def m_pad(self):
        return self.signs.shape[0]


def draw_sketch(m, d, transform="dct2", seed=0):
    """src/sketch.py:89-112."""
    if transform not in ("dct2", "wht"):
        raise ValueError(f"unknown transform {transform!r}")
    if m < 1 or d < 1:
        raise ValueError(f"need m >= 1 and d >= 1, got m={m}, d={d}")
    mp = padded_height(m, transform)
    if d > mp:
        raise ValueError(f"sample count d={d} exceeds padded height {mp}")
    signs = philox(seed, LANE_SIGNS).integers(0, 2, mp) * 2.0 - 1.0
    rows = philox(seed, LANE_ROWS).integers(0, mp, d)
    return Sketch(int(m), int(d), transform, int(seed), signs, rows)


def _butterflies(x):
    """src/sketch.py:121-135: radix-2 WHT in the dtype of x, then 1/sqrt(n)."""
    n = x.shape[0]
    h = 1
    while h < n:
        blk = x.reshape(-1, 2, h, *x.shape[1:])
        lo, hi = blk[:, 0].copy(), blk[:, 1].copy()
        blk[:, 0] = lo + hi
        blk[:, 1] = lo - hi
        h *= 2
    x *= x.dtype.type(1.0 / math.sqrt(n))
    return x


def sketch_apply(op: Sketch, a):
    """src/sketch.py:138-169: signs, transform, sample, scale in a's dtype."""
    a = as_float_matrix(a)
    if a.shape[0] != op.m:
        raise DimensionMismatch(f"operator built for {op.m} rows, got {a.shape[0]}")
    dt = a.dtype
    with np.errstate(over="ignore", invalid="ignore", under="ignore"):
        if op.m_pad == op.m:
            work = a * op.signs[:, None].astype(dt)
        else:
            work = np.zeros((op.m_pad, a.shape[1]), dtype=dt)
            work[:op.m] = a * op.signs[:op.m, None].astype(dt)
        if op.transform == "wht":
            work = _butterflies(work)
        elif dt == np.float16:
            work = _scipy_dct(work.astype(np.float32), type=2, axis=0,
                              norm="ortho").astype(np.float16)
        else:
            work = _scipy_dct(work, type=2, axis=0, norm="ortho")
        return work[op.rows] * dt.type(math.sqrt(op.m_pad / op.d))


def sketch_matrix(op: Sketch):
    """Dense d x m_pad operator in float64 (closed form of TL;DR #2 of SURVEY):
    row i is sqrt(m_pad/d) * F[rows[i], :] * signs."""
    mp = op.m_pad
    k = op.rows.astype(np.float64)[:, None]
    if op.transform == "wht":
        bits = np.bitwise_and(op.rows[:, None], np.arange(mp)[None, :])
        par = np.array([bin(int(v)).count("1") & 1 for v in bits.ravel()]).reshape(bits.shape)
        f = np.where(par == 1, -1.0, 1.0) / math.sqrt(mp)
    else:
        j = np.arange(mp, dtype=np.float64)[None, :]
        f = np.sqrt(2.0 / mp) * np.cos(np.pi * k * (2 * j + 1) / (2 * mp))
        f[op.rows == 0, :] = math.sqrt(1.0 / mp)
    return math.sqrt(mp / op.d) * f * op.signs[None, :]


# --------------------------------------------------------------------------
# Solvers (src/solvers.py)
# --------------------------------------------------------------------------
@dataclass
class Pre:
    r_s: np.ndarray
    level: str
    kappa_rs: float
    kappa_ap: float | None = None
    sketch: dict | None = None


@dataclass
class Report:
    method: str
    x_hat: np.ndarray
    residual_norm: float
    relative_residual: float
    relative_error: float | None
    wall_ms: float
    pre: Pre | None = None
    decision: tuple | None = None
    escalated_from: str | None = None
    timings: dict = field(default_factory=dict)


def report(method, a, b, x, t0, x_star=None, pre=None):
    """src/solvers.py:99-117 (relative_error uses ||x*||, as the code does)."""
    res = float(np.linalg.norm(a @ x - b))
    den = float(np.linalg.norm(a)) * float(np.linalg.norm(x))
    rel_err = None
    if x_star is not None:
        xs = np.asarray(x_star, dtype=np.float64)
        rel_err = float(np.linalg.norm(x - xs) / np.linalg.norm(xs))
    return Report(method, x, res, res / den if den > 0 else math.inf, rel_err,
                  (time.perf_counter() - t0) * 1e3, pre)


def solve_qr(a, b, x_star=None):                       # src/solvers.py:120-126
    a, b = checked_system(a, b)
    t0 = time.perf_counter()
    q, r = householder_qr(a)
    return report("qr", a, b, tri_solve(r, q.T @ b), t0, x_star)


def solve_ne(a, b, x_star=None):                       # src/solvers.py:129-138
    a, b = checked_system(a, b)
    t0 = time.perf_counter()
    return report("ne", a, b, spd_solve(a.T @ a, a.T @ b), t0, x_star)


def solve_sne(a, b, x_star=None):                      # src/solvers.py:141-148
    a, b = checked_system(a, b)
    t0 = time.perf_counter()
    r = householder_steps(a)[2]
    x = tri_solve(r, tri_solve(r, a.T @ b, transposed=True))
    return report("sne", a, b, x, t0, x_star)


def solve_nne(a, bmat, b, x_star=None):                # src/solvers.py:151-165
    a, b = checked_system(a, b)
    bmat = as_float_matrix(bmat, "b_matrix").astype(np.float64)
    if bmat.shape != a.shape:
        raise DimensionMismatch(f"b_matrix shape {bmat.shape} != a shape {a.shape}")
    t0 = time.perf_counter()
    return report("nne", a, b, lu_pivoted_solve(bmat.T @ a, bmat.T @ b), t0, x_star)


def build_pre(a, d_factor=3.0, transform="dct2", level="binary64", seed=0,
              diagnostics=True, timings=None):
    """src/solvers.py:168-202."""
    tm = timings if timings is not None else {}
    a = as_float_matrix(a)
    m, n = a.shape
    if m < n:
        raise DimensionMismatch(f"need rows >= cols, got {m} x {n}")
    d = int(math.ceil(d_factor * n))
    if d < n:
        raise ValueError(f"d_factor {d_factor} gives d={d} < n={n}")
    t = time.perf_counter()
    data, over = demote(a, level)
    if over:
        raise Overflow(f"input exceeds the {level} range")
    op = draw_sketch(m, d, transform, seed)
    a_s = sketch_apply(op, data)
    tm["sketch"] = tm.get("sketch", 0.0) + time.perf_counter() - t
    t = time.perf_counter()
    r_s = qr_at_level(a_s, level)[1]
    tm["level_qr"] = tm.get("level_qr", 0.0) + time.perf_counter() - t
    if (np.diagonal(r_s) == 0).any():
        raise RankDeficient("sketched factor has a zero diagonal entry")
    t = time.perf_counter()
    kappa_rs = condition_number(r_s)[1] if diagnostics else math.nan
    tm["diag_rs"] = tm.get("diag_rs", 0.0) + time.perf_counter() - t
    return Pre(r_s, level, kappa_rs, None,
               {"m": op.m, "d": op.d, "transform": op.transform, "seed": op.seed})


def precondition(a, pre, diagnostics=True, timings=None):
    """src/solvers.py:205-215: A_p = A R_s^{-1} by substitution on A^T."""
    tm = timings if timings is not None else {}
    a = as_float_matrix(a).astype(np.float64)
    t = time.perf_counter()
    a_p = np.ascontiguousarray(tri_solve(pre.r_s, a.T, transposed=True).T)
    tm["trsm"] = tm.get("trsm", 0.0) + time.perf_counter() - t
    t = time.perf_counter()
    pre.kappa_ap = condition_number(a_p)[1] if diagnostics else math.nan
    tm["diag_ap"] = tm.get("diag_ap", 0.0) + time.perf_counter() - t
    return a_p


def solve_pne(a, b, pre, x_star=None, a_p=None):      # src/solvers.py:218-237
    a, b = checked_system(a, b)
    t0 = time.perf_counter()
    if a_p is None:
        a_p = precondition(a, pre)
    g, rhs = a_p.T @ a_p, a_p.T @ b
    try:
        y = spd_solve(g, rhs)
    except NotPositiveDefinite:
        y = lu_pivoted_solve(g, rhs)
    return report("pne", a, b, tri_solve(pre.r_s, y), t0, x_star, pre)


def solve_hpne(a, b, pre, x_star=None, a_p=None):     # src/solvers.py:240-252
    a, b = checked_system(a, b)
    t0 = time.perf_counter()
    if a_p is None:
        a_p = precondition(a, pre)
    return report("hpne", a, b, lu_pivoted_solve(a_p.T @ a, a_p.T @ b), t0, x_star, pre)


def prepare(a, d_factor=3.0, transform="dct2", level="binary64", seed=0,
            diagnostics=True, timings=None):
    """src/solvers.py:255-279: exactly one escalation on RankDeficient."""
    failed = None
    while True:
        try:
            pre = build_pre(a, d_factor, transform, level, seed, diagnostics, timings)
            return pre, precondition(a, pre, diagnostics, timings), failed
        except RankDeficient:
            wider = WIDER.get(level)
            if failed is not None or wider is None:
                raise
            failed, level = level, wider


def pipeline(a, b, method="pne", precision="auto", d_factor=3.0, transform="dct2",
             seed=0, x_star=None, diagnostics=True, timings=None):
    """src/solvers.py:282-324 (Algorithm 1)."""
    tm = timings if timings is not None else {}
    a, b = checked_system(a, b)
    if method not in ("pne", "hpne"):
        raise ValueError(f"pipeline method must be pne or hpne, got {method!r}")
    t0 = time.perf_counter()
    decision = None
    if precision == "auto":
        t = time.perf_counter()
        decision = decide(a)
        tm["kappa0"] = time.perf_counter() - t
        level = decision[1]
    else:
        level = canonical_level(precision)
    pre, a_p, failed = prepare(a, d_factor, transform, level, seed, diagnostics, tm)
    t = time.perf_counter()
    rep = (solve_pne if method == "pne" else solve_hpne)(a, b, pre, x_star=x_star, a_p=a_p)
    tm["solve"] = time.perf_counter() - t
    rep.decision = decision
    rep.escalated_from = failed
    rep.wall_ms = (time.perf_counter() - t0) * 1e3
    rep.timings = tm
    return rep
