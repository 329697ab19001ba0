"""Algorithm-2 planted problems on the GPU, under the reference's
names (src/probgen.py:22-123): `LeastSquaresProblem`, `random_orthogonal_columns`,
`triangular_with_condition`, `generate_problem`, plus the device-scale
`generate_problem_device` (optionally one row shard of a multi-GPU problem).

Construction (src/probgen.py:78-123): A = Q1 R with Q1 orthonormal, R upper
triangular with log-spaced singular values 1 .. 1/kappa, x* a unit Gaussian,
b = A x* + rho e with e orthogonal to range(A).  All arithmetic runs in libsklsq:

  Q1 (m <= 262144)   householder_qr of the reference's Philox Gaussian (the host draw
                     is bitwise the reference's, src/probgen.py:50-55; the Q is the
                     device Householder Q, equal to numpy's to rounding)
  Q1 (device scale)  CholQR2 of a device Gaussian: G^T G (INT8/DMMA Gram),
                     Cholesky (sk_chol_factor_f64), in-place TRSM, twice
  R                  householder_reduce((U diag(sv)) V^T), U, V Haar (device QR)
  A = Q1 R           as the triangular solve A = Q1 (R^-1)^-1 (sk_trsm; R^-1 from an
                     n x n TRSM), in place over Q1 (the library has no NN GEMM; the
                     row-wise backward error is u kappa(R), the GEMM's own size)
  b = A x*, Q1 c     the residual kernel (sk_residual: r = A x - b)

Multi-GPU (`rank`, `world`): every rank draws the SAME R and x* and its own Q1_g and
w_g, and holds A_g = Q1_g R / sqrt(P) and e_g (norm rho / sqrt(P), orthogonal to
range(Q1_g)).  The stacked A then has A^T A = R^T R (so kappa(A) = kappa(R)), the
stacked e is orthogonal to range(A) with norm rho, and x* is the global solution.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, rng
from .dense import (TALL_QR_MAX_ROWS, _chol_factor, _gemv_t, _gram, _householder_r64, _qr_factors_dev, _trsm)
from .device import WORKSPACE, call, device, stream_handle, to_host
from .errors import DegenerateResidual


@dataclass(frozen=True)
class LeastSquaresProblem:
    """src/probgen.py:25-45: minimize ||a x - b|| with known x*."""

    a: np.ndarray
    b: np.ndarray
    x_star: np.ndarray
    rho: float
    kappa: float
    seed: int

    @property
    def m(self):
        return self.a.shape[0]

    @property
    def n(self):
        return self.a.shape[1]


# ------------------------------------------------------------- device pieces --
def _apply_residual(a: torch.Tensor, x: torch.Tensor, b: torch.Tensor | None, out: torch.Tensor) -> float:
    """out = A x - b (b None: A x); returns ||out||^2 (sk_residual)."""
    m, n = a.shape
    res = (C.c_double * 2)()
    zb = b if b is not None else torch.zeros(m, dtype=torch.float64, device=a.device)
    wp, wn = WORKSPACE.get(_lib.lib().sk_matrix_stats_workspace(m, n))
    call("sk_residual", a.data_ptr(), m, n, a.stride(0), x.data_ptr(), zb.data_ptr(), out.data_ptr(), res, wp, wn,
         stream_handle())
    return float(res[0])


def _matmul_nn(x: torch.Tensor, y: torch.Tensor) -> torch.Tensor:
    """X Y for n x n device matrices as the Gram (X^T)^T Y (sk_gram_f64 / INT8)."""
    return _gram(x.t().contiguous(), y.contiguous())


def _haar(n: int, gen: torch.Generator, dev) -> torch.Tensor:
    g = torch.randn(n, n, dtype=torch.float64, device=dev, generator=gen)
    r, q = _qr_factors_dev(g, 64, True)
    return q * torch.sign(torch.diagonal(r))[None, :]


def _rinv(r: torch.Tensor, scale: float = 1.0) -> torch.Tensor:
    """scale * R^-1 (upper) by an n x n right TRSM of the identity."""
    n = r.shape[0]
    eye = torch.eye(n, dtype=torch.float64, device=r.device) * scale
    return _trsm(eye, r, engine="dmma")


def planted_triangle_device(n: int, kappa: float, seed: int, dev=None) -> torch.Tensor:
    """R (n x n, upper) with singular values 10**linspace(0, -log10 kappa, n)
    (triangular_with_condition's spectrum, src/probgen.py:58-75)."""
    dev = dev or device()
    gen = torch.Generator(device=dev)
    gen.manual_seed(int(seed) & 0x7FFFFFFFFFFFFFFF)
    sv = 10.0 ** torch.linspace(0.0, -math.log10(kappa), n, dtype=torch.float64, device=dev)
    u, v = _haar(n, gen, dev), _haar(n, gen, dev)
    return _householder_r64(_matmul_nn(u * sv[None, :], v.t()))


def orthonormal_columns_device(m: int, n: int, seed: int, dev=None, out=None) -> torch.Tensor:
    """CholQR2 of an m x n device Gaussian, in place (one m x n buffer)."""
    dev = dev or device()
    gen = torch.Generator(device=dev)
    gen.manual_seed((int(seed) * 2654435761 + 1) & 0x7FFFFFFFFFFFFFFF)
    x = out if out is not None else torch.empty((m, n), dtype=torch.float64, device=dev)
    rows = 1 << 22
    for r0 in range(0, m, rows):      # chunked to bound the generator's scratch
        x[r0:r0 + rows].normal_(generator=gen)
    for _ in range(2):
        _trsm(x, _chol_factor(_gram(x)), out=x)
    return x


def generate_problem_device(m: int, n: int, kappa: float, rho: float, seed: int, dev=None, rank: int = 0,
                            world: int = 1):
    """-> (A, b, x_star) as CUDA float64 tensors (A row-major m x n): the whole problem
    (world = 1) or row shard `rank` of a `world`-shard problem with world * m rows (see
    the module docstring).  Synthetic-data setup; not part of any timed solve."""
    if not m > n >= 1:
        raise ValueError(f"need m > n >= 1, got m={m}, n={n}")
    if kappa < 1 or rho < 0:
        raise ValueError("need kappa >= 1 and rho >= 0")
    dev = dev or device()
    q1 = orthonormal_columns_device(m, n, seed + 7919 * rank, dev)      # Q1_g: per rank
    r = planted_triangle_device(n, kappa, seed + 1, dev)                # R: the same on every rank
    gen = torch.Generator(device=dev)
    gen.manual_seed((int(seed) * 40503 + 7) & 0x7FFFFFFFFFFFFFFF)
    g = torch.randn(n, dtype=torch.float64, device=dev, generator=gen)
    x_star = g / torch.linalg.vector_norm(g)                           # x*: the same on every rank
    e = None
    if rho > 0:
        wgen = torch.Generator(device=dev)
        wgen.manual_seed((int(seed) * 40503 + 11 + 104729 * rank) & 0x7FFFFFFFFFFFFFFF)
        w = torch.randn(m, dtype=torch.float64, device=dev, generator=wgen)
        e = torch.empty(m, dtype=torch.float64, device=dev)
        ee = _apply_residual(q1, _gemv_t(q1, w), w, e)                  # e = -(w - Q1 Q1^T w)
        e *= -(rho / math.sqrt(world)) / math.sqrt(ee)
    a = _trsm(q1, _rinv(r, math.sqrt(world)), out=q1)                   # A_g = Q1_g R / sqrt(P), in place
    b = torch.empty(m, dtype=torch.float64, device=dev)
    _apply_residual(a, x_star, None, b)                                 # b = A x*
    if e is not None:
        b += e
    return a, b, x_star


# -------------------------------------------------- the reference's entry points --
def random_orthogonal_columns(m, k, seed):
    """src/probgen.py:50-55: Q of the seeded Philox Gaussian (lane 3), on the device."""
    if not 1 <= k <= m:
        raise ValueError(f"need 1 <= k <= m, got k={k}, m={m}")
    return to_host(_orthonormal_from_host_gaussian(m, k, seed))


def _orthonormal_from_host_gaussian(m, k, seed) -> torch.Tensor:
    g = torch.from_numpy(rng.stream(seed, rng.LANE_GAUSSIAN).standard_normal((m, k))).to(device())
    if m <= TALL_QR_MAX_ROWS:
        return _qr_factors_dev(g, 64, True)[1]
    for _ in range(2):   # beyond the Householder kernel's height: CholQR2
        _trsm(g, _chol_factor(_gram(g)), out=g)
    return g


def _triangle_dev(n, kappa, seed) -> torch.Tensor:
    if n < 1:
        raise ValueError(f"need n >= 1, got {n}")
    if kappa < 1:
        raise ValueError(f"need kappa >= 1, got {kappa}")
    if n == 1 and kappa != 1:
        raise ValueError("a 1 x 1 triangle always has condition 1")
    sv = torch.from_numpy(10.0 ** np.linspace(0.0, -math.log10(kappa), n)).to(device())
    u = _orthonormal_from_host_gaussian(n, n, rng.mix64(seed, 1))
    v = _orthonormal_from_host_gaussian(n, n, rng.mix64(seed, 2))
    return _householder_r64(_matmul_nn(u * sv[None, :], v.t()))


def triangular_with_condition(n, kappa, seed):
    """src/probgen.py:58-75: upper R with ||R|| = 1 and condition number kappa."""
    return to_host(_triangle_dev(n, kappa, seed))


def generate_problem(m, n, kappa, rho, seed):
    """src/probgen.py:78-123: the reference's random streams (Philox lanes, mix64
    sub-seeds; the Gaussians are bitwise the reference's), device arithmetic.
    Raises DegenerateResidual after three residual draws in range(A)."""
    if not m > n >= 1:
        raise ValueError(f"need m > n >= 1, got m={m}, n={n}")
    if kappa < 1:
        raise ValueError(f"need kappa >= 1, got {kappa}")
    if rho < 0:
        raise ValueError(f"need rho >= 0, got {rho}")
    dev = device()
    q1 = _orthonormal_from_host_gaussian(m, n, rng.mix64(seed, 1))
    r = _triangle_dev(n, kappa, rng.mix64(seed, 2))
    g = rng.stream(rng.mix64(seed, 3), rng.LANE_GAUSSIAN).standard_normal(n)
    x_star = g / np.linalg.norm(g)
    xd = torch.from_numpy(x_star).to(dev)
    e = None
    if rho > 0:
        e = torch.empty(m, dtype=torch.float64, device=dev)
        for attempt in range(3):
            w = torch.from_numpy(rng.stream(rng.mix64(seed, 4, attempt), rng.LANE_GAUSSIAN).standard_normal(m)).to(dev)
            ee = _apply_residual(q1, _gemv_t(q1, w), w, e)             # -(w - Q1 Q1^T w)
            if math.sqrt(ee) >= 1e-12:
                break
        else:
            raise DegenerateResidual("residual draws collapsed into range(a)")
        e *= -rho / math.sqrt(ee)
    a = _trsm(q1, _rinv(r), out=q1)
    b = torch.empty(m, dtype=torch.float64, device=dev)
    _apply_residual(a, xd, None, b)
    if e is not None:
        b += e
    return LeastSquaresProblem(a=to_host(a), b=to_host(b), x_star=x_star, rho=float(rho), kappa=float(kappa),
                               seed=int(seed))


# archive I/O (src/probgen.py:126-159) lives in mmio.py; re-exported under the reference's names
from .mmio import FORMAT_VERSION, load_problem, save_problem  # noqa: E402,F401
