"""Algorithm-2 planted problems generated directly on the GPU.

Same construction as the reference generator (src/probgen.py:58-123): A = Q1 R
with Q1 orthonormal, R upper triangular with log-spaced singular values
1 .. 1/kappa, x* a unit Gaussian, b = A x* + rho e with e orthogonal to
range(A).  The reference builds Q1 with a Python Householder QR of an m x n
Gaussian, which is infeasible at m = 4M; here:

  Q1 = CholQR2 of a device Gaussian   (Gram on the DMMA pipe (sk_gram_f64),
                                        n x n Cholesky, in-place TRSM (sk_trsm))
  R  = R factor (sk_qr_r, binary64) of U diag(sv) V^T, U, V Haar orthogonal
  A  = Q1 R,  e = w - Q1 (Q1^T w)

Synthetic-data setup only: it is not part of the timed solve.  The few n x n
factorisations and the one tall GEMM use torch (cuSOLVER/cuBLAS) as plumbing.
It is a different random stream from the reference generator (torch Philox on
the device), so problems are statistically, not bitwise, equivalent; parity
tests use the oracle generator at small sizes.
"""

from __future__ import annotations

import math

import torch

from .dense import _gemv_t, _gram, _householder_r64, _trsm


def _haar(n: int, gen: torch.Generator, dev) -> torch.Tensor:
    g = torch.randn(n, n, dtype=torch.float64, device=dev, generator=gen)
    q, r = torch.linalg.qr(g)
    return q * torch.sign(torch.diagonal(r))[None, :]


def planted_triangle_device(n: int, kappa: float, seed: int, dev=None) -> torch.Tensor:
    """R (n x n, upper) with singular values 10**linspace(0, -log10 kappa, n)."""
    dev = dev or torch.device("cuda")
    gen = torch.Generator(device=dev)
    gen.manual_seed(int(seed) & 0x7FFFFFFFFFFFFFFF)
    sv = 10.0 ** torch.linspace(0.0, -math.log10(kappa), n, dtype=torch.float64, device=dev)
    u, v = _haar(n, gen, dev), _haar(n, gen, dev)
    return _householder_r64((u * sv[None, :]) @ v.T)


def orthonormal_columns_device(m: int, n: int, seed: int, dev=None, out=None) -> torch.Tensor:
    """CholQR2 of an m x n Gaussian, in place (one m x n buffer)."""
    dev = dev or torch.device("cuda")
    gen = torch.Generator(device=dev)
    gen.manual_seed((int(seed) * 2654435761 + 1) & 0x7FFFFFFFFFFFFFFF)
    x = out if out is not None else torch.empty((m, n), dtype=torch.float64, device=dev)
    rows = 1 << 22
    for r0 in range(0, m, rows):      # chunked to bound the generator's scratch
        x[r0:r0 + rows].normal_(generator=gen)
    for _ in range(2):
        g = _gram(x)
        rx = torch.linalg.cholesky(g).T.contiguous()
        _trsm(x, rx, out=x)
    return x


def generate_problem_device(m: int, n: int, kappa: float, rho: float, seed: int, dev=None):
    """-> (A, b, x_star) as CUDA float64 tensors (A row-major m x n)."""
    if not m > n >= 1:
        raise ValueError(f"need m > n >= 1, got m={m}, n={n}")
    dev = dev or torch.device("cuda")
    q1 = orthonormal_columns_device(m, n, seed, dev)
    r = planted_triangle_device(n, kappa, seed + 1, dev)
    a = q1 @ r
    gen = torch.Generator(device=dev)
    gen.manual_seed((int(seed) * 40503 + 7) & 0x7FFFFFFFFFFFFFFF)
    g = torch.randn(n, dtype=torch.float64, device=dev, generator=gen)
    x_star = g / torch.linalg.vector_norm(g)
    b = a @ x_star
    if rho > 0:
        w = torch.randn(m, dtype=torch.float64, device=dev, generator=gen)
        e = w - q1 @ _gemv_t(q1, w)
        b = b + (rho / torch.linalg.vector_norm(e)) * e
    del q1
    return a, b, x_star
