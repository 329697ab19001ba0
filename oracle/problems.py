"""Algorithm-2 planted least-squares problems (restates src/probgen.py:50-123).

TEST INFRASTRUCTURE (see oracle/__init__.py).  Bit-identical to the reference
generator for the same (m, n, kappa, rho, seed); used by the tests and the
bench's CPU legs on the GPU box, where `/root/reference` does not exist.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .restatement import LANE_GAUSS, householder_qr, householder_steps, mix64, philox


@dataclass(frozen=True)
class Problem:
    a: np.ndarray
    b: np.ndarray
    x_star: np.ndarray
    rho: float
    kappa: float
    seed: int


def orthonormal_columns(m, k, seed):
    """src/probgen.py:50-55: Q of a seeded Gaussian (lane 3)."""
    if not 1 <= k <= m:
        raise ValueError(f"need 1 <= k <= m, got k={k}, m={m}")
    return householder_qr(philox(seed, LANE_GAUSS).standard_normal((m, k)))[0]


def planted_triangle(n, kappa, seed):
    """src/probgen.py:58-75: R with log-spaced singular values 1 .. 1/kappa."""
    if n < 1:
        raise ValueError(f"need n >= 1, got {n}")
    if kappa < 1:
        raise ValueError(f"need kappa >= 1, got {kappa}")
    if n == 1 and kappa != 1:
        raise ValueError("a 1 x 1 triangle always has condition 1")
    sv = 10.0 ** np.linspace(0.0, -math.log10(kappa), n)
    u = orthonormal_columns(n, n, mix64(seed, 1))
    v = orthonormal_columns(n, n, mix64(seed, 2))
    return householder_steps((u * sv) @ v.T)[2]


def planted_problem(m, n, kappa, rho, seed):
    """src/probgen.py:78-123: A = Q1 R, x* unit Gaussian, b = A x* + rho e,
    e orthogonal to range(A)."""
    if not m > n >= 1:
        raise ValueError(f"need m > n >= 1, got m={m}, n={n}")
    if kappa < 1 or rho < 0:
        raise ValueError("need kappa >= 1 and rho >= 0")
    q1 = orthonormal_columns(m, n, mix64(seed, 1))
    a = q1 @ planted_triangle(n, kappa, mix64(seed, 2))
    g = philox(mix64(seed, 3), LANE_GAUSS).standard_normal(n)
    x_star = g / np.linalg.norm(g)
    b = a @ x_star
    if rho > 0:
        for attempt in range(3):
            w = philox(mix64(seed, 4, attempt), LANE_GAUSS).standard_normal(m)
            e = w - q1 @ (q1.T @ w)
            ne = np.linalg.norm(e)
            if ne >= 1e-12:
                break
        else:
            raise RuntimeError("residual draws collapsed into range(a)")
        b = b + (rho / ne) * e
    return Problem(a, b, x_star, float(rho), float(kappa), int(seed))


def planted_problem_lapack(m, n, kappa, rho, seed):
    """Algorithm 2 (src/probgen.py:78-123) with LAPACK QR in place of the reference's
    Python Householder: the same problem distribution (Q1 orthonormal, R with log-spaced
    singular values 1 .. 1/kappa, x* unit, e orthogonal to range(A), ||e|| = rho), NOT
    bitwise the reference's draw.  For test sizes where the restated generator takes
    minutes (m x n >= 1e6); GPU and oracle are then compared on this same A, b."""
    if not m > n >= 1:
        raise ValueError(f"need m > n >= 1, got m={m}, n={n}")
    q1 = np.linalg.qr(philox(mix64(seed, 1), LANE_GAUSS).standard_normal((m, n)))[0]
    sv = 10.0 ** np.linspace(0.0, -math.log10(kappa), n)
    u = np.linalg.qr(philox(mix64(seed, 2, 1), LANE_GAUSS).standard_normal((n, n)))[0]
    v = np.linalg.qr(philox(mix64(seed, 2, 2), LANE_GAUSS).standard_normal((n, n)))[0]
    r = np.linalg.qr((u * sv) @ v.T, mode="r")
    a = q1 @ r
    g = philox(mix64(seed, 3), LANE_GAUSS).standard_normal(n)
    x_star = g / np.linalg.norm(g)
    b = a @ x_star
    if rho > 0:
        w = philox(mix64(seed, 4, 0), LANE_GAUSS).standard_normal(m)
        e = w - q1 @ (q1.T @ w)
        b = b + (rho / np.linalg.norm(e)) * e
    return Problem(np.ascontiguousarray(a), b, x_star, float(rho), float(kappa), int(seed))
