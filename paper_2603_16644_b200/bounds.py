"""Measured inputs of the paper's error bounds, on the device.

Mirrors the measurement half of src/bounds.py (the reference's `BoundInputs`,
`ProblemDiagnostics`, `measure_problem` :178-199 and `measure_bound_inputs`
:202-255): the condition numbers kappa(A), kappa(R_s), kappa(A_p), kappa(A_p^T A), the
nu factors and the residual ratios, from the device condition diagnostics
(`condition_diagnostics`: Householder / TSQR R factor + one-sided Jacobi) and the
residual kernel.  The closed-form bound formulas (`eta1`, `bound_ls`, `bound_ne_family`,
`bound_pne`, `bound_hpne`, `bound_notnormal`, src/bounds.py:55-156) are scalar host
arithmetic on those measurements; they are restated here for the sweep harness
(harness.py) with the reference's argument checks and exceptions.

Tall matrices: the reference reduces a tall matrix to its Householder R before the
Jacobi sweep; here `tall_route="tsqr"` (the default) does the same through TSQR, which
stays accurate at any kappa; "gram" takes the n x n Cholesky factor of the Gram instead
(fast, accurate while kappa << 1e8).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, replace

import numpy as np
import torch

from .dense import ConditionDiagnostics, _gemv_t, _householder_r64, _jacobi_sv, _gram, _rm, TALL_QR_MAX_ROWS
from .device import DMat, as_dmat, as_dvec, to_host
from .errors import MissingField, NoConvergence, PoleAtOne, RankDeficient

_U2_DEFAULT = 2.0 ** -52


@dataclass(frozen=True)
class BoundInputs:
    """src/bounds.py:29-50: measured quantities a bound evaluation may need."""

    kappa_a: float | None = None
    kappa_rs: float | None = None
    kappa_ap: float | None = None
    kappa_apta: float | None = None
    nu_pne: float | None = None
    nu_hpne: float | None = None
    u1: float | None = None
    u2: float | None = None
    eps_a: float | None = None
    eps_b: float | None = None
    eps_p: float | None = None
    eps_s: float | None = None
    res_ratio_a: float | None = None
    res_ratio_ap: float | None = None

    def updated(self, **kwargs):
        return replace(self, **kwargs)

    def need(self, *names):
        for name in names:
            if getattr(self, name) is None:
                raise MissingField(f"bound needs {name!r} but it was not measured")


def _need(inputs, *names):
    inputs.need(*names)


def eta1(kappa_rs, u1):
    """src/bounds.py:55-66: |k u / (1 - k u)|; PoleAtOne within 1e-15 of the pole."""
    x = kappa_rs * u1
    if abs(x - 1.0) <= 1e-15:
        raise PoleAtOne(f"kappa_rs * u1 = {x} is at the pole")
    return abs(x / (1.0 - x))


def bound_ls(inputs):
    """src/bounds.py:69-76: kappa_a eps_a (1 + kappa_a res_ratio_a)."""
    _need(inputs, "kappa_a", "eps_a", "res_ratio_a")
    k = inputs.kappa_a
    return k * inputs.eps_a * (1.0 + k * inputs.res_ratio_a)


def bound_ne_family(inputs, kind="normal"):
    """src/bounds.py:79-90: kappa_a^2 eps_a (res_ratio_a + 1 + eps_a)."""
    if kind not in ("normal", "seminormal"):
        raise ValueError(f"kind must be normal or seminormal, got {kind!r}")
    _need(inputs, "kappa_a", "eps_a", "res_ratio_a")
    k = inputs.kappa_a
    return k * k * inputs.eps_a * (inputs.res_ratio_a + 1.0 + inputs.eps_a)


def bound_pne(inputs, variant="new"):
    """src/bounds.py:93-115 ("old": residual of the preconditioned system, "new": of
    the original system)."""
    if variant == "old":
        _need(inputs, "kappa_rs", "kappa_ap", "nu_pne", "u1", "u2", "res_ratio_ap")
        e1 = eta1(inputs.kappa_rs, inputs.u1)
        return inputs.kappa_rs * inputs.kappa_ap * inputs.nu_pne * (
            inputs.u2 + inputs.kappa_ap * e1 * (inputs.res_ratio_ap + inputs.u2))
    if variant == "new":
        _need(inputs, "kappa_rs", "kappa_ap", "kappa_a", "u2", "res_ratio_a")
        return inputs.kappa_rs * inputs.kappa_ap * inputs.u2 * (
            inputs.kappa_ap * inputs.kappa_rs * inputs.res_ratio_a + 1.0 + inputs.kappa_a * inputs.u2)
    raise ValueError(f"variant must be old or new, got {variant!r}")


def bound_hpne(inputs, variant="new"):
    """src/bounds.py:118-140."""
    if variant == "old":
        _need(inputs, "kappa_apta", "nu_hpne", "kappa_rs", "u1", "u2", "res_ratio_a")
        e1 = eta1(inputs.kappa_rs, inputs.u1)
        return inputs.kappa_apta * inputs.nu_hpne * (e1 * inputs.res_ratio_a + (1.0 + e1) * inputs.u2)
    if variant == "new":
        _need(inputs, "kappa_apta", "nu_hpne", "kappa_rs", "kappa_a", "u2", "res_ratio_a")
        return inputs.kappa_apta * inputs.nu_hpne * inputs.u2 * (
            inputs.kappa_rs * inputs.res_ratio_a + 1.0 + inputs.kappa_a * inputs.u2)
    raise ValueError(f"variant must be old or new, got {variant!r}")


def bound_notnormal(inputs, kappa_bta, nu_b):
    """src/bounds.py:143-156: kappa_bta nu_b (eps_b res_ratio_a + (1 + eps_b) eps_a)."""
    _need(inputs, "eps_a", "eps_b", "res_ratio_a")
    return kappa_bta * nu_b * (inputs.eps_b * inputs.res_ratio_a + (1.0 + inputs.eps_b) * inputs.eps_a)


@dataclass
class ProblemDiagnostics:
    """src/bounds.py:160-175: solution-independent norms and condition numbers."""

    norm_a: float
    kappa_a: float
    norm_rs: float | None = None
    kappa_rs: float | None = None
    norm_ap: float | None = None
    kappa_ap: float | None = None
    norm_apta: float | None = None
    kappa_apta: float | None = None
    a_p: torch.Tensor | None = None


def _cond(at: torch.Tensor, tall_route: str) -> ConditionDiagnostics:
    """condition_diagnostics (src/dense.py:418-448) of a device matrix; tall inputs are
    reduced to their R factor (TSQR) or Gram Cholesky factor first."""
    from .dense import _chol_factor
    at = _rm(at)
    if at.shape[0] < at.shape[1]:
        at = at.t().contiguous()
    m, n = at.shape
    w = at
    if m > n:
        if m > TALL_QR_MAX_ROWS and tall_route == "gram":
            w = _chol_factor(_gram(at))
        else:
            try:
                w = _householder_r64(at)
            except RankDeficient:
                w = at
    sv = _jacobi_sv(w)
    cond = float(sv[0] / sv[-1]) if sv[-1] > 0 else float("inf")
    return ConditionDiagnostics(two_norm=float(sv[0]), two_norm_condition=cond, singular_values=sv)


def _resid_norm(a: torch.Tensor, x: torch.Tensor, b: torch.Tensor) -> float:
    """||A x - b|| by the residual kernel (sk_residual)."""
    import ctypes as C
    from . import _lib
    from .device import WORKSPACE, call, stream_handle
    a = _rm(a)
    m, n = a.shape
    out = (C.c_double * 2)()
    wp, wn = WORKSPACE.get(_lib.lib().sk_matrix_stats_workspace(m, n))
    call("sk_residual", a.data_ptr(), m, n, a.stride(0), x.contiguous().data_ptr(), b.contiguous().data_ptr(), None,
         out, wp, wn, stream_handle())
    return math.sqrt(out[0])


def measure_problem(problem, pre=None, a_p=None, *, tall_route="tsqr"):
    """src/bounds.py:178-199: kappa(A) and, with a preconditioner, kappa(R_s),
    kappa(A_p), kappa(A_p^T A) and their norms (A_p computed on the device when not
    given).  `problem` needs `.a` (numpy or torch)."""
    from .solvers import _precondition_dev
    ad = as_dmat(problem.a)
    diag_a = _cond(ad.t, tall_route)
    if pre is None:
        return ProblemDiagnostics(norm_a=diag_a.two_norm, kappa_a=diag_a.two_norm_condition)
    if a_p is None:
        ap = _precondition_dev(ad, pre, diagnostics=False)
    else:
        ap = a_p if isinstance(a_p, torch.Tensor) and a_p.is_cuda else as_dmat(a_p, "a_p").t
    diag_rs = _cond(pre.r_device(), tall_route)
    diag_ap = _cond(ap, tall_route)
    diag_apta = _cond(_gram(ap, ad.t), tall_route)          # a_p.T @ a (n x n)
    return ProblemDiagnostics(norm_a=diag_a.two_norm, kappa_a=diag_a.two_norm_condition,
                              norm_rs=diag_rs.two_norm, kappa_rs=diag_rs.two_norm_condition,
                              norm_ap=diag_ap.two_norm, kappa_ap=diag_ap.two_norm_condition,
                              norm_apta=diag_apta.two_norm, kappa_apta=diag_apta.two_norm_condition, a_p=ap)


def measure_bound_inputs(problem, report, pre=None, u1=None, u2=None, a_p=None, diagnostics=None, *,
                         tall_route="tsqr"):
    """src/bounds.py:202-255: fill a BoundInputs record from a solved instance
    (eps_a = eps_p = u2, eps_s = u1, eps_b left None as in the reference)."""
    if u2 is None:
        u2 = _U2_DEFAULT
    if u1 is None:
        u1 = pre.computed_in.bound_roundoff if pre is not None else u2
    if diagnostics is None:
        diagnostics = measure_problem(problem, pre, a_p, tall_route=tall_route)
    ad = as_dmat(problem.a)
    bd = as_dvec(problem.b, ad.shape[0])
    x = torch.from_numpy(np.ascontiguousarray(report.x_hat, dtype=np.float64)).to(bd.device)
    norm_x = float(torch.linalg.vector_norm(x))
    res_ratio_a = _resid_norm(ad.t, x, bd) / (diagnostics.norm_a * norm_x)
    inputs = BoundInputs(kappa_a=diagnostics.kappa_a, u1=u1, u2=u2, eps_a=u2, eps_p=u2, eps_s=u1,
                         res_ratio_a=res_ratio_a)
    if pre is None:
        return inputs
    r = pre.r_device()
    y = _gemv_t(r.t().contiguous(), x)                      # R_s x (upper-triangular matvec)
    norm_y = float(torch.linalg.vector_norm(y))
    ap = diagnostics.a_p if diagnostics.a_p is not None else measure_problem(problem, pre, a_p).a_p
    return inputs.updated(
        kappa_rs=diagnostics.kappa_rs, kappa_ap=diagnostics.kappa_ap, kappa_apta=diagnostics.kappa_apta,
        nu_pne=norm_y / (diagnostics.norm_rs * norm_x),
        nu_hpne=diagnostics.norm_ap * diagnostics.norm_a / diagnostics.norm_apta,
        res_ratio_ap=_resid_norm(ap, y, bd) / (diagnostics.norm_ap * norm_y))
