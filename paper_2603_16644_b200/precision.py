"""Precision levels, demotion, level-precision QR and the kappa0 selector.

Mirrors src/precision.py of the reference.  Level constants and the selection
rule are host logic; the kappa0 estimate (FP64 Gram of the full A on the DMMA
pipe, Cholesky, Hager) and the level QR (binary16 emulated op for op) run in
libsklsq.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .dense import QRFactors, _gram, _qr_r
from .device import WORKSPACE, DMat, as_dmat, call, device, stream_handle, to_host
from .errors import DimensionMismatch, Overflow


@dataclass(frozen=True)
class PrecisionLevel:
    """One of the three IEEE binary formats (src/precision.py:32-44)."""

    name: str
    unit_roundoff: float
    bound_roundoff: float
    dtype: type

    @property
    def code(self) -> int:
        return _lib.LEVEL_CODE[self.name]

    @property
    def torch_dtype(self):
        return {"binary16": torch.float16, "binary32": torch.float32, "binary64": torch.float64}[self.name]


BINARY16 = PrecisionLevel("binary16", 2.0 ** -11, 2.0 ** -11, np.float16)
BINARY32 = PrecisionLevel("binary32", 2.0 ** -24, 2.0 ** -23, np.float32)
BINARY64 = PrecisionLevel("binary64", 2.0 ** -53, 2.0 ** -52, np.float64)

_BY_NAME = {
    "binary16": BINARY16, "half": BINARY16,
    "binary32": BINARY32, "single": BINARY32,
    "binary64": BINARY64, "double": BINARY64,
}
_NEXT_HIGHER = {"binary16": BINARY32, "binary32": BINARY64}


def level_from_name(name):
    """src/precision.py:55-60."""
    try:
        return _BY_NAME[name]
    except (KeyError, TypeError):
        raise ValueError(f"unknown precision name {name!r}") from None


def next_higher(level):
    """src/precision.py:63-65."""
    return _NEXT_HIGHER.get(level.name)


@dataclass(frozen=True)
class PrecisionDecision:
    """src/precision.py:68-79."""

    kappa0: float
    selected: PrecisionLevel
    overflowed: bool


@dataclass(frozen=True)
class RoundedMatrix:
    """src/precision.py:82-87."""

    data: np.ndarray
    overflowed: bool


def round_to_precision(a, level):
    """Demotion with overflow flag (src/precision.py:90-103).  The flag comes
    from the device overflow pass; the data is the rounded matrix."""
    if isinstance(a, torch.Tensor):
        src = a
    else:
        src = torch.from_numpy(np.ascontiguousarray(np.asarray(a)))
    src64 = src.to(device(), dtype=torch.float64)
    if src64.dim() == 1:
        src64 = src64[:, None]
    over = C.c_int(0)
    if level.name != "binary64" and src64.numel():
        s2 = src64.contiguous()
        wp, wn = WORKSPACE.get(64)
        call("sk_level_overflow", s2.data_ptr(), s2.shape[0], s2.shape[1], s2.stride(0), level.code,
             C.byref(over), wp, wn, stream_handle())
    data = src.to(level.torch_dtype) if isinstance(a, torch.Tensor) else np.asarray(a).astype(level.dtype)
    return RoundedMatrix(data=data, overflowed=bool(over.value))


def select_precision(kappa0, overflowed):
    """src/precision.py:254-266: <4 half, <=8 single, else (or overflow) double."""
    if overflowed or not math.isfinite(kappa0):
        return BINARY64
    if kappa0 < 4:
        return BINARY16
    if kappa0 <= 8:
        return BINARY32
    return BINARY64


def _kappa0_from_gram(g: torch.Tensor):
    n = g.shape[0]
    k0 = C.c_double(math.nan)
    over = C.c_int(1)
    wp, wn = WORKSPACE.get(_lib.lib().sk_nxn_workspace(n))
    call("sk_kappa0_from_gram", g.data_ptr(), n, C.byref(k0), C.byref(over), wp, wn, stream_handle())
    return (math.nan, True) if over.value else (float(k0.value), False)


def _estimate_dev(ad: DMat):
    """kappa0 on a validated device matrix: FP64 SYRK + sk_kappa0_from_gram."""
    return _kappa0_from_gram(_gram(ad))


def estimate_log10_condition(a):
    """src/precision.py:205-251 -> (kappa0, overflowed)."""
    return _estimate_dev(as_dmat(a))


def decide_precision(a):
    """src/precision.py:269-276."""
    kappa0, overflowed = estimate_log10_condition(a)
    return PrecisionDecision(kappa0=kappa0, selected=select_precision(kappa0, overflowed),
                             overflowed=overflowed)


def _decide_dev(ad: DMat) -> PrecisionDecision:
    kappa0, overflowed = _estimate_dev(ad)
    return PrecisionDecision(kappa0=kappa0, selected=select_precision(kappa0, overflowed),
                             overflowed=overflowed)


def _qr_level_dev(a_s_colmajor: torch.Tensor, level: PrecisionLevel, d: int, n: int) -> torch.Tensor:
    """R of the (column-major, level dtype) sketch; raises RankDeficient / Overflow."""
    return _qr_r(a_s_colmajor, level.code, d, n)


def qr_in_precision(a, level):
    """Householder QR with all arithmetic in the given precision, factors promoted
    to binary64 (src/precision.py:153-202): binary16 takes the power-of-two scale
    from the f64 max and rounds a * scale once (:188-194), runs the op-for-op
    binary16 emulation and un-scales R after promotion; binary32 raises Overflow
    when the demotion overflows (:181-184); binary64 is householder_qr.  Q is
    accumulated from the reflectors in the same arithmetic (accumulate_thin_q).
    All on the device (sk_qr_in_precision_f64)."""
    from .dense import _qr_factors_dev
    ad = as_dmat(a)
    m, n = ad.shape
    if m < n:
        raise DimensionMismatch(f"need rows >= cols, got {m} x {n}")
    r, q = _qr_factors_dev(ad.t, level.code, True)
    return QRFactors(q=to_host(q), r=to_host(r))
