"""Compiled pieces of the CPU oracle (TEST INFRASTRUCTURE, see oracle/__init__.py).

`qr_at_level16` is src/precision.py:188-202 (binary16 branch of qr_in_precision,
R only) with the Householder loop in C (oracle/csrc/householder16.c, built by the
Makefile into oracle/_build/liboracle.so): the same prescale and demotion in numpy,
the same per-operation binary16 rounding and pairwise trees, so R is bitwise the
reference's (pinned in tests/test_oracle_golden.py against qr16_golden.json).
"""

from __future__ import annotations

import ctypes as C
import math
import os

import numpy as np

from .restatement import Overflow, RankDeficient, demote

_LIB = None
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_build", "liboracle.so")


def lib():
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing: run `make oracle`")
        _LIB = C.CDLL(LIB_PATH)
        _LIB.oracle_householder16.restype = C.c_int
        _LIB.oracle_householder16.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.POINTER(C.c_int)]
    return _LIB


_MSG = {1: "pivot column {} is zero at working precision", 2: "reflector {} vanished at working precision",
        3: "reflector {} norm underflowed at working precision"}


def householder16_r(data16: np.ndarray) -> np.ndarray:
    """R (binary16, n x n) of householder_reduce(data16, HALF_OPS), src/dense.py:108-161."""
    d, n = data16.shape
    w = np.asfortranarray(data16.astype(np.float16, copy=True))
    fail = C.c_int(-1)
    rc = lib().oracle_householder16(w.ctypes.data, d, n, None, C.byref(fail))
    if rc:
        raise RankDeficient(_MSG[rc].format(fail.value))
    return np.array(w[:n, :], copy=True)


def qr_at_level16(a) -> np.ndarray:
    """qr_in_precision(a, BINARY16).r (src/precision.py:188-202), R only."""
    work = np.asarray(a, dtype=np.float64)
    peak = float(np.abs(work).max())
    if peak == 0:
        raise RankDeficient("zero matrix")
    scale = 2.0 ** -math.frexp(peak)[1]
    data, _ = demote(work * scale, "binary16")
    r16 = householder16_r(data)
    if not np.isfinite(r16).all():
        raise Overflow("binary16 computation produced non-finite values")
    return r16.astype(np.float64) / scale
