"""SRTT sketch operators (mirrors src/sketch.py of the reference).

`make_sketch` draws signs and sampled rows on the host with the reference's
Philox streams (so the operator is bitwise the reference's for the same seed);
`apply_sketch` runs on the device: the sampled rows of the orthonormal DCT-II /
WHT are generated in-kernel from the closed form and multiplied against the
level-rounded, sign-flipped A on the tensor pipe (libsklsq sk_sketch_partial),
then scaled and rounded to the level (sk_sketch_finalize).
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, rng
from .device import WORKSPACE, DMat, as_dmat, call, device, stream_handle, to_host
from .errors import DimensionMismatch, Overflow

DCT2 = "dct2"
WHT = "wht"
TRANSFORMS = (DCT2, WHT)


@dataclass(frozen=True)
class SketchOperator:
    """A realised sketch (src/sketch.py:59-82): signs (length m_pad) and d
    sampled rows of the padded transform."""

    m: int
    d: int
    transform: str
    seed: int
    signs: np.ndarray
    sampled_rows: np.ndarray

    @property
    def m_pad(self):
        if self.signs is None:   # device-drawn operator (_make_sketch_dev): signs live on the GPU
            return _next_pow2(self.m) if self.transform == WHT else self.m
        return self.signs.shape[0]

    def descriptor(self):
        return {"m": self.m, "d": self.d, "transform": self.transform, "seed": self.seed}


def _next_pow2(m):
    return 1 << max(m - 1, 0).bit_length() if m > 1 else 1


def make_sketch(m, d, transform=DCT2, seed=0):
    """src/sketch.py:89-112 (same Philox lanes -> bitwise the same operator)."""
    if transform not in TRANSFORMS:
        raise ValueError(f"unknown transform {transform!r}, expected {TRANSFORMS}")
    if m < 1 or d < 1:
        raise ValueError(f"need m >= 1 and d >= 1, got m={m}, d={d}")
    m_pad = _next_pow2(m) if transform == WHT else m
    if d > m_pad:
        raise ValueError(f"sample count d={d} exceeds padded height {m_pad}")
    signs = rng.stream(seed, rng.LANE_SKETCH_SIGNS).integers(0, 2, m_pad) * 2.0 - 1.0
    rows = rng.stream(seed, rng.LANE_SKETCH_ROWS).integers(0, m_pad, d)
    return SketchOperator(m=int(m), d=int(d), transform=transform, seed=int(seed), signs=signs,
                          sampled_rows=rows)


def _make_sketch_dev(m, d, transform=DCT2, seed=0):
    """make_sketch for the device pipeline: the d sampled rows are drawn on the host
    (same Philox lane, d draws), the m_pad signs on the device by sk_sketch_signs
    (bitwise the host draw, no m_pad-long host loop or copy).  Returns
    (SketchOperator with signs=None, DeviceSketch)."""
    if transform not in TRANSFORMS:
        raise ValueError(f"unknown transform {transform!r}, expected {TRANSFORMS}")
    if m < 1 or d < 1:
        raise ValueError(f"need m >= 1 and d >= 1, got m={m}, d={d}")
    m_pad = _next_pow2(m) if transform == WHT else m
    if d > m_pad:
        raise ValueError(f"sample count d={d} exceeds padded height {m_pad}")
    rows = rng.stream(seed, rng.LANE_SKETCH_ROWS).integers(0, m_pad, d)
    op = SketchOperator(m=int(m), d=int(d), transform=transform, seed=int(seed), signs=None, sampled_rows=rows)
    return op, DeviceSketch(op)


def sketch_from_descriptor(desc):
    """src/sketch.py:115-118."""
    return make_sketch(int(desc["m"]), int(desc["d"]), desc["transform"], int(desc["seed"]))


class DeviceSketch:
    """Device-resident operator data (signs as +-1 doubles, rows as int64)."""

    def __init__(self, op: SketchOperator):
        dev = device()
        self.op = op
        if op.signs is None:
            self.signs = torch.empty(op.m_pad, dtype=torch.float64, device=dev)
            key_lo = int(op.seed) & rng.MASK64
            key_hi = int(rng.LANE_SKETCH_SIGNS) & rng.MASK64
            call("sk_sketch_signs", key_lo, key_hi, op.m_pad, self.signs.data_ptr(), stream_handle())
        else:
            self.signs = torch.from_numpy(np.ascontiguousarray(op.signs, dtype=np.float64)).to(dev)
        self.rows = torch.from_numpy(np.ascontiguousarray(op.sampled_rows, dtype=np.int64)).to(dev)


ALGO = {"auto": 0, "dmma": 1, "tc": 2, "fft": 3}


def _sketch_sum(dsk: DeviceSketch, at: torch.Tensor, level_code: int, row_offset: int = 0,
                out: torch.Tensor | None = None, accumulate: bool = False,
                overflow_flag: torch.Tensor | None = None, algo: str = "auto") -> tuple[torch.Tensor, torch.Tensor]:
    """Unscaled partial sum (d x n, column-major) of Omega[:, rows of this block] A_block.
    algo: "auto" (tcgen05 for binary16, DMMA otherwise), "tc" or "dmma"."""
    op = dsk.op
    m_local, n = at.shape
    d = op.d
    dev = at.device
    if out is None:
        out = torch.zeros((n, d), dtype=torch.float64, device=dev)   # column-major d x n
    if overflow_flag is None:
        overflow_flag = torch.zeros(1, dtype=torch.int32, device=dev)
    wp, wn = WORKSPACE.get(_lib.lib().sk_sketch_workspace_ex(level_code, _lib.TRANSFORM_CODE[op.transform],
                                                             m_local, op.m_pad, n, d))
    call("sk_sketch_partial_ex", level_code, _lib.TRANSFORM_CODE[op.transform], at.data_ptr(), at.stride(0),
         m_local, row_offset, op.m_pad, n, dsk.signs.data_ptr(), dsk.rows.data_ptr(), d, out.data_ptr(),
         d, int(accumulate), overflow_flag.data_ptr(), wp, wn, stream_handle(), ALGO[algo])
    return out, overflow_flag


def _sketch_finalize(total: torch.Tensor, op: SketchOperator, level, want_f64: bool = False):
    """-> (A_s column-major in the level dtype [n x d storage], optional f64 row-major d x n)."""
    n, d = total.shape
    a_s = torch.empty((n, d), dtype=level.torch_dtype, device=total.device)
    f64 = torch.empty((d, n), dtype=torch.float64, device=total.device) if want_f64 else None
    call("sk_sketch_finalize", level.code, total.data_ptr(), d, d, n, op.m_pad, a_s.data_ptr(),
         f64.data_ptr() if f64 is not None else None, stream_handle())
    return a_s, f64


def _apply_dev(op: SketchOperator, ad: DMat, level, dsk: DeviceSketch | None = None, want_f64=False):
    """Device sketch of a validated matrix at `level` (demotion fused into the
    operand load).  Raises Overflow when the demotion leaves the level's range
    (src/solvers.py:191-193)."""
    if ad.shape[0] != op.m:
        raise DimensionMismatch(f"operator built for {op.m} rows, got {ad.shape[0]}")
    dsk = dsk or DeviceSketch(op)
    total, flag = _sketch_sum(dsk, ad.t, level.code)
    if int(flag.item()):
        raise Overflow(f"input exceeds the {level.name} range")
    return _sketch_finalize(total, op, level, want_f64)


def apply_sketch(op, a):
    """src/sketch.py:138-169: the d x n sketch in the dtype of `a`."""
    from .precision import BINARY16, BINARY32, BINARY64   # local: avoid an import cycle
    if isinstance(a, torch.Tensor):
        tdt = a.dtype
        level = {torch.float16: BINARY16, torch.float32: BINARY32}.get(tdt, BINARY64)
    else:
        arr = np.asarray(a)
        level = {np.dtype(np.float16): BINARY16, np.dtype(np.float32): BINARY32}.get(arr.dtype, BINARY64)
    ad = as_dmat(a)
    if ad.shape[0] != op.m:
        raise DimensionMismatch(f"operator built for {op.m} rows, got {ad.shape[0]}")
    dsk = DeviceSketch(op)
    total, _ = _sketch_sum(dsk, ad.t, level.code)
    _, f64 = _sketch_finalize(total, op, level, want_f64=True)
    out = to_host(f64).astype(level.dtype)   # exact: every value is representable in the level
    return out if not isinstance(a, torch.Tensor) else torch.from_numpy(out).to(a.device)


# ------------------------------------------------ embedding theory helpers ---
@dataclass(frozen=True)
class EmbeddingParams:
    """src/sketch.py:29-57: inputs to the subspace-embedding sample-size bound
    (m >= n >= 1, coherence mu in (0, 1] and >= n/m, eps and delta in (0, 1))."""

    m: int
    n: int
    mu: float
    eps: float
    delta: float

    def __post_init__(self):
        if self.n < 1 or self.m < self.n:
            raise ValueError(f"need m >= n >= 1, got m={self.m}, n={self.n}")
        if not 0 < self.mu <= 1:
            raise ValueError(f"coherence must be in (0, 1], got {self.mu}")
        if self.mu * self.m < self.n * (1 - 1e-12):
            raise ValueError(f"coherence {self.mu} below the floor n/m = {self.n / self.m}")
        if not 0 < self.eps < 1:
            raise ValueError(f"distortion must be in (0, 1), got {self.eps}")
        if not 0 < self.delta < 1:
            raise ValueError(f"failure probability must be in (0, 1), got {self.delta}")


def sample_size_lower_bound(params):
    """src/sketch.py:172-179: ceil(2 m mu (1 + eps/3) ln(n/delta) / eps^2)."""
    raw = 2.0 * params.m * params.mu * (1.0 + params.eps / 3.0) * math.log(params.n / params.delta) / params.eps ** 2
    return int(math.ceil(raw))


def coherence(q):
    """src/sketch.py:182-195: largest squared row norm of an orthonormal-column q, on the
    device (q^T q by the Gram kernel, ||q^T q - I|| by the Jacobi diagnostics);
    NotOrthonormal beyond 1e-10."""
    from .dense import _gram, condition_diagnostics
    from .errors import NotOrthonormal
    qd = as_dmat(q, "q")
    n = qd.shape[1]
    dev = _gram(qd) - torch.eye(n, dtype=torch.float64, device=qd.t.device)
    if condition_diagnostics(dev).two_norm > 1e-10:
        raise NotOrthonormal("columns are not orthonormal to 1e-10")
    return float(torch.einsum("ij,ij->i", qd.t, qd.t).max())
