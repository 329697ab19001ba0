"""Device plumbing: validated device matrices, workspaces, streams, C-ABI calls.

PyTorch is used only for device memory, streams and host<->device copies.  All
arithmetic on the solve path happens in libsklsq.so (see `_lib`).
"""

from __future__ import annotations

import ctypes as C
import math
import threading
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import DimensionMismatch, raise_for_code

_FLOAT_NP = (np.float16, np.float32, np.float64)
_TORCH_CODE = {torch.float16: 2, torch.float32: 4, torch.float64: 8}


def device() -> torch.device:
    if not torch.cuda.is_available():
        raise _lib.LibraryUnavailable("no CUDA device: the B200 path has no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def stream_handle() -> int:
    return torch.cuda.current_stream().cuda_stream


def call(fn_name: str, *args, status: "_lib.SkStatus | None" = None) -> int:
    """Invoke an sk_* entry point and raise the reference exception on failure."""
    lib = _lib.lib()
    rc = getattr(lib, fn_name)(*args)
    if rc != 0:
        msg = _lib.last_error()
        raise_for_code(rc, msg)
    return rc


# ---------------------------------------------------------------- workspace --
class _WorkspacePool:
    """One growable scratch buffer per (device, stream); calls on a stream are
    ordered, so consecutive kernels can share it."""

    def __init__(self):
        self._bufs = {}
        self._lock = threading.Lock()

    def get(self, nbytes: int) -> tuple[int, int]:
        nbytes = int(max(nbytes, 256))
        key = (torch.cuda.current_device(), stream_handle())
        with self._lock:
            buf = self._bufs.get(key)
            if buf is None or buf.numel() < nbytes:
                grow = max(nbytes, int(buf.numel() * 1.25) if buf is not None else 0)
                buf = torch.empty(grow, dtype=torch.uint8, device=device())
                self._bufs[key] = buf
            return buf.data_ptr(), buf.numel()

    def release(self):
        with self._lock:
            self._bufs.clear()


WORKSPACE = _WorkspacePool()


# ----------------------------------------------------------- device matrix --
@dataclass
class DMat:
    """A validated, C-contiguous float64 device matrix (row-major m x n).

    frob2 is ||A||_F^2 from the validation pass (src/solvers.py:102 needs it);
    kind records whether the caller handed us numpy ("numpy") or torch ("torch")
    so results can be returned in the same kind.
    """

    t: torch.Tensor
    frob2: float | None = None
    kind: str = "numpy"
    colstats: torch.Tensor | None = None   # column max|A| and sum A^2 (2n), set by the pipeline for the INT8 Gram

    @property
    def shape(self):
        return tuple(self.t.shape)

    @property
    def ptr(self) -> int:
        return self.t.data_ptr()

    @property
    def ld(self) -> int:
        return self.t.stride(0)


def _host_matrix_checks(a, name):
    """The shape/dtype half of src/dense.py:57-65 for numpy input."""
    arr = np.asarray(a)
    if arr.ndim != 2:
        raise ValueError(f"{name} must be 2-D, got ndim={arr.ndim}")
    if arr.dtype not in _FLOAT_NP:
        arr = arr.astype(np.float64)
    return np.ascontiguousarray(arr)


def as_dmat(a, name: str = "a") -> DMat:
    """_as_matrix + astype(float64) on the device (src/dense.py:57-65).

    Accepts numpy arrays (any dtype; non-float is cast to float64 like the
    reference) or torch tensors (CPU or CUDA).  Non-finite entries raise
    ValueError.  One streaming pass validates, promotes and measures ||A||_F^2.
    """
    if isinstance(a, DMat):
        return a
    dev = device()
    if isinstance(a, torch.Tensor):
        kind = "torch"
        if a.dim() != 2:
            raise ValueError(f"{name} must be 2-D, got ndim={a.dim()}")
        src = a if a.dtype in _TORCH_CODE else a.to(torch.float64)
        src = src.to(dev, non_blocking=True).contiguous()
    else:
        kind = "numpy"
        arr = _host_matrix_checks(a, name)
        src = torch.from_numpy(arr).to(dev, non_blocking=False)
    m, n = src.shape
    if n == 0 or m == 0:
        out = src.to(torch.float64)
        return DMat(out, 0.0, kind)
    if src.dtype == torch.float64:
        out = src if src.is_contiguous() else src.contiguous()
        dst_ptr = 0   # validate in place, no copy
    else:
        out = torch.empty((m, n), dtype=torch.float64, device=dev)
        dst_ptr = out.data_ptr()
    stats = (C.c_double * 2)()
    lib = _lib.lib()
    wsb = lib.sk_matrix_stats_workspace(m, n)
    wp, wn = WORKSPACE.get(wsb)
    call("sk_cast_stats", src.data_ptr(), _TORCH_CODE[src.dtype], m, n, src.stride(0),
         dst_ptr if dst_ptr else None, n, stats, wp, wn, stream_handle())
    if stats[0] > 0:
        raise ValueError(f"{name} contains non-finite entries")
    return DMat(out, float(stats[1]), kind)


def as_dvec(b, length: int | None = None) -> torch.Tensor:
    """np.asarray(b, dtype=float64) on the device; 1-D check (src/solvers.py:87-96)."""
    dev = device()
    if isinstance(b, torch.Tensor):
        t = b.to(dev, dtype=torch.float64, non_blocking=True)
    else:
        arr = np.asarray(b, dtype=np.float64)
        t = torch.from_numpy(np.ascontiguousarray(arr)).to(dev)
    if t.dim() != 1:
        raise ValueError(f"b must be 1-D, got ndim={t.dim()}")
    if length is not None and t.shape[0] != length:
        raise DimensionMismatch(f"b length {t.shape[0]} != rows {length}")
    return t.contiguous()


def to_host(t: torch.Tensor) -> np.ndarray:
    return t.detach().contiguous().to("cpu").numpy()


def like_input(t: torch.Tensor, kind: str):
    return to_host(t) if kind == "numpy" else t


def nan_to_none(x):
    return None if x is None or (isinstance(x, float) and math.isnan(x)) else x
