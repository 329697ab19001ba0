"""ctypes binding of the in-tree C-ABI library `libsklsq.so` (include/sklsq.h).

The library is the product: there is no CPU or eager-PyTorch fallback.  If the
shared object is missing or no CUDA device is present, `lib()` raises.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsklsq.so")

SK_OK = 0
CODES = {
    1: "RankDeficient", 2: "SingularTriangular", 3: "NumericallySingular",
    4: "NotPositiveDefinite", 5: "Overflow", 6: "DimensionMismatch", 7: "NoConvergence",
    8: "NotSymmetric", 9: "NonFinite", -1: "CudaError", -2: "BadArgument",
}
LEVEL_CODE = {"binary16": 16, "binary32": 32, "binary64": 64}
TRANSFORM_CODE = {"dct2": 0, "wht": 1}
DTYPE_CODE = {"float16": 2, "float32": 4, "float64": 8}


class SkStatus(C.Structure):
    _fields_ = [("code", C.c_int32), ("pad", C.c_int32), ("index", C.c_int64),
                ("value", C.c_double), ("aux", C.c_double)]


_p, _i64, _i32, _sz, _d = C.c_void_p, C.c_int64, C.c_int, C.c_size_t, C.c_double
_pd = C.POINTER(C.c_double)
_pi = C.POINTER(C.c_int)
_ps = C.POINTER(SkStatus)

# name -> (restype, argtypes); mirrors include/sklsq.h one for one.
SIGNATURES = {
    "sk_version": (_i32, []),
    "sk_last_error": (C.c_char_p, []),
    "sk_sm_count": (_i32, [_i32]),
    "sk_launch_count": (C.c_uint64, []),
    "sk_matrix_stats_workspace": (_sz, [_i64, _i64]),
    "sk_cast_stats": (_i32, [_p, _i32, _i64, _i64, _i64, _p, _i64, _pd, _p, _sz, _p]),
    "sk_cast_stats_async": (_i32, [_p, _i32, _i64, _i64, _i64, _p, _i64, _p, _p, _sz, _p]),
    "sk_level_overflow": (_i32, [_p, _i64, _i64, _i64, _i32, _pi, _p, _sz, _p]),
    "sk_residual": (_i32, [_p, _i64, _i64, _i64, _p, _p, _p, _pd, _p, _sz, _p]),
    "sk_residual_async": (_i32, [_p, _i64, _i64, _i64, _p, _p, _p, _p, _p, _sz, _p]),
    "sk_defer_verdicts": (_i32, [_p]),
    "sk_note_flag": (_i32, [_p, _i32, _p]),
    "sk_note_positive": (_i32, [_p, _i32, _p]),
    "sk_note_zero_diagonal": (_i32, [_p, _i64, _i64, _i32, _p]),
    "sk_guard_identity": (_i32, [_i32, _p, _i64, _i64, _i64, _i32, _p]),
    "sk_gram_workspace": (_sz, [_i64, _i64]),
    "sk_gram_f64": (_i32, [_p, _i64, _p, _i64, _i64, _i64, _p, _i64, _i32, _p, _sz, _p]),
    "sk_gram_ozaki_workspace": (_sz, [_i64, _i64, _i32]),
    "sk_gram_ozaki_f64": (_i32, [_p, _i64, _p, _i64, _i64, _i64, _p, _i64, _p, _sz, _p]),
    "sk_gram_ozaki_ex_f64": (_i32, [_p, _i64, _p, _i64, _i64, _i64, _p, _p, _p, _i64, _p, _sz, _p]),
    "sk_gram_ozaki_acc_f64": (_i32, [_p, _i64, _p, _i64, _i64, _i64, _p, _p, _p, _i64, _i32, _p, _sz, _p]),
    "sk_gram_ozaki_fell_back": (_i32, []),
    "sk_colstats_workspace": (_sz, [_i64]),
    "sk_colstats_f64": (_i32, [_p, _i64, _i64, _i64, _p, _p, _p, _sz, _p]),
    "sk_gemv_t_workspace": (_sz, [_i64, _i64]),
    "sk_gemv_t_f64": (_i32, [_p, _i64, _i64, _i64, _p, _p, _i32, _p, _sz, _p]),
    "sk_trsm_right_upper_f64": (_i32, [_p, _i64, _i64, _i64, _p, _i64, _p, _i64, _ps, _p]),
    "sk_trsm_ozaki_workspace": (_sz, [_i64, _i64]),
    "sk_trsm_ozaki_f64": (_i32, [_p, _i64, _i64, _i64, _p, _i64, _p, _i64, _ps, _p, _sz, _p]),
    "sk_trsm_ozaki_fell_back": (_i32, []),
    "sk_sketch_workspace": (_sz, [_i32, _i64, _i64, _i64]),
    "sk_sketch_workspace_ex": (_sz, [_i32, _i32, _i64, _i64, _i64, _i64]),
    "sk_sketch_partial": (_i32, [_i32, _i32, _p, _i64, _i64, _i64, _i64, _i64, _p, _p, _i64,
                                 _p, _i64, _i32, _p, _p, _sz, _p]),
    "sk_sketch_partial_ex": (_i32, [_i32, _i32, _p, _i64, _i64, _i64, _i64, _i64, _p, _p, _i64,
                                    _p, _i64, _i32, _p, _p, _sz, _p, _i32]),
    "sk_sketch_signs": (_i32, [C.c_uint64, C.c_uint64, _i64, _p, _p]),
    "sk_sketch_finalize": (_i32, [_i32, _p, _i64, _i64, _i64, _i64, _p, _p, _p]),
    "sk_qr_workspace": (_sz, [_i32, _i64, _i64]),
    "sk_qr_r": (_i32, [_i32, _p, _i64, _i64, _p, _i64, _ps, _p, _sz, _p]),
    "sk_qr_factors_workspace": (_sz, [_i32, _i64, _i64]),
    "sk_qr_in_precision_f64": (_i32, [_i32, _p, _i64, _i64, _i64, _p, _i64, _p, _i64, _ps, _p, _sz, _p]),
    "sk_householder_f64": (_i32, [_p, _i64, _i64, _i64, _p, _i64, _p, _i64, _p, _ps, _p, _sz, _p]),
    "sk_accumulate_q": (_i32, [_i32, _p, _i64, _p, _i64, _i64, _p, _i64, _p]),
    "sk_nxn_workspace": (_sz, [_i64]),
    "sk_chol_solve_f64": (_i32, [_p, _i64, _p, _p, _ps, _p, _sz, _p]),
    "sk_gram_check": (_i32, [_p, _i64, _pd, _p, _sz, _p]),
    "sk_chol_factor_f64": (_i32, [_p, _i64, _p, _ps, _p, _sz, _p]),
    "sk_lu_solve_f64": (_i32, [_p, _i64, _p, _p, _ps, _p, _sz, _p]),
    "sk_trsv_f64": (_i32, [_p, _i64, _i64, _i32, _p, _p, _ps, _p, _sz, _p]),
    "sk_kappa0_from_gram": (_i32, [_p, _i64, _pd, _pi, _p, _sz, _p]),
    "sk_jacobi_workspace": (_sz, [_i64, _i64]),
    "sk_jacobi_sv_f64": (_i32, [_p, _i64, _i64, _i64, _i32, _d, _pd, _p, _sz, _p]),
    "sk_gemm_tn_workspace": (_sz, [_i64, _i64]),
    "sk_gemm_tn_f64": (_i32, [_p, _i64, _p, _i64, _i64, _i64, _p, _p, _i64, _p, _p, _sz, _p]),
    "sk_syrk_f64": (_i32, [_p, _i64, _i64, _i64, _p, _i64, _p, _sz, _p]),
    "sk_kappa0_workspace": (_sz, [_i64, _i64]),
    "sk_kappa0_f64": (_i32, [_p, _i64, _i64, _i64, _pd, _pi, _p, _sz, _p]),
    "sk_sketch": (_i32, [_i32, _i32, _p, _i64, _i64, _i64, _i64, _i64, _p, _p, _i64, _p, _i64, _p, _p, _sz, _p]),
    "sk_demote_check": (_i32, [_p, _i64, _i64, _i64, _i32, _pi, _p, _sz, _p]),
    "sk_residual_norms": (_i32, [_p, _i64, _i64, _i64, _p, _p, _p, _pd, _p, _sz, _p]),
}

_LOCK = threading.Lock()
_LIB = None


class LibraryUnavailable(RuntimeError):
    """libsklsq.so is not built or no CUDA device is visible (no fallback exists)."""


def load(require_device: bool = True):
    """Load and bind libsklsq.so.  Raises LibraryUnavailable loudly."""
    global _LIB
    with _LOCK:
        if _LIB is None:
            if not os.path.exists(LIB_PATH):
                raise LibraryUnavailable(
                    f"{LIB_PATH} is missing: build it with `make` or __graft_entry__.build(); "
                    "this package has no CPU fallback")
            lib = C.CDLL(LIB_PATH)
            missing = []
            for name, (res, args) in SIGNATURES.items():
                try:
                    fn = getattr(lib, name)
                except AttributeError:
                    missing.append(name)
                    continue
                fn.restype = res
                fn.argtypes = args
            lib.sk_missing_symbols = missing
            _LIB = lib
    if require_device:
        import torch
        if not torch.cuda.is_available():
            raise LibraryUnavailable("no CUDA device: the sketchlsq B200 path has no CPU fallback")
    return _LIB


def lib():
    return load(True)


def last_error() -> str:
    return (load(False).sk_last_error() or b"").decode(errors="replace")
