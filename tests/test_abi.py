"""CPU checks of the C-ABI boundary: the library builds, loads and exports every
symbol include/sklsq.h declares (no compute calls: no GPU here)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sklsq.h")
LIB = os.path.join(ROOT, "paper_2603_16644_b200", "libsklsq.so")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sk_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_hot_path():
    syms = declared_symbols()
    for must in ("sk_gram_f64", "sk_trsm_right_upper_f64", "sk_sketch_partial", "sk_qr_r",
                 "sk_chol_solve_f64", "sk_lu_solve_f64", "sk_trsv_f64", "sk_kappa0_from_gram",
                 "sk_residual", "sk_cast_stats", "sk_jacobi_sv_f64"):
        assert must in syms


def test_library_exports_every_declared_symbol():
    if not os.path.exists(LIB):
        pytest.skip("libsklsq.so not built (run make / __graft_entry__.build())")
    lib = ctypes.CDLL(LIB)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_python_binding_table_matches_header():
    from paper_2603_16644_b200 import _lib
    assert sorted(_lib.SIGNATURES) == declared_symbols()


def test_library_metadata_calls_without_gpu():
    if not os.path.exists(LIB):
        pytest.skip("libsklsq.so not built")
    from paper_2603_16644_b200 import _lib
    lib = _lib.load(require_device=False)
    assert lib.sk_version() == 1
    assert isinstance(_lib.last_error(), str)
    # workspace queries are pure host arithmetic
    assert lib.sk_nxn_workspace(64) > 0
    assert lib.sk_qr_workspace(16, 600, 40) > 0
    assert lib.sk_jacobi_workspace(40, 40) >= 40 * 40 * 8


def test_product_path_fails_loudly_without_device(monkeypatch):
    import torch
    from paper_2603_16644_b200 import _lib
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(_lib.LibraryUnavailable):
        _lib.lib()
    import numpy as np
    import paper_2603_16644_b200 as sq
    with pytest.raises(_lib.LibraryUnavailable):
        sq.algorithm1_pipeline(np.eye(4, 2), np.ones(4))


def test_deferred_verdict_entry_points_refuse_without_a_record():
    """sk_note_* / sk_guard_identity need sk_defer_verdicts first: without a device
    status record they fail loudly (SK_ERR_ARG) before touching any device memory."""
    if not os.path.exists(LIB):
        pytest.skip("libsklsq.so not built")
    lib = ctypes.CDLL(LIB)
    lib.sk_last_error.restype = ctypes.c_char_p
    lib.sk_defer_verdicts(None)
    assert lib.sk_note_flag(ctypes.c_void_p(1), ctypes.c_int(5), None) == -2
    assert lib.sk_note_positive(ctypes.c_void_p(1), ctypes.c_int(9), None) == -2
    assert lib.sk_note_zero_diagonal(ctypes.c_void_p(1), ctypes.c_int64(4), ctypes.c_int64(4), ctypes.c_int(1),
                                     None) == -2
    assert lib.sk_guard_identity(8, ctypes.c_void_p(1), ctypes.c_int64(4), ctypes.c_int64(4), ctypes.c_int64(4), 1,
                                 None) == -2
    assert b"sk_defer_verdicts" in lib.sk_last_error()


def test_pipeline_plan_validates_before_touching_the_device():
    """PipelinePlan checks its arguments like algorithm1_pipeline (ValueError) before it
    needs a GPU; with no GPU the product path fails loudly (no CPU fallback)."""
    import paper_2603_16644_b200 as sq
    from paper_2603_16644_b200 import _lib
    with pytest.raises(ValueError):
        sq.PipelinePlan(100, 10, method="sne")
    with pytest.raises(ValueError):
        sq.PipelinePlan(100, 10, precision="quad")
    with pytest.raises(ValueError):
        sq.PipelinePlan(5, 10)
    with pytest.raises(ValueError):
        sq.PipelinePlan(100, 10, d_factor=0.5)
    import torch
    if not torch.cuda.is_available():
        with pytest.raises(_lib.LibraryUnavailable):
            sq.PipelinePlan(100, 10, method="hpne", precision="single")
