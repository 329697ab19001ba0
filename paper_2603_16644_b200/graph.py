"""Algorithm 1 for a fixed shape as ONE CUDA graph (latency-bound sizes).

`algorithm1_pipeline` (src/solvers.py:282-324) raises the reference's exceptions where
the reference does, so the eager path reads every numerical verdict on the host: the
finiteness scan, the sketch's demotion overflow, the level QR's collapse, the zero
diagonal of R_s, the TRSM's zero pivot, the Cholesky / LU pivots, then the residual
norms -- about seven stream synchronisations and ~25 ctypes calls per solve.  At
config-1 size (1000 x 100) the kernels take a fraction of that time.

`PipelinePlan` runs the same C-ABI sequence with the verdicts deferred
(`sk_defer_verdicts`, include/sklsq.h): every check stores its SK_* code into one
device status record (first failure in stream order wins) and the data-dependent
kernels after a recorded failure run on the identity.  The whole solve -- validation,
sketch, level QR, TRSM, Gram + A_p^T b on two streams, Cholesky / LU, TRSV, residual
and the device->host copy of (status, norms, x) -- is captured once per precision
level and replayed per call; the host reads the record once.  Any recorded failure
re-runs the eager `algorithm1_pipeline` on the same inputs, which raises exactly the
reference's exception (or escalates binary16 -> binary32 on RankDeficient, or falls
back from Cholesky to LU on NotPositiveDefinite, src/solvers.py:227-231, 255-279), so
a plan's results equal the eager call's bit for bit in every case.

The plan owns every buffer (inputs, sketch operator, A_s, R_s, A_p, G, workspaces), so
nothing it captured can be reallocated underneath the graph.  It covers the engines
of every engine the eager pipeline picks: the FFT / DMMA / tcgen05 sketches, the FP64
DMMA or INT8 Ozaki-II TRSM and Gram (whose operand guards, which choose the DMMA
fallback, stay on the device: the fallback kernels run gated on the guard flag).  The
solve's A_p is held in full (the eager pipeline's row-chunked TRSM -> Gram for A_p that
does not fit beside A is not captured).  Not in the reference's API: an addition for serving many small solves.
"""

from __future__ import annotations

import math
import time

import numpy as np
import torch

from . import _lib
from .device import device
from .errors import DeviceError
from .precision import PrecisionDecision, PrecisionLevel, level_from_name, select_precision
from .sketch import DCT2, WHT, _make_sketch_dev

SK_RANK_DEFICIENT, SK_SINGULAR_TRIANGULAR, SK_OVERFLOW, SK_NON_FINITE = 1, 2, 5, 9
_HEAD = 8          # doubles before x in the result record: status (4), ||A||_F stats (2), residual norms (2)


def _c(rc: int, what: str):
    if rc != 0:
        raise DeviceError(f"{what}: libsklsq error {rc}: {_lib.last_error()}")


class _LevelGraph:
    """Buffers and the captured graph of one precision level."""

    def __init__(self, plan: "PipelinePlan", level: PrecisionLevel):
        from .dense import _gram_engine, _new_ap, _trsm_engine
        lib = _lib.lib()
        m, n, d = plan.m, plan.n, plan.d
        dev = plan.dev
        self.level = level
        self.op, self.dsk = _make_sketch_dev(m, d, plan.transform, plan.seed)
        self.total = torch.zeros((n, d), dtype=torch.float64, device=dev)
        self.flag = torch.zeros(1, dtype=torch.int32, device=dev)
        self.a_s = torch.empty((n, d), dtype=level.torch_dtype, device=dev)
        self.r = torch.empty((n, n), dtype=torch.float64, device=dev)
        self.ap = _new_ap(m, n, dev)
        self.g = torch.empty((n, n), dtype=torch.float64, device=dev)
        self.rhs = torch.empty(n, dtype=torch.float64, device=dev)
        self.y = torch.empty(n, dtype=torch.float64, device=dev)
        # the engines the eager pipeline picks for this shape (INT8 Ozaki Gram with A_p^T b
        # from the column scan, INT8 Ozaki TRSM; their fallbacks gated on device flags that
        # sit 256 bytes past their workspaces under deferred verdicts)
        self.gram_oz = _gram_engine(m, n, False, None) == "ozaki"
        self.trsm_oz = _trsm_engine(m, n, False, None) == "ozaki"
        self.st = torch.empty(3 * n, dtype=torch.float64, device=dev)   # column max, sum of squares, A_p^T b
        tc = _lib.TRANSFORM_CODE[plan.transform]
        sizes = [lib.sk_matrix_stats_workspace(m, n), lib.sk_sketch_workspace_ex(level.code, tc, m, self.op.m_pad, n, d),
                 lib.sk_qr_workspace(level.code, d, n), lib.sk_gram_workspace(m, n), lib.sk_nxn_workspace(n),
                 2 * 8 * n + 1024, lib.sk_colstats_workspace(n)]
        if self.gram_oz:
            syrk = plan.method == "pne"
            sizes.append(max(lib.sk_gram_ozaki_workspace(m, n, int(syrk)), lib.sk_gram_workspace(m, n)) + 256)
        if self.trsm_oz:
            sizes.append(lib.sk_trsm_ozaki_workspace(m, n) + 256)
        ws = max(sizes)
        self.ws = torch.empty(int(ws) + 256, dtype=torch.uint8, device=dev)
        self.ws_side = torch.empty(int(lib.sk_gemv_t_workspace(m, n)) + 256, dtype=torch.uint8, device=dev)
        self.side = torch.cuda.Stream(device=dev)
        self.graph = None
        # one untimed pass with verdicts deferred (sets kernel attributes, creates the QR
        # lookahead stream, touches every buffer), then the capture
        with torch.cuda.stream(plan.stream):
            self._run(plan)
        plan.stream.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=plan.stream, capture_error_mode="thread_local"):
            self._run(plan)
        self.graph = g

    def _run(self, plan: "PipelinePlan"):
        lib = _lib.lib()
        m, n, d = plan.m, plan.n, plan.d
        st = torch.cuda.current_stream().cuda_stream
        a, b, out = plan.a.data_ptr(), plan.b.data_ptr(), plan.out.data_ptr()
        status, stats, res, x = out, out + 32, out + 48, out + 8 * _HEAD
        ws, wn = self.ws.data_ptr(), self.ws.numel()
        lv = self.level.code
        plan.out[:6].zero_()
        self.total.zero_()
        self.flag.zero_()
        _c(lib.sk_defer_verdicts(status), "sk_defer_verdicts")
        try:
            # src/dense.py:57-65: finiteness of A (ValueError) and ||A||_F^2 for the report
            _c(lib.sk_cast_stats_async(a, 8, m, n, n, None, n, stats, ws, wn, st), "sk_cast_stats_async")
            _c(lib.sk_note_positive(stats, SK_NON_FINITE, st), "sk_note_positive")
            # src/solvers.py:185-199: sketch at the level (Overflow), level QR, zero diagonal
            _c(lib.sk_sketch_partial_ex(lv, _lib.TRANSFORM_CODE[plan.transform], a, n, m, 0, self.op.m_pad, n,
                                        self.dsk.signs.data_ptr(), self.dsk.rows.data_ptr(), d,
                                        self.total.data_ptr(), d, 0, self.flag.data_ptr(), ws, wn, st, 0),
               "sk_sketch_partial_ex")
            _c(lib.sk_note_flag(self.flag.data_ptr(), SK_OVERFLOW, st), "sk_note_flag")
            _c(lib.sk_sketch_finalize(lv, self.total.data_ptr(), d, d, n, self.op.m_pad, self.a_s.data_ptr(),
                                      None, st), "sk_sketch_finalize")
            _c(lib.sk_guard_identity(self.a_s.element_size(), self.a_s.data_ptr(), d, n, d, 1, st),
               "sk_guard_identity")
            _c(lib.sk_qr_r(lv, self.a_s.data_ptr(), d, n, self.r.data_ptr(), n, None, ws, wn, st), "sk_qr_r")
            _c(lib.sk_note_zero_diagonal(self.r.data_ptr(), n, n, SK_RANK_DEFICIENT, st), "sk_note_zero_diagonal")
            # src/solvers.py:205-215: A_p = A R_s^-1
            ap, ldap = self.ap.data_ptr(), self.ap.stride(0)
            if self.trsm_oz:
                _c(lib.sk_trsm_ozaki_f64(a, n, m, n, self.r.data_ptr(), n, ap, ldap, None, ws, wn, st),
                   "sk_trsm_ozaki_f64")
            else:
                _c(lib.sk_trsm_right_upper_f64(a, n, m, n, self.r.data_ptr(), n, ap, ldap, None, st), "sk_trsm")
            yp, ldy = (ap, ldap) if plan.method == "pne" else (a, n)
            if self.gram_oz:
                # src/solvers.py:218-252 on the INT8 engine: one column scan of A_p gives its
                # scales and A_p^T b (solvers._gram_and_rhs), then the Ozaki-II product
                stp = self.st.data_ptr()
                _c(lib.sk_colstats_f64(ap, ldap, m, n, b, stp, ws, wn, st), "sk_colstats_f64")
                _c(lib.sk_gram_ozaki_acc_f64(ap, ldap, yp, ldy, m, n, stp, stp if plan.method == "pne" else None,
                                             self.g.data_ptr(), n, 0, ws, wn, st), "sk_gram_ozaki_acc_f64")
                rhs = stp + 16 * n
            else:
                # A_p^T b on a second stream under the DMMA Gram
                cur = torch.cuda.current_stream()
                self.side.wait_stream(cur)
                with torch.cuda.stream(self.side):
                    _c(lib.sk_gemv_t_f64(ap, ldap, m, n, b, self.rhs.data_ptr(), 0, self.ws_side.data_ptr(),
                                         self.ws_side.numel(), self.side.cuda_stream), "sk_gemv_t_f64")
                _c(lib.sk_gram_f64(ap, ldap, yp, ldy, m, n, self.g.data_ptr(), n, 0, ws, wn, st), "sk_gram_f64")
                cur.wait_stream(self.side)
                rhs = self.rhs.data_ptr()
            if plan.method == "pne":
                _c(lib.sk_chol_solve_f64(self.g.data_ptr(), n, rhs, self.y.data_ptr(), None, ws, wn, st),
                   "sk_chol_solve_f64")
                _c(lib.sk_trsv_f64(self.r.data_ptr(), n, n, 0, self.y.data_ptr(), x, None, ws, wn, st), "sk_trsv_f64")
            else:
                _c(lib.sk_lu_solve_f64(self.g.data_ptr(), n, rhs, x, None, ws, wn, st), "sk_lu_solve_f64")
            # src/solvers.py:99-117: ||A x - b||^2 and ||x||^2
            _c(lib.sk_residual_async(a, m, n, n, x, b, None, res, ws, wn, st), "sk_residual_async")
        finally:
            lib.sk_defer_verdicts(None)
        plan.out_h.copy_(plan.out, non_blocking=True)


class PipelinePlan:
    """algorithm1_pipeline(a, b, method, precision, d_factor, transform, seed,
    diagnostics=False) for m x n inputs, replayed as one CUDA graph per level.

        plan = PipelinePlan(1000, 100, method="hpne", precision="single")
        rep = plan.solve(a, b, x_star)        # numpy or torch (host or device) inputs

    `plan.a` / `plan.b` are the graph's input buffers: a caller that fills them in place
    (e.g. a serving loop producing A on the device) can call `plan.solve()` with no
    arguments and skip the copy.  precision="auto" estimates kappa0 eagerly (the
    reference's estimator, one host read) and replays the chosen level's graph.
    """

    def __init__(self, m: int, n: int, method: str = "pne", precision="auto", d_factor: float = 3.0,
                 transform: str = DCT2, seed: int = 0):
        if method not in ("pne", "hpne"):
            raise ValueError(f"pipeline method must be pne or hpne, got {method!r}")
        if not isinstance(precision, PrecisionLevel) and precision != "auto":
            precision = level_from_name(precision)
        if transform not in (DCT2, WHT):
            raise ValueError(f"unknown transform {transform!r}")
        if m < n or n < 1:
            raise ValueError(f"PipelinePlan needs m >= n >= 1, got {m} x {n}")
        self.m, self.n, self.method, self.precision = int(m), int(n), method, precision
        self.d_factor, self.transform, self.seed = float(d_factor), transform, int(seed)
        self.d = int(math.ceil(d_factor * n))
        if self.d < n:
            raise ValueError(f"d_factor {d_factor} gives d={self.d} < n={n}")
        self.dev = device()
        self.a = torch.empty((m, n), dtype=torch.float64, device=self.dev)
        self.b = torch.empty(m, dtype=torch.float64, device=self.dev)
        self.out = torch.zeros(_HEAD + n, dtype=torch.float64, device=self.dev)
        self.out_h = torch.empty(_HEAD + n, dtype=torch.float64, pin_memory=True)
        self.stream = torch.cuda.Stream(device=self.dev)
        self._graphs: dict = {}
        if isinstance(precision, PrecisionLevel):
            self._level_graph(precision)

    def _level_graph(self, level: PrecisionLevel) -> _LevelGraph:
        lg = self._graphs.get(level.name)
        if lg is None:
            lg = self._graphs[level.name] = _LevelGraph(self, level)
        return lg

    def _load(self, a, b):
        if a is not None:
            src = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
            if tuple(src.shape) != (self.m, self.n):
                raise ValueError(f"plan is for {self.m} x {self.n}, got a of shape {tuple(src.shape)}")
            self.a.copy_(src, non_blocking=True)
        if b is not None:
            src = b if isinstance(b, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(b, dtype=np.float64))
            if src.dim() != 1:
                raise ValueError(f"b must be 1-D, got ndim={src.dim()}")
            if src.shape[0] != self.m:
                from .errors import DimensionMismatch
                raise DimensionMismatch(f"b length {src.shape[0]} != rows {self.m}")
            self.b.copy_(src, non_blocking=True)

    def solve(self, a=None, b=None, x_star=None):
        """One solve; returns the SolveReport algorithm1_pipeline(..., diagnostics=False)
        returns (stage_ms empty), or raises what it raises."""
        from .solvers import Preconditioner, SolveReport, algorithm1_pipeline
        t0 = time.perf_counter()
        self._load(a, b)
        decision, frob2 = None, None
        if isinstance(self.precision, PrecisionLevel):
            level = self.precision
        else:
            try:
                decision, frob2 = self._decide()
            except Exception:   # noqa: BLE001 -- e.g. non-finite A: the eager call raises the reference's error
                decision = None
            if decision is None:
                return algorithm1_pipeline(self.a, self.b, self.method, self.precision, self.d_factor,
                                           self.transform, self.seed, x_star, diagnostics=False)
            level = decision.selected
        lg = self._level_graph(level)
        cur = torch.cuda.current_stream()
        self.stream.wait_stream(cur)          # the input copies
        with torch.cuda.stream(self.stream):  # replay() launches on the current stream
            lg.graph.replay()
        self.stream.synchronize()
        head = self.out_h[:_HEAD].numpy()
        code = int(np.frombuffer(head[:1].tobytes(), dtype=np.int32)[0])
        if code != 0:   # the eager pipeline raises / escalates / falls back exactly as the reference
            rep = algorithm1_pipeline(self.a, self.b, self.method, self.precision, self.d_factor, self.transform,
                                      self.seed, x_star, diagnostics=False)
            rep.wall_ms = (time.perf_counter() - t0) * 1e3
            return rep
        x_hat = self.out_h[_HEAD:].numpy().copy()
        res2, x2 = float(head[6]), float(head[7])
        if frob2 is None:
            frob2 = float(head[5])
        residual_norm = math.sqrt(res2)
        denom = math.sqrt(frob2) * math.sqrt(x2)
        rel_err = None
        if x_star is not None:
            xs = np.asarray(x_star.detach().cpu() if isinstance(x_star, torch.Tensor) else x_star, dtype=np.float64)
            rel_err = float(np.linalg.norm(x_hat - xs) / np.linalg.norm(xs))
        with torch.cuda.stream(self.stream):
            r_s = lg.r.clone()
        cur.wait_stream(self.stream)
        pre = Preconditioner(r_s=r_s, computed_in=level, kappa_rs=math.nan, kappa_ap=math.nan,
                             sketch_descriptor=lg.op.descriptor())
        return SolveReport(method=self.method, x_hat=x_hat, residual_norm=residual_norm,
                           relative_residual=residual_norm / denom if denom > 0 else math.inf,
                           relative_error=rel_err, wall_ms=(time.perf_counter() - t0) * 1e3, preconditioner=pre,
                           precision_decision=decision)

    def _decide(self):
        """kappa0 exactly as algorithm1_pipeline does for device-resident A under "auto":
        the Gram doubles as the validation pass and its trace is ||A||_F^2.  Returns
        (decision, ||A||_F^2), or (None, None) for a non-finite A."""
        import ctypes as C
        from .dense import _colstats, _gram, _gram_engine
        from .device import WORKSPACE, DMat, call, stream_handle
        from .precision import _kappa0_from_gram
        cm = _colstats(self.a) if _gram_engine(self.m, self.n, False, None) == "ozaki" else None
        g = _gram(DMat(self.a, None, "torch", cm))
        chk = (C.c_double * 2)()
        wp, wn = WORKSPACE.get(256)
        call("sk_gram_check", g.data_ptr(), self.n, chk, wp, wn, stream_handle())
        if chk[0] > 0:
            return None, None
        k0, over = _kappa0_from_gram(g)
        return PrecisionDecision(kappa0=k0, selected=select_precision(k0, over), overflowed=over), float(chk[1])
