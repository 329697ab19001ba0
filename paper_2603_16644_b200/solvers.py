"""Least-squares solvers: PNE / HPNE / NE / SNE / NNE / QR and Algorithm 1.

Same entry points, signatures, dataclasses and error behaviour as the reference
(src/solvers.py).  Every m x n pass runs in libsklsq on the device:

  check      sk_cast_stats                (validation + f64 + ||A||_F^2, one pass)
  kappa0     sk_gram_ozaki_ex_f64 (INT8 SYRK; sk_gram_f64 DMMA below 2^33 m n^2)
             + sk_kappa0_from_gram
  sketch     sk_sketch_partial/finalize   (on-the-fly SRTT operator, level demotion fused)
  level QR   sk_qr_r                      (binary16 op-for-op emulation)
  A_p        sk_trsm_ozaki_f64            (DMMA leaves + INT8 updates; sk_trsm_right_upper_f64
                                           DMMA for small solves)
  Gram       sk_gram_ozaki_ex_f64 / sk_gram_f64 (SYRK for PNE, GEMM-TN for HPNE/NNE),
             A_p^T b from sk_colstats_f64's column scan (or sk_gemv_t_f64)
  n x n      sk_chol_solve_f64 / sk_lu_solve_f64 / sk_trsv_f64
  report     sk_residual

Inputs may be numpy arrays (the reference's convention) or torch tensors (CPU
or CUDA; a CUDA tensor avoids the host->device copy).  x_hat is returned as a
numpy array like the reference; A_p from precondition_matrix follows the input
kind (numpy in -> numpy out, torch in -> CUDA tensor out).

Diagnostics: the reference always fills Preconditioner.kappa_rs / kappa_ap with
one-sided Jacobi (src/solvers.py:200, :214).  Here they run on the device too
(sk_jacobi_sv_f64; kappa_ap via the R factor of A_p) and are on by default for
API parity; pass diagnostics=False to skip them (they are not part of
Algorithm 1 and are excluded from the bench's solve time).  With
strict_diagnostics=False (default) a Jacobi NoConvergence is recorded as NaN
instead of aborting the solve; strict_diagnostics=True raises
like the reference.
"""

from __future__ import annotations

import math
import threading
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from .dense import (_chol_solve, _diagnostics_dev, _gemv_t, _gram, _householder_r64, _lu_solve, _trsm, _trsv)
from .device import DMat, as_dmat, as_dvec, call, like_input, stream_handle, to_host, WORKSPACE
from .errors import DimensionMismatch, NoConvergence, NotPositiveDefinite, RankDeficient
from .precision import (BINARY64, PrecisionDecision, PrecisionLevel, _decide_dev, _qr_level_dev,
                        level_from_name, next_higher)
from .sketch import DCT2, DeviceSketch, _apply_dev, _make_sketch_dev, make_sketch
from . import _lib

import ctypes as C


class Preconditioner:
    """src/solvers.py:47-59: the promoted binary64 factor and its diagnostics.

    Same fields as the reference dataclass.  r_s may be given as a numpy array or
    a CUDA tensor; the device copy stays resident for the solve and the numpy view
    (`.r_s`) is materialised lazily on first access, so the pipeline never pays
    an n x n device->host copy it does not need."""

    def __init__(self, r_s, computed_in, kappa_rs, kappa_ap=None, sketch_descriptor=None):
        if isinstance(r_s, torch.Tensor) and r_s.is_cuda:
            self._r_dev, self._r_host = r_s, None
        else:
            self._r_dev, self._r_host = None, np.asarray(r_s)
        self.computed_in = computed_in
        self.kappa_rs = kappa_rs
        self.kappa_ap = kappa_ap
        self.sketch_descriptor = sketch_descriptor

    @property
    def r_s(self) -> np.ndarray:
        if self._r_host is None:
            self._r_host = to_host(self._r_dev)
        return self._r_host

    @r_s.setter
    def r_s(self, value):
        self._r_dev, self._r_host = None, np.asarray(value)

    def r_device(self) -> torch.Tensor:
        if self._r_dev is None or self._r_dev.device != torch.device("cuda", torch.cuda.current_device()):
            self._r_dev = torch.from_numpy(np.ascontiguousarray(self.r_s, dtype=np.float64)).cuda()
        return self._r_dev

    def __repr__(self):
        return (f"Preconditioner(r_s=<{tuple(self.r_device().shape if self._r_host is None else self._r_host.shape)}>, "
                f"computed_in={self.computed_in!r}, kappa_rs={self.kappa_rs!r}, kappa_ap={self.kappa_ap!r}, "
                f"sketch_descriptor={self.sketch_descriptor!r})")


@dataclass
class SolveReport:
    """src/solvers.py:62-84 (+ stage_ms: per-stage device times, ours)."""

    method: str
    x_hat: np.ndarray
    residual_norm: float
    relative_residual: float
    relative_error: float | None
    wall_ms: float
    preconditioner: Preconditioner | None = None
    bounds: dict = field(default_factory=dict)
    norm_is_frobenius: bool = True
    precision_decision: PrecisionDecision | None = None
    escalated_from: PrecisionLevel | None = None
    stage_ms: dict = field(default_factory=dict)


# ------------------------------------------------------------------ helpers --
class _Stages:
    """CUDA-event stage timer on the current stream (no host sync until read)."""

    def __init__(self, enabled=True):
        self.enabled = enabled
        self.marks = []

    def mark(self, name):
        if self.enabled:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record()
            self.marks.append((name, ev))

    def result(self):
        out = {}
        if len(self.marks) < 2:
            return out
        self.marks[-1][1].synchronize()
        for (name, e0), (_, e1) in zip(self.marks[:-1], self.marks[1:]):
            out[name] = out.get(name, 0.0) + e0.elapsed_time(e1)
        return out


def _host_f64_matrix(a):
    """A 2-D float64 host matrix as a CPU torch tensor (no copy), else None."""
    if isinstance(a, torch.Tensor):
        return a if (not a.is_cuda and a.dim() == 2 and a.dtype == torch.float64 and a.is_contiguous()) else None
    if isinstance(a, np.ndarray) and a.ndim == 2 and a.dtype == np.float64 and a.flags.c_contiguous:
        if not a.flags.writeable:   # e.g. a memory-mapped .npy archive: only ever read here
            import warnings
            with warnings.catch_warnings():
                warnings.simplefilter("ignore", UserWarning)
                return torch.from_numpy(a)
        return torch.from_numpy(a)
    return None


def _check_system(a, b):
    """src/solvers.py:87-96 on the device."""
    ad = as_dmat(a)
    m, n = ad.shape
    if isinstance(b, torch.Tensor):
        if b.dim() != 1:
            raise ValueError(f"b must be 1-D, got ndim={b.dim()}")
    else:
        bn = np.asarray(b, dtype=np.float64)
        if bn.ndim != 1:
            raise ValueError(f"b must be 1-D, got ndim={bn.ndim}")
    if m < n:
        raise DimensionMismatch(f"need rows >= cols, got {ad.shape}")
    bd = b if isinstance(b, torch.Tensor) and b.is_cuda and b.dtype == torch.float64 else None
    if bd is None:
        bd = as_dvec(b)
    if bd.shape[0] != m:
        raise DimensionMismatch(f"b length {bd.shape[0]} != rows {m}")
    return ad, bd.contiguous()


def _report(method, ad: DMat, bd, x_dev, t0, x_star=None, preconditioner=None, stages=None):
    """src/solvers.py:99-117: residual on the device, norms, relative error."""
    m, n = ad.shape
    out = (C.c_double * 2)()
    wp, wn = WORKSPACE.get(_lib.lib().sk_matrix_stats_workspace(m, n))
    call("sk_residual", ad.ptr, m, n, ad.ld, x_dev.data_ptr(), bd.data_ptr(), None, out, wp, wn,
         stream_handle())
    if stages is not None:
        stages.mark("end")
    x_hat = to_host(x_dev)
    residual_norm = float(math.sqrt(out[0]))
    denom = float(math.sqrt(ad.frob2)) * float(math.sqrt(out[1]))
    relative_residual = residual_norm / denom if denom > 0 else math.inf
    relative_error = None
    if x_star is not None:
        xs = np.asarray(x_star.detach().cpu() if isinstance(x_star, torch.Tensor) else x_star, dtype=np.float64)
        relative_error = float(np.linalg.norm(x_hat - xs) / np.linalg.norm(xs))
    return SolveReport(method=method, x_hat=x_hat, residual_norm=residual_norm,
                       relative_residual=relative_residual, relative_error=relative_error,
                       wall_ms=(time.perf_counter() - t0) * 1e3, preconditioner=preconditioner,
                       stage_ms=stages.result() if stages is not None else {})


def _kappa_from_gram(g: torch.Tensor, strict: bool) -> float:
    """kappa(A_p) from the PNE Gram A_p^T A_p (singular values of its Cholesky factor;
    the chunked path has no A_p to factor).  NaN when the Cholesky breaks down."""
    from .dense import _chol_factor, _jacobi_sv
    try:
        sv = _jacobi_sv(_chol_factor(g))
    except NoConvergence:
        if strict:
            raise
        return math.nan
    except NotPositiveDefinite:
        return math.nan
    return float(sv[0] / sv[-1]) if sv[-1] > 0 else float("inf")


def _kappa(at: torch.Tensor, strict: bool) -> float:
    try:
        return _diagnostics_dev(at).two_norm_condition
    except NoConvergence:
        if strict:
            raise
        return math.nan


# ---------------------------------------------------------- baseline solvers --
def solve_qr_baseline(a, b, x_star=None):
    """src/solvers.py:120-126: Householder QR, x = R^{-1} Q^T b.  Q^T b is read
    off the last column of the R factor of [A | b] (the same reflectors applied
    to b), so Q is never formed."""
    ad, bd = _check_system(a, b)
    t0 = time.perf_counter()
    m, n = ad.shape
    aug = torch.cat([ad.t, bd[:, None]], dim=1)
    if m == n:   # a zero row leaves R and Q^T b unchanged and makes room for column n
        aug = torch.cat([aug, torch.zeros((1, n + 1), dtype=aug.dtype, device=aug.device)], dim=0)
    r_aug = _householder_r64(aug)
    r = r_aug[:n, :n].contiguous()
    qtb = r_aug[:n, n].contiguous()
    x = _trsv(r, qtb)
    return _report("qr", ad, bd, x, t0, x_star)


def solve_normal(a, b, x_star=None):
    """src/solvers.py:129-138: Cholesky of A^T A, no fallback."""
    ad, bd = _check_system(a, b)
    t0 = time.perf_counter()
    x = _chol_solve(_gram(ad), _gemv_t(ad, bd))
    return _report("ne", ad, bd, x, t0, x_star)


def solve_seminormal(a, b, x_star=None):
    """src/solvers.py:141-148: R of A, then R^T y = A^T b, R x = y."""
    ad, bd = _check_system(a, b)
    t0 = time.perf_counter()
    r = _householder_r64(ad.t)
    y = _trsv(r, _gemv_t(ad, bd), transposed=True)
    x = _trsv(r, y)
    return _report("sne", ad, bd, x, t0, x_star)


def solve_notnormal(a, b_matrix, b, x_star=None):
    """src/solvers.py:151-165: LU of B^T A."""
    ad, bd = _check_system(a, b)
    bm = as_dmat(b_matrix, "b_matrix")
    if bm.shape != ad.shape:
        raise DimensionMismatch(f"b_matrix shape {bm.shape} != a shape {ad.shape}")
    t0 = time.perf_counter()
    x = _lu_solve(_gram(bm, ad), _gemv_t(bm, bd))
    return _report("nne", ad, bd, x, t0, x_star)


# ------------------------------------------------------- streamed ingestion --
STREAM_MIN_BYTES = 1 << 30      # host matrices at least this large are streamed in row chunks
STREAM_CHUNKS = 16


class _PinnedRing:
    """K page-locked staging buffers for pageable host input (numpy arrays, the
    reference's convention): the driver would otherwise stage a pageable copy through
    its own small bounce buffers at ~10 GB/s.  Host threads copy a row chunk into a free
    slot (torch's multi-threaded CPU copy, GIL released) while the copy engine moves
    the previous slot over PCIe; a slot is reused once its H2D event has completed.
    Rings are per host thread (the reference's API is safe for concurrent calls)."""

    SLOTS = 4
    PIECE_BYTES = 256 << 20

    def __init__(self):
        self._local = threading.local()    # one ring per host thread: concurrent calls stay safe

    def slots(self, nbytes: int):
        loc = self._local
        if not getattr(loc, "bufs", None) or loc.bufs[0].numel() < nbytes:
            loc.bufs = [torch.empty(nbytes, dtype=torch.uint8, pin_memory=True) for _ in range(self.SLOTS)]
            loc.events = [None] * self.SLOTS
        return loc.bufs, loc.events

    def release(self):
        self._local.bufs, self._local.events = [], []


_PINNED = _PinnedRing()


def _ingest_streamed(a_cpu: torch.Tensor, want_gram: bool, sketch_plan=None):
    """Host -> device copy of A in row chunks on a side stream, overlapped with the
    per-chunk work that does not need all of A: validation + ||A||_F^2, the kappa0
    SYRK (accumulated chunk by chunk) and the (speculative) sketch partial sums
    with global row offsets.  Pageable input is staged through a pinned ring
    (`_PinnedRing`), chunk by chunk, interleaved with the enqueueing of that chunk's
    device work.  Returns (DMat, G or None, sketch (total, flag) or None)."""
    from .device import device as _device
    from .sketch import _sketch_sum
    dev = _device()
    m, n = a_cpu.shape
    out = torch.empty((m, n), dtype=torch.float64, device=dev)
    compute = torch.cuda.current_stream()
    copier = torch.cuda.Stream(device=dev)
    copier.wait_stream(compute)          # `out` may reuse memory still read by queued kernels
    rows = max(64, -(-m // STREAM_CHUNKS))
    rows = -(-rows // 64) * 64
    chunks = [(r0, min(m, r0 + rows)) for r0 in range(0, m, rows)]
    pinned = a_cpu.is_pinned()
    if not pinned:
        piece = max(1, min(rows, _PINNED.PIECE_BYTES // (n * 8)))   # rows per staged piece
        bufs, slot_events = _PINNED.slots(piece * n * 8)
        nslot = [0]
    stats = torch.zeros(2, dtype=torch.float64, device=dev)
    g = torch.zeros((n, n), dtype=torch.float64, device=dev) if want_gram else None
    sk_total = sk_flag = None
    if sketch_plan is not None:
        dsk, level_code = sketch_plan
        sk_total = torch.zeros((n, dsk.op.d), dtype=torch.float64, device=dev)
        sk_flag = torch.zeros(1, dtype=torch.int32, device=dev)
    lib = _lib.lib()

    def enqueue_copy(i, r0, r1):
        with torch.cuda.stream(copier):
            if pinned:
                out[r0:r1].copy_(a_cpu[r0:r1], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(copier)
                return ev
            for p0 in range(r0, r1, piece):
                p1 = min(r1, p0 + piece)
                slot = nslot[0] % len(bufs)
                nslot[0] += 1
                if slot_events[slot] is not None:
                    slot_events[slot].synchronize()     # the H2D that last used this slot is done
                stage = bufs[slot][: (p1 - p0) * n * 8].view(torch.float64).view(p1 - p0, n)
                stage.copy_(a_cpu[p0:p1])                # host threads, pageable -> pinned
                out[p0:p1].copy_(stage, non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(copier)
                slot_events[slot] = ev
        return ev

    # pinned input: every copy is enqueued up front; pageable input: the host stages
    # chunk i + 1 while the GPU copies and processes chunk i
    events = [enqueue_copy(i, r0, r1) for i, (r0, r1) in enumerate(chunks)] if pinned else []
    for i, (r0, r1) in enumerate(chunks):
        ev = events[i] if pinned else enqueue_copy(i, r0, r1)
        compute.wait_event(ev)
        part = out[r0:r1]
        wp, wn = WORKSPACE.get(lib.sk_matrix_stats_workspace(r1 - r0, n))
        call("sk_cast_stats_async", part.data_ptr(), 8, r1 - r0, n, n, None, n, stats.data_ptr(), wp, wn,
             stream_handle())
        if g is not None:
            _gram(part, out=g, accumulate=i > 0)
        if sketch_plan is not None:
            _sketch_sum(dsk, part, level_code, row_offset=r0, out=sk_total, accumulate=i > 0,
                        overflow_flag=sk_flag)
    out.record_stream(copier)
    st = stats.cpu()
    if st[0] > 0:
        raise ValueError("a contains non-finite entries")
    ad = DMat(out, float(st[1]), "numpy")
    return ad, g, ((sk_total, sk_flag) if sketch_plan is not None else None)


# ------------------------------------------------------------ preconditioner --
def _build_dev(ad: DMat, d_factor, transform, level, seed, diagnostics=True, strict=False, stages=None,
               presketch=None):
    m, n = ad.shape
    if m < n:
        raise DimensionMismatch(f"need rows >= cols, got {m} x {n}")
    d = int(math.ceil(d_factor * n))
    if d < n:
        raise ValueError(f"d_factor {d_factor} gives d={d} < n={n}")
    if stages is not None:
        stages.mark("sketch")
    if presketch is not None and presketch[0] == (level.name, d, transform, seed):
        # the streamed ingestion already accumulated this exact sketch
        from .errors import Overflow
        from .sketch import _sketch_finalize
        _, op, total, flag = presketch
        if int(flag.item()):
            raise Overflow(f"input exceeds the {level.name} range")
        a_s, _ = _sketch_finalize(total, op, level)
    else:
        op, dsk = _make_sketch_dev(m, d, transform, seed)
        a_s, _ = _apply_dev(op, ad, level, dsk)   # Overflow on demotion (src/solvers.py:191-193)
    if stages is not None:
        stages.mark("level_qr")
    r_s = _qr_level_dev(a_s, level, d, n)       # RankDeficient / Overflow
    if bool((torch.diagonal(r_s) == 0).any().item()):
        raise RankDeficient("sketched factor has a zero diagonal entry")
    if stages is not None:
        stages.mark("diag_rs")
    kappa_rs = _kappa(r_s, strict) if diagnostics else math.nan
    pre = Preconditioner(r_s=r_s, computed_in=level, kappa_rs=kappa_rs, sketch_descriptor=op.descriptor())
    return pre


def build_preconditioner(a, d_factor=3.0, transform=DCT2, level=BINARY64, seed=0, *, diagnostics=True,
                         strict_diagnostics=False):
    """src/solvers.py:168-202."""
    return _build_dev(as_dmat(a), d_factor, transform, level, seed, diagnostics, strict_diagnostics)


def _precondition_dev(ad: DMat, pre: Preconditioner, diagnostics=True, strict=False, stages=None,
                      out: torch.Tensor | None = None) -> torch.Tensor:
    r = pre.r_device()
    if r.shape[0] != ad.shape[1]:
        raise DimensionMismatch(f"r_s is {tuple(r.shape)} but A has {ad.shape[1]} columns")
    if stages is not None:
        stages.mark("trsm")
    a_p = _trsm(ad, r, out=out)                 # SingularTriangular on a zero diagonal
    if stages is not None:
        stages.mark("diag_ap")
    pre.kappa_ap = _kappa(a_p, strict) if diagnostics else math.nan
    return a_p


def precondition_matrix(a, pre, *, diagnostics=True, strict_diagnostics=False):
    """src/solvers.py:205-215: A_p = A R_s^{-1}; sets pre.kappa_ap."""
    ad = as_dmat(a)
    return like_input(_precondition_dev(ad, pre, diagnostics, strict_diagnostics), ad.kind)


class _ApScratch:
    """One reusable A_p buffer per device for algorithm1_pipeline, where A_p never
    leaves the call: a fresh 68.7 GB allocation per solve (config 3) costs a
    variable 0-300 ms of page mapping.  `release_scratch()` drops it."""

    def __init__(self):
        self._lock = threading.Lock()
        self._bufs = {}

    def take(self, m, n, device):
        from .dense import _new_ap
        key = (torch.device(device).index, m, n)
        with self._lock:
            t = self._bufs.pop(key, None)
        return key, (t if t is not None else _new_ap(m, n, device))

    def give(self, key, t):
        with self._lock:
            self._bufs = {key: t}          # keep at most one (the most recent shape)

    def release(self):
        with self._lock:
            self._bufs = {}


_AP_SCRATCH = _ApScratch()

AP_CHUNK_ROWS = None        # rows per A_p chunk when A_p is produced chunk by chunk (None: auto)
AP_HEADROOM = 24 << 30      # device bytes kept free beside a full A_p (workspaces, sketch, LU)


def _ap_chunk_rows(m: int, n: int, dev) -> int:
    """0 when the full m x n A_p fits beside A (the default, one TRSM, one Gram), else
    the row-chunk height of the streamed TRSM -> Gram (at config 4 on
    two GPUs, A_p of 8M x 2048 rows does not fit next to A).  SK_AP_CHUNK_ROWS or
    AP_CHUNK_ROWS forces a height (tests)."""
    import os
    forced = AP_CHUNK_ROWS or int(os.environ.get("SK_AP_CHUNK_ROWS", "0") or 0)
    if forced:
        return forced if forced < m else 0
    need = 8 * m * n
    key = (torch.device(dev).index, m, n)
    if key in _AP_SCRATCH._bufs:          # already resident from an earlier solve
        return 0
    free, _ = torch.cuda.mem_get_info(dev)
    if need + AP_HEADROOM <= free:
        return 0
    rows = 1 << 20
    while rows > 65536 and 8 * rows * n * 2 + AP_HEADROOM > free:
        rows //= 2
    return rows


def _trsm_gram_chunked(ad: DMat, r: torch.Tensor, bd: torch.Tensor, method: str, rows: int):
    """A_p = A R^-1 produced `rows` rows at a time and consumed at once by the Gram:
    G = sum_c A_p,c^T A_c (HPNE) or A_p,c^T A_p,c (PNE), rhs = sum_c A_p,c^T b_c.  A_p is
    never materialised; each chunk's Gram is formed on the same engine as the whole
    (INT8 Ozaki-II at scale, per-chunk FP64 results summed in FP64; A's column scales
    from its one full scan) and its A_p^T b comes from the chunk's column scan."""
    from .dense import _colstats, _gram_engine, _new_ap
    at = ad.t
    m, n = at.shape
    dev = at.device
    g = torch.empty((n, n), dtype=torch.float64, device=dev)
    rhs = torch.zeros(n, dtype=torch.float64, device=dev)
    buf = _new_ap(rows, n, dev)
    ozaki = _gram_engine(rows, n, True, None) == "ozaki"
    a_stats = ad.colstats if (method != "pne" and ozaki) else None
    if method != "pne" and ozaki and a_stats is None:
        a_stats = _colstats(at)
    for i, r0 in enumerate(range(0, m, rows)):
        r1 = min(m, r0 + rows)
        a_c, ap_c, b_c = at[r0:r1], buf[: r1 - r0], bd[r0:r1]
        _trsm(a_c, r, out=ap_c)
        y = None if method == "pne" else (DMat(a_c, None, "torch", a_stats) if ozaki else a_c)
        if ozaki and (r1 - r0) * n * n >= 1 << 33:
            st = _colstats(ap_c, b_c)
            _gram(DMat(ap_c, None, "torch", st[: 2 * n]), y, out=g, accumulate=i > 0)
            rhs += st[2 * n:]
        else:
            _gram(ap_c, y if not isinstance(y, DMat) else y.t, out=g, accumulate=i > 0, engine="dmma")
            _gemv_t(ap_c, b_c, out=rhs, accumulate=True)
    del buf
    return g, rhs


def release_scratch():
    """Free the cached A_p buffer of algorithm1_pipeline and the pinned staging ring."""
    _AP_SCRATCH.release()
    _PINNED.release()


def _prepare_dev(ad, d_factor, transform, level, seed, diagnostics=True, strict=False, stages=None,
                 presketch=None, out=None, build_only=False):
    escalated_from = None
    while True:
        try:
            pre = _build_dev(ad, d_factor, transform, level, seed, diagnostics, strict, stages, presketch)
            if build_only:   # A_p is produced chunk by chunk by the caller
                return pre, None, escalated_from
            a_p = _precondition_dev(ad, pre, diagnostics, strict, stages, out=out)
            return pre, a_p, escalated_from
        except RankDeficient:
            wider = next_higher(level)
            if escalated_from is not None or wider is None:
                raise
            escalated_from = level
            level = wider


def prepare_preconditioner(a, d_factor=3.0, transform=DCT2, level=BINARY64, seed=0, *, diagnostics=True,
                           strict_diagnostics=False):
    """src/solvers.py:255-279: one escalation on RankDeficient."""
    ad = as_dmat(a)
    pre, a_p, esc = _prepare_dev(ad, d_factor, transform, level, seed, diagnostics, strict_diagnostics)
    return pre, like_input(a_p, ad.kind), esc


# -------------------------------------------------------------- PNE / HPNE ---
def _a_p_dev(a_p, ad: DMat) -> torch.Tensor:
    if isinstance(a_p, torch.Tensor) and a_p.is_cuda and a_p.dtype == torch.float64 and a_p.is_contiguous():
        t = a_p
    else:
        t = as_dmat(a_p, "a_p").t
    if tuple(t.shape) != ad.shape:
        raise DimensionMismatch(f"a_p shape {tuple(t.shape)} != a shape {ad.shape}")
    return t


_SIDE_STREAMS: dict = {}


def _gram_and_rhs(x, y, bd):
    """G = X^T Y and rhs = X^T b.  On the INT8 engine the column scan of X that sets its
    scales forms X^T b in the same pass; on DMMA the streaming GEMV runs on a second
    stream under the Gram."""
    from .dense import _colstats, _gram_engine
    xt = x.t if isinstance(x, DMat) else x
    m, n = xt.shape
    if _gram_engine(m, n, False, None) == "ozaki":
        st = _colstats(xt, bd)
        g = _gram(DMat(xt, None, "torch", st[: 2 * n]), y)
        return g, st[2 * n:]
    cur = torch.cuda.current_stream()
    side = _SIDE_STREAMS.get(cur.device.index)
    if side is None:
        side = _SIDE_STREAMS.setdefault(cur.device.index, torch.cuda.Stream(device=cur.device))
    side.wait_stream(cur)
    with torch.cuda.stream(side):
        rhs = _gemv_t(x, bd)
    g = _gram(x, y)
    cur.wait_stream(side)
    rhs.record_stream(cur)
    return g, rhs


def _pne_dev(ad, bd, pre, a_p, stages=None, gram=None):
    if stages is not None and gram is None:
        stages.mark("gram")
    g, rhs = gram if gram is not None else _gram_and_rhs(a_p, None, bd)
    if stages is not None:
        stages.mark("nxn")
    try:
        y = _chol_solve(g, rhs)
    except NotPositiveDefinite:
        y = _lu_solve(g, rhs)
    return _trsv(pre.r_device(), y)


def _hpne_dev(ad, bd, pre, a_p, stages=None, gram=None):
    if stages is not None and gram is None:
        stages.mark("gram")
    g, rhs = gram if gram is not None else _gram_and_rhs(a_p, ad, bd)
    if stages is not None:
        stages.mark("nxn")
    return _lu_solve(g, rhs)


def solve_pne(a, b, pre, x_star=None, a_p=None, *, diagnostics=True, strict_diagnostics=False):
    """src/solvers.py:218-237: Cholesky of A_p^T A_p (LU fallback), x = R_s^{-1} y."""
    ad, bd = _check_system(a, b)
    t0 = time.perf_counter()
    ap = _precondition_dev(ad, pre, diagnostics, strict_diagnostics) if a_p is None else _a_p_dev(a_p, ad)
    x = _pne_dev(ad, bd, pre, ap)
    return _report("pne", ad, bd, x, t0, x_star, preconditioner=pre)


def solve_hpne(a, b, pre, x_star=None, a_p=None, *, diagnostics=True, strict_diagnostics=False):
    """src/solvers.py:240-252: LU of A_p^T A."""
    ad, bd = _check_system(a, b)
    t0 = time.perf_counter()
    ap = _precondition_dev(ad, pre, diagnostics, strict_diagnostics) if a_p is None else _a_p_dev(a_p, ad)
    x = _hpne_dev(ad, bd, pre, ap)
    return _report("hpne", ad, bd, x, t0, x_star, preconditioner=pre)


def algorithm1_pipeline(a, b, method="pne", precision="auto", d_factor=3.0, transform=DCT2, seed=0,
                        x_star=None, *, diagnostics=True, strict_diagnostics=False, stage_timing=False):
    """Algorithm 1 end to end (src/solvers.py:282-324), entirely on the device.

    Extra keyword-only options (not in the reference): diagnostics,
    strict_diagnostics (see module docstring) and stage_timing (fills
    SolveReport.stage_ms with CUDA-event times per stage).
    """
    stages = _Stages(stage_timing)
    stages.mark("check")
    # wall_ms covers the estimate, sketch, factor, precondition and solve like the
    # reference's (src/solvers.py:300-306).  For device-resident input under "auto" the
    # validation pass is fused into the kappa0 Gram and for streamed host input into the
    # H2D copy, so there the clock starts before them (it then also covers validation).
    t0 = time.perf_counter()
    if method not in ("pne", "hpne"):
        raise ValueError(f"pipeline method must be pne or hpne, got {method!r}")
    if not isinstance(precision, PrecisionLevel) and precision != "auto":
        level_from_name(precision)      # ValueError before any work, like the reference
    host = _host_f64_matrix(a)
    presketch = None
    gram_auto = None
    if host is not None and host.numel() * 8 >= STREAM_MIN_BYTES and host.shape[0] >= host.shape[1]:
        # Streamed ingestion: the H2D copy of A overlaps with validation, the kappa0
        # Gram and the sketch (the real one for a fixed level, a speculative binary16
        # one under "auto", reused if kappa0 selects binary16).
        from .precision import BINARY16
        from .sketch import DeviceSketch
        m, n = host.shape
        fixed = precision if isinstance(precision, PrecisionLevel) else (
            None if precision == "auto" else level_from_name(precision))
        spec_level = fixed or BINARY16
        d = int(math.ceil(d_factor * n))
        # only the tensor-core (binary16) sketch is chunk-friendly; the FFT sketch of
        # binary32/64 transforms all M rows per call, so it runs once after ingestion
        op, dsk = _make_sketch_dev(m, d, transform, seed) if (d >= n and spec_level is BINARY16) else (None, None)
        plan = (dsk, spec_level.code) if op is not None else None
        ad, gram_auto, sk = _ingest_streamed(host, want_gram=precision == "auto", sketch_plan=plan)
        if sk is not None:
            presketch = ((spec_level.name, d, transform, seed), op, sk[0], sk[1])
        bd = as_dvec(b, m)
    elif (precision == "auto" and isinstance(a, torch.Tensor) and a.is_cuda and a.dim() == 2
          and a.dtype == torch.float64 and a.stride(-1) == 1 and a.shape[0] >= a.shape[1] > 0):
        # device-resident A under "auto": the kappa0 Gram reads A anyway, so it doubles
        # as the validation pass (non-finite A => non-finite G; ||A||_F^2 = trace G)
        from .dense import _colstats, _gram_engine, _rm
        at = _rm(a)
        m, n = at.shape
        bd = as_dvec(b, m)
        # the INT8 Gram engine scales columns by max|A[:, j]| (and checks them against
        # ||A[:, j]||): scan A once for both of its Grams (kappa0 SYRK, A_p^T A in HPNE)
        cm = _colstats(at) if _gram_engine(m, n, False, None) == "ozaki" else None
        gram_auto = _gram(DMat(at, None, "torch", cm))
        chk = (C.c_double * 2)()
        wp, wn = WORKSPACE.get(256)
        call("sk_gram_check", gram_auto.data_ptr(), n, chk, wp, wn, stream_handle())
        if chk[0] > 0:
            ad = as_dmat(at)          # raises ValueError on non-finite A, like _as_matrix
        else:
            ad = DMat(at, float(chk[1]), "torch", cm)
    else:
        ad, bd = _check_system(a, b)
        t0 = time.perf_counter()     # src/solvers.py:303: after _check_system, before the estimate
    decision = None
    if isinstance(precision, PrecisionLevel):
        level = precision
    elif precision == "auto":
        stages.mark("kappa0")
        if gram_auto is not None:
            from .precision import _kappa0_from_gram, select_precision
            k0, over = _kappa0_from_gram(gram_auto)
            decision = PrecisionDecision(kappa0=k0, selected=select_precision(k0, over), overflowed=over)
        else:
            decision = _decide_dev(ad)
        level = decision.selected
    else:
        level = level_from_name(precision)
    m_rows, n_cols = ad.shape
    chunk = _ap_chunk_rows(m_rows, n_cols, ad.t.device)
    if chunk:
        # A_p does not fit beside A: TRSM -> Gram per row chunk, A_p never materialised
        pre, _, escalated_from = _prepare_dev(ad, d_factor, transform, level, seed, diagnostics,
                                              strict_diagnostics, stages, presketch, build_only=True)
        stages.mark("trsm_gram")
        gr = _trsm_gram_chunked(ad, pre.r_device(), bd, method, chunk)
        pre.kappa_ap = _kappa_from_gram(gr[0], strict_diagnostics) if (diagnostics and method == "pne") \
            else math.nan
        x = (_pne_dev if method == "pne" else _hpne_dev)(ad, bd, pre, None, stages, gram=gr)
    else:
        ap_key, ap_buf = _AP_SCRATCH.take(m_rows, n_cols, ad.t.device)
        try:
            pre, a_p, escalated_from = _prepare_dev(ad, d_factor, transform, level, seed, diagnostics,
                                                    strict_diagnostics, stages, presketch, out=ap_buf)
            x = (_pne_dev if method == "pne" else _hpne_dev)(ad, bd, pre, a_p, stages)
        finally:
            _AP_SCRATCH.give(ap_key, ap_buf)
    stages.mark("report")
    report = _report(method, ad, bd, x, t0, x_star, preconditioner=pre, stages=stages)
    report.precision_decision = decision
    report.escalated_from = escalated_from
    report.wall_ms = (time.perf_counter() - t0) * 1e3
    return report
