/*
 * sklsq.h — C ABI of the B200-native sketch-preconditioned least-squares kernels.
 *
 * Drop-in boundary for the hot path of the reference package `sketchlsq` 0.1.0
 * (arXiv 2603.16644, Algorithm 1).  The reference is pure Python/numpy, so it has
 * no native FFI of its own; these entry points replace, one for one, the numpy /
 * BLAS / pocketfft calls that its Python functions make (cited per function as
 * `src/<file>:<line>` = /root/reference/pkg/src/sketchlsq/<file>:<line>).  The
 * Python layer `paper_2603_16644_b200` binds them with ctypes.
 *
 * Conventions
 *  - All matrix pointers are DEVICE pointers (cudaMalloc / torch CUDA storage).
 *    Matrices are row-major with an explicit leading dimension (elements) unless
 *    a function says otherwise.  No torch types appear in any signature.
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).  Work is
 *    stream-ordered.  Functions that return a numerical verdict (QR, Cholesky, LU,
 *    kappa0, finiteness) synchronise `stream` before returning it -- unless verdicts
 *    are deferred to a device record (sk_defer_verdicts, below), which makes a whole
 *    solve capturable as one CUDA graph.
 *  - `ws` / `ws_bytes`: caller-owned device workspace; query the size with the
 *    matching *_workspace() call.  No allocation happens on the hot path.
 *  - Return: SK_OK (0), a numerical failure code (>0, 1:1 with the reference
 *    exception classes of src/errors.py:10-55), SK_ERR_CUDA (-1) or SK_ERR_ARG (-2).
 *    Detail (offending column / pivot value) goes to the optional sk_status*;
 *    sk_last_error() returns a thread-local message.
 */
#ifndef SKLSQ_H
#define SKLSQ_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *sk_stream_t;

enum sk_code {
    SK_OK = 0,
    SK_RANK_DEFICIENT = 1,        /* errors.RankDeficient        src/errors.py:14 */
    SK_SINGULAR_TRIANGULAR = 2,   /* errors.SingularTriangular   src/errors.py:18 */
    SK_NUMERICALLY_SINGULAR = 3,  /* errors.NumericallySingular  src/errors.py:22 */
    SK_NOT_POSITIVE_DEFINITE = 4, /* errors.NotPositiveDefinite  src/errors.py:26 */
    SK_OVERFLOW = 5,              /* errors.Overflow             src/errors.py:54 */
    SK_DIMENSION_MISMATCH = 6,    /* errors.DimensionMismatch    src/errors.py:34 */
    SK_NO_CONVERGENCE = 7,        /* errors.NoConvergence        src/errors.py:30 */
    SK_NOT_SYMMETRIC = 8,         /* ValueError, src/dense.py:332-335 */
    SK_NON_FINITE = 9,            /* ValueError, src/dense.py:63-64 */
    SK_ERR_CUDA = -1,
    SK_ERR_ARG = -2
};

enum sk_level { SK_BINARY16 = 16, SK_BINARY32 = 32, SK_BINARY64 = 64 };
enum sk_transform { SK_DCT2 = 0, SK_WHT = 1 };
enum sk_dtype { SK_F16 = 2, SK_F32 = 4, SK_F64 = 8 };

typedef struct sk_status {
    int32_t code;     /* sk_code */
    int32_t pad;
    int64_t index;    /* column / pivot index of the failure, -1 if none */
    double value;     /* pivot value or magnitude at the failure */
    double aux;       /* threshold (LU) or extra detail */
} sk_status;

/* ---- library ------------------------------------------------------------ */
int sk_version(void);
const char *sk_last_error(void);
int sk_sm_count(int device);
/* Number of kernels this library has launched in the process (instrumentation:
 * the bench reports launches inside its timed region from the difference). */
uint64_t sk_launch_count(void);

/* ---- streaming passes over A (HBM-bound) --------------------------------- */
/* _as_matrix + astype(float64) + ||A||_F^2 in one pass: src/dense.py:57-65,
 * src/solvers.py:87-96, src/solvers.py:102.  src dtype SK_F16/F32/F64 -> dst f64.
 * stats_host[0] = number of non-finite entries, stats_host[1] = sum of squares. */
size_t sk_matrix_stats_workspace(int64_t rows, int64_t cols);
int sk_cast_stats(const void *src, int src_dtype, int64_t rows, int64_t cols, int64_t ld_src,
                  double *dst, int64_t ld_dst, double *stats_host,
                  void *ws, size_t ws_bytes, sk_stream_t stream);

/* Stream-ordered variant for row chunks arriving while earlier chunks are being
 * processed: stats_dev[0] += #non-finite, stats_dev[1] += sum of squares (device
 * doubles, caller-zeroed), no host synchronisation. */
int sk_cast_stats_async(const void *src, int src_dtype, int64_t rows, int64_t cols, int64_t ld_src,
                        double *dst, int64_t ld_dst, double *stats_dev, void *ws, size_t ws_bytes,
                        sk_stream_t stream);

/* round_to_precision(A, level).overflowed without materialising the rounding:
 * src/precision.py:90-103, src/solvers.py:191-193.  *overflowed_host = 0/1. */
int sk_level_overflow(const double *a, int64_t rows, int64_t cols, int64_t lda, int level,
                      int *overflowed_host, void *ws, size_t ws_bytes, sk_stream_t stream);

/* r = A x - b; out_host[0] = ||r||^2, out_host[1] = ||x||^2: src/solvers.py:99-117. */
int sk_residual(const double *a, int64_t rows, int64_t cols, int64_t lda, const double *x,
                const double *b, double *r, double *out_host, void *ws, size_t ws_bytes,
                sk_stream_t stream);

/* Stream-ordered sk_residual: out_dev[0] = ||A x - b||^2, out_dev[1] = ||x||^2 (device
 * doubles), no host synchronisation (the deferred-verdict / CUDA-graph solve path). */
int sk_residual_async(const double *a, int64_t rows, int64_t cols, int64_t lda, const double *x,
                      const double *b, double *r, double *out_dev, void *ws, size_t ws_bytes,
                      sk_stream_t stream);

/* ---- deferred numerical verdicts (CUDA-graph capture of a whole solve) ----
 * sk_defer_verdicts(status_dev) installs a DEVICE sk_status record (caller-zeroed) on
 * the calling host thread; NULL removes it.  While installed, the entry points that
 * return a numerical verdict on a device-resident path (sk_qr_r, sk_trsm_right_upper_f64,
 * sk_lu_solve_f64, sk_chol_solve_f64, sk_trsv_f64) do not synchronise: they enqueue a
 * check that stores the verdict (code, index, value, aux as in sk_status) into the
 * record and return SK_OK.  The first failure in stream order wins, so one read of the
 * record after the solve raises what the eager calls would have raised first.  The INT8
 * Ozaki-II engines (sk_gram_ozaki_acc_f64 with accumulate = 0, sk_trsm_ozaki_f64) keep
 * their operand guard on the device too (flag 256 bytes past their workspace, which must
 * then be 256 bytes larger) and run the DMMA fallback gated on it.  Kernels
 * with data-dependent control flow (LU, Cholesky) run on the identity once a failure is
 * recorded (their outputs are then meaningless; the record says so).  Entry points whose
 * result is a host value (sk_cast_stats, sk_residual, sk_kappa0_*, sk_jacobi_sv_f64,
 * sk_level_overflow, ...) return
 * SK_ERR_ARG while verdicts are deferred.  Replaces the host-side exception points of
 * src/solvers.py:168-252 (raise sites kept in order). */
int sk_defer_verdicts(sk_status *status_dev);
/* *flag_dev != 0 -> record `code` (e.g. the sketch's overflow flag -> SK_OVERFLOW). */
int sk_note_flag(const int *flag_dev, int code, sk_stream_t stream);
/* *x_dev > 0 -> record `code` (e.g. sk_cast_stats_async's non-finite count -> SK_NON_FINITE). */
int sk_note_positive(const double *x_dev, int code, sk_stream_t stream);
/* first exactly-zero diagonal entry of the row-major n x n R -> `code` with its index
 * (src/solvers.py:197-199's RankDeficient on the sketched factor). */
int sk_note_zero_diagonal(const double *r, int64_t ldr, int64_t n, int code, sk_stream_t stream);
/* if a failure is recorded: overwrite the rows x cols matrix (2/4/8-byte elements, ld
 * elements, col_major 0/1) with the identity, so later data-dependent kernels see a
 * well-conditioned operand. */
int sk_guard_identity(int elem_bytes, void *a, int64_t rows, int64_t cols, int64_t ld, int col_major,
                      sk_stream_t stream);

/* ---- FP64 tensor-pipe (DMMA) products ------------------------------------ */
/* G (n x n, row-major, ldg) = X^T Y with X (m x n, ldx), Y (m x n, ldy).
 * If Y == X the SYRK path runs (lower tiles + exact mirror; numpy's a.T @ a is
 * exactly symmetric, src/dense.py:332-335 relies on it).
 * Replaces `a.T @ a` src/precision.py:230, `a_p.T @ a_p` src/solvers.py:230,
 * `a_p.T @ a` src/solvers.py:251, `b_matrix.T @ a` src/solvers.py:164,
 * `a.T @ a` src/solvers.py:137.  If `accumulate` != 0, G += X^T Y. */
size_t sk_gram_workspace(int64_t m, int64_t n);
int sk_gram_f64(const double *x, int64_t ldx, const double *y, int64_t ldy, int64_t m, int64_t n,
                double *g, int64_t ldg, int accumulate, void *ws, size_t ws_bytes,
                sk_stream_t stream);

/* Same product on the INT8 tensor cores (tcgen05 kind::i8, Ozaki scheme II): X and Y
 * scaled per column to t-bit integers, nm exact modular INT8 GEMMs (nm and t chosen so
 * the worst case stays 2^8 under the FP64 GEMM's gamma_m bound: 15 moduli, t = 47 at
 * m = 4M rows; 16, t = 51 below 2^17 rows), Chinese-remainder reconstruction in
 * 128-bit integers.  The only
 * rounding is the t-bit scaling: |G - X^T Y|_ij <= 2^-t (2^e_i sum|Y_j| + 2^f_j
 * sum|X_i|) / 2, with 2^e_i > max|X_i|.  SYRK when Y == X (exactly symmetric).
 * Workspace from sk_gram_ozaki_workspace(m, n, syrk). */
size_t sk_gram_ozaki_workspace(int64_t m, int64_t n, int syrk);
int sk_gram_ozaki_f64(const double *x, int64_t ldx, const double *y, int64_t ldy, int64_t m, int64_t n,
                      double *g, int64_t ldg, void *ws, size_t ws_bytes, sk_stream_t stream);
/* Same with the column statistics supplied (device, 2n doubles each, from
 * sk_colstats_f64 of the same matrix; NULL = computed here), so a matrix used by two
 * Grams (A in the kappa0 SYRK and the HPNE product) is scanned once.
 * Guard: if any column has max|x| sqrt(m) > 64 ||x||_2 (a spiky column, where the
 * scaled-integer error bound would exceed an FP64 GEMM's) or a non-finite entry, the
 * product runs on the FP64 DMMA path instead (sk_gram_ozaki_fell_back() == 1). */
int sk_gram_ozaki_ex_f64(const double *x, int64_t ldx, const double *y, int64_t ldy, int64_t m, int64_t n,
                         const double *xstats, const double *ystats, double *g, int64_t ldg, void *ws,
                         size_t ws_bytes, sk_stream_t stream);
/* Same, G += X^T Y when accumulate != 0 (the per-call FP64 result is added to G, so
 * row-chunked products, e.g. A_p produced chunk by chunk, sum their Grams in FP64). */
int sk_gram_ozaki_acc_f64(const double *x, int64_t ldx, const double *y, int64_t ldy, int64_t m, int64_t n,
                          const double *xstats, const double *ystats, double *g, int64_t ldg, int accumulate,
                          void *ws, size_t ws_bytes, sk_stream_t stream);
/* 1 if the last sk_gram_ozaki_* call on this host thread took the FP64 fallback. */
int sk_gram_ozaki_fell_back(void);
/* stats[j] = max_k |X[k,j]|, stats[n + j] = sum_k X[k,j]^2 and, if v != NULL,
 * stats[2n + j] = sum_k X[k,j] v[k] (the right-hand side a_p.T @ b of
 * src/solvers.py:231/251 from the same pass); device, fixed-order, deterministic; a
 * non-finite column gives max = +inf. */
size_t sk_colstats_workspace(int64_t n);
int sk_colstats_f64(const double *x, int64_t ldx, int64_t m, int64_t n, const double *v, double *stats, void *ws,
                    size_t ws_bytes, sk_stream_t stream);

/* out (n) = X^T v (X m x n row-major): `a_p.T @ b` src/solvers.py:231/251. */
size_t sk_gemv_t_workspace(int64_t m, int64_t n);
int sk_gemv_t_f64(const double *x, int64_t ldx, int64_t m, int64_t n, const double *v,
                  double *out, int accumulate, void *ws, size_t ws_bytes, sk_stream_t stream);

/* A_p = A R^{-1} (R n x n upper, row-major ldr): precondition_matrix
 * src/solvers.py:205-215 via triangular_solve(R, A^T, transposed=True)
 * src/dense.py:204-242.  Returns SK_SINGULAR_TRIANGULAR on an exactly zero
 * diagonal (index in status).  ap may alias a. */
int sk_trsm_right_upper_f64(const double *a, int64_t lda, int64_t m, int64_t n, const double *r,
                            int64_t ldr, double *ap, int64_t ldap, sk_status *status,
                            sk_stream_t stream);
/* Same solve, blocked: columns are halved recursively (h = n/2 rounded to 256) down to
 * leaves of <= 1024 columns solved by the kernel above; each off-diagonal update
 * A_p[:, h:] = A[:, h:] - A_p[:, :h] R[:h, h:] runs on the INT8 tensor cores (Ozaki
 * scheme II as in sk_gram_ozaki_f64, row scales for A_p, column scales for R), error
 * 2^-t (2^e_r sum|R_j| + 2^f_j sum|A_p,r|) / 2 per entry, an FP64 GEMM's size.  Spiky
 * rows / columns or non-finite values re-run the whole solve on the DMMA kernel
 * (sk_trsm_ozaki_fell_back() == 1).  ap must not alias a.  Workspace from
 * sk_trsm_ozaki_workspace(m, n). */
size_t sk_trsm_ozaki_workspace(int64_t m, int64_t n);
int sk_trsm_ozaki_f64(const double *a, int64_t lda, int64_t m, int64_t n, const double *r, int64_t ldr,
                      double *ap, int64_t ldap, sk_status *status, void *ws, size_t ws_bytes,
                      sk_stream_t stream);
int sk_trsm_ozaki_fell_back(void);

/* ---- sketch --------------------------------------------------------------- */
/* Partial SRTT sketch of a row block: out (d x n, COLUMN-major, ldo >= d, f64)
 * (+)= Omega[:, row_offset : row_offset+m_local] * round_level(A_local) where
 * Omega = S F D is the unscaled operator of src/sketch.py:138-169 (signs of
 * length m_pad as +-1 doubles, sampled rows int64).  The sqrt(m_pad/d) scale and
 * the final rounding happen in sk_sketch_finalize so that partials can be summed
 * across row shards (NCCL) first.  Overflow of the demotion is OR-ed into
 * *overflow_flag_dev (device int).  transform SK_DCT2/SK_WHT, level 16/32/64. */
enum sk_sketch_algo { SK_SKETCH_AUTO = 0, SK_SKETCH_DMMA = 1, SK_SKETCH_TC = 2, SK_SKETCH_FFT = 3 };
/* The sign vector of make_sketch (src/sketch.py:89-112):
 *   rng.stream(seed, LANE).integers(0, 2, count) * 2.0 - 1.0     (src/rng.py:23-34)
 * drawn on the device, bitwise numpy's: Philox4x64-10 with key (key_lo, key_hi),
 * output block b at counter b + 1, each 64-bit word split into two 32-bit draws
 * (low half first), draw j -> +1 if its top bit is set else -1. */
int sk_sketch_signs(uint64_t key_lo, uint64_t key_hi, int64_t count, double *signs, sk_stream_t stream);
size_t sk_sketch_workspace(int level, int64_t m_local, int64_t n, int64_t d);
/* Exact workspace for one (level, transform, row shard of an m_pad-row operator). */
size_t sk_sketch_workspace_ex(int level, int transform, int64_t m_local, int64_t m_pad, int64_t n, int64_t d);
int sk_sketch_partial(int level, int transform, const double *a, int64_t lda, int64_t m_local,
                      int64_t row_offset, int64_t m_pad, int64_t n, const double *signs,
                      const int64_t *rows, int64_t d, double *out, int64_t ldo, int accumulate,
                      int *overflow_flag_dev, void *ws, size_t ws_bytes, sk_stream_t stream);
/* Same, choosing the engine: SK_SKETCH_TC = tcgen05 kind::f16 GEMM with TMEM
 * accumulators and TMA-staged operands (binary16 only), SK_SKETCH_DMMA = FP64
 * DMMA GEMM (any level), SK_SKETCH_AUTO = TC for binary16, else DMMA. */
int sk_sketch_partial_ex(int level, int transform, const double *a, int64_t lda, int64_t m_local,
                         int64_t row_offset, int64_t m_pad, int64_t n, const double *signs,
                         const int64_t *rows, int64_t d, double *out, int64_t ldo, int accumulate,
                         int *overflow_flag_dev, void *ws, size_t ws_bytes, sk_stream_t stream, int algo);

/* Finish the sketch: A_s = level(level(sum) * level(sqrt(m_pad/d))) written as a
 * COLUMN-major d x n matrix in the level dtype (f16/f32/f64), the layout the
 * level QR works on.  Also writes the f64 promotion to out_f64 (row-major, may
 * be NULL) for apply_sketch's return value. */
int sk_sketch_finalize(int level, const double *sum, int64_t ldsum, int64_t d, int64_t n,
                       int64_t m_pad, void *a_s_level, double *out_f64, sk_stream_t stream);

/* ---- level-precision Householder QR (R only) ------------------------------ */
/* qr_in_precision(A_s, level).r : src/precision.py:153-202 + householder_reduce
 * src/dense.py:108-161.  A_s: d x n COLUMN-major in the level dtype, overwritten.
 * binary16 follows the reference op for op (power-of-two prescale, every scalar
 * op rounded to binary16, pairwise trees of src/precision.py:106-115).
 * R (n x n row-major f64, upper, exact zeros below) is the exact promotion (and,
 * for binary16, un-scaling).  Failures: SK_RANK_DEFICIENT (index = column),
 * SK_OVERFLOW. */
size_t sk_qr_workspace(int level, int64_t d, int64_t n);
int sk_qr_r(int level, void *a_s, int64_t d, int64_t n, double *r, int64_t ldr,
            sk_status *status, void *ws, size_t ws_bytes, sk_stream_t stream);

/* qr_in_precision(a, level) in full: src/precision.py:153-202.  a is the f64 input
 * (d x n row-major, lda; not modified).  The demotion follows the reference: binary16
 * takes max|a| and the power-of-two scale on the f64 values and rounds a * scale once
 * (src/precision.py:188-194), binary32 raises SK_OVERFLOW when the demotion overflows
 * (:181-184), binary64 is householder_qr (:179-180).  R as sk_qr_r; if q != NULL the thin
 * Q (d x n row-major f64, ldq) is accumulated backward from the reflectors in the level
 * arithmetic (accumulate_thin_q src/dense.py:164-172; binary16 op for op with HALF_OPS) and
 * a non-finite binary16 Q or R gives SK_OVERFLOW (src/precision.py:200-201).
 * d <= 262144.  Workspace from sk_qr_factors_workspace(level, d, n). */
size_t sk_qr_factors_workspace(int level, int64_t d, int64_t n);
int sk_qr_in_precision_f64(int level, const double *a, int64_t lda, int64_t d, int64_t n, double *r, int64_t ldr,
                           double *q, int64_t ldq, sk_status *status, void *ws, size_t ws_bytes, sk_stream_t stream);
/* householder_reduce(a) src/dense.py:108-161 in binary64: R (n x n), the reflectors
 * (v, m x n row-major ldv: reflector j = v[j:, j] with its unnormalised first entry
 * x_0 - alpha on the diagonal, zeros above; NULL to skip) and taus (n, tau_j = 2 / v_j.v_j;
 * NULL to skip).  m <= 262144.  Workspace from sk_qr_factors_workspace(64, m, n). */
int sk_householder_f64(const double *a, int64_t lda, int64_t m, int64_t n, double *r, int64_t ldr, double *v,
                       int64_t ldv, double *taus, sk_status *status, void *ws, size_t ws_bytes, sk_stream_t stream);
/* accumulate_thin_q(reflectors, taus, m, n, ops, dtype) src/dense.py:164-172 in the level
 * dtype (16: HALF_OPS semantics; 32 / 64 native): v COLUMN-major m x n (ldv >= m),
 * reflector j in v[j:, j]; taus (n); q COLUMN-major m x n (ldq >= m), overwritten. */
int sk_accumulate_q(int level, const void *v, int64_t ldv, const void *taus, int64_t m, int64_t n, void *q,
                    int64_t ldq, sk_stream_t stream);

/* ---- n x n FP64 kernels (replicated, latency-bound) ---------------------- */
/* x = S^{-1} rhs by Cholesky: cholesky_solve src/dense.py:314-342 (symmetry gate
 * 10 eps max|S| -> SK_NOT_SYMMETRIC, pivot <= 0 or non-finite ->
 * SK_NOT_POSITIVE_DEFINITE).  S row-major n x n (symmetric).  x may alias rhs. */
size_t sk_nxn_workspace(int64_t n);
int sk_chol_solve_f64(const double *s, int64_t n, const double *rhs, double *x,
                      sk_status *status, void *ws, size_t ws_bytes, sk_stream_t stream);

/* out_host[0] = #non-finite entries of G (n x n), out_host[1] = trace(G).  With
 * G = A^T A this validates A (non-finite A => non-finite G) and gives ||A||_F^2,
 * which lets the kappa0 pass replace the separate validation pass over A. */
int sk_gram_check(const double *g, int64_t n, double *out_host, void *ws, size_t ws_bytes, sk_stream_t stream);

/* Upper Cholesky factor R = L^T (row-major n x n, zeros below) of (S + S^T)/2:
 * cholesky_factor src/dense.py:289-311 (pivot <= 0 or non-finite ->
 * SK_NOT_POSITIVE_DEFINITE).  Used for the Gram route to kappa(A_p) on tall A_p. */
int sk_chol_factor_f64(const double *s, int64_t n, double *r, sk_status *status, void *ws, size_t ws_bytes,
                       sk_stream_t stream);

/* x = G^{-1} rhs by LU with partial pivoting: lu_solve src/dense.py:245-286
 * (lowest index on ties; pivot < n eps max|G| -> SK_NUMERICALLY_SINGULAR). */
int sk_lu_solve_f64(const double *g, int64_t n, const double *rhs, double *x,
                    sk_status *status, void *ws, size_t ws_bytes, sk_stream_t stream);

/* Triangular solve R x = rhs (or R^T x = rhs): triangular_solve src/dense.py:204-242
 * for a single right-hand side.  R row-major upper.  x may alias rhs. */
int sk_trsv_f64(const double *r, int64_t ldr, int64_t n, int transposed, const double *rhs,
                double *x, sk_status *status, void *ws, size_t ws_bytes, sk_stream_t stream);

/* kappa0 from a Gram matrix G = A^T A (n x n row-major): the remainder of
 * estimate_log10_condition src/precision.py:205-251 (finite check, ||G||_1,
 * Cholesky without fallback, <=5 Hager iterations src/dense.py:451-480).
 * *kappa0_host = NaN and *overflowed_host = 1 on any breakdown. */
int sk_kappa0_from_gram(const double *g, int64_t n, double *kappa0_host, int *overflowed_host,
                        void *ws, size_t ws_bytes, sk_stream_t stream);

/* Singular values of an n x n (row-major) matrix by one-sided Jacobi with the
 * reference's round-robin schedule, gate and tolerance (jacobi_singular_values
 * src/dense.py:365-415).  sv (host, n) descending.  SK_NO_CONVERGENCE after
 * max_sweeps. Diagnostic only. */
size_t sk_jacobi_workspace(int64_t rows, int64_t n);
int sk_jacobi_sv_f64(const double *a, int64_t rows, int64_t n, int64_t lda, int max_sweeps,
                     double tol, double *sv_host, void *ws, size_t ws_bytes, sk_stream_t stream);

/* ---- the SURVEY §8(b) contract names ------------------------------------- */
/* These run on the production Gram engine, the one algorithm1_pipeline uses: the INT8
 * tensor-core Ozaki-II product (sk_gram_ozaki_ex_f64, its column scan forming X^T v in
 * the same pass) when m n^2 >= 2^33 and n >= 128, FP64 DMMA (sk_gram_f64 +
 * sk_gemv_t_f64) below; the environment variable SK_GRAM_ENGINE=dmma|ozaki overrides.
 * Gram plus rhs in one call: G = X^T Y (SYRK when Y == X) and, if v != NULL,
 * rhs = X^T v.  solve_pne / solve_hpne / solve_notnormal: `g, rhs = a_p.T @ a_p,
 * a_p.T @ b` src/solvers.py:230-231, `a_p.T @ a, a_p.T @ b` :251, `b_matrix.T @ a`
 * :164.  sk_gemm_tn_workspace(m, n) also sizes sk_syrk_f64. */
size_t sk_gemm_tn_workspace(int64_t m, int64_t n);
int sk_gemm_tn_f64(const double *x, int64_t ldx, const double *y, int64_t ldy, int64_t m, int64_t n,
                   const double *v, double *g, int64_t ldg, double *rhs, void *ws, size_t ws_bytes,
                   sk_stream_t stream);
/* G = X^T X (exactly symmetric): `a.T @ a` src/precision.py:230, src/solvers.py:137. */
int sk_syrk_f64(const double *x, int64_t ldx, int64_t m, int64_t n, double *g, int64_t ldg, void *ws,
                size_t ws_bytes, sk_stream_t stream);
/* kappa0 straight from A: estimate_log10_condition src/precision.py:205-251 (SYRK +
 * sk_kappa0_from_gram). */
size_t sk_kappa0_workspace(int64_t m, int64_t n);
int sk_kappa0_f64(const double *a, int64_t lda, int64_t m, int64_t n, double *kappa0_host, int *overflowed_host,
                  void *ws, size_t ws_bytes, sk_stream_t stream);
/* The contract's names for sk_sketch_partial (accumulate = 0), sk_level_overflow and
 * sk_residual (apply_sketch src/sketch.py:138-169, the Overflow check
 * src/solvers.py:191-193, _report src/solvers.py:99-117). */
int sk_sketch(int level, int transform, const double *a, int64_t lda, int64_t m_local, int64_t row_offset,
              int64_t m_pad, int64_t n, const double *signs, const int64_t *rows, int64_t d, double *out_partial,
              int64_t ldo, int *overflow_flag_dev, void *ws, size_t ws_bytes, sk_stream_t stream);
int sk_demote_check(const double *a, int64_t rows, int64_t cols, int64_t lda, int level, int *overflowed_host,
                    void *ws, size_t ws_bytes, sk_stream_t stream);
int sk_residual_norms(const double *a, int64_t rows, int64_t cols, int64_t lda, const double *x, const double *b,
                      double *r, double *out_host, void *ws, size_t ws_bytes, sk_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* SKLSQ_H */
