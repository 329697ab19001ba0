// The C-ABI entry points under the names of the SURVEY §8(b) contract that are
// compositions of the primitive entry points (Gram + rhs in one call, SYRK,
// kappa0 straight from A, all on the production Gram engine: INT8 Ozaki-II at
// scale, FP64 DMMA below) or the contract's names for existing primitives.
// All stream-ordered; caller-owned workspace; no allocation.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"

using namespace sk;

namespace {
size_t align256(size_t b) { return (b + 255) & ~size_t(255); }

// The production Gram engine, as the Python layer picks it (dense._gram_engine):
// the INT8 tensor-core Ozaki-II product once m n^2 >= 2^33 and n >= 128, FP64 DMMA
// below.  SK_GRAM_ENGINE=dmma|ozaki overrides (A/B and tests).
bool use_ozaki(int64_t m, int64_t n) {
    static const char *env = getenv("SK_GRAM_ENGINE");
    if (env && strcmp(env, "dmma") == 0) return false;
    if (env && strcmp(env, "ozaki") == 0) return n >= 1;
    return n >= 128 && (double)m * (double)n * (double)n >= 8589934592.0;
}

size_t stats_bytes(int64_t n) { return align256((size_t)3 * n * sizeof(double)); }

size_t gram_ws(int64_t m, int64_t n) {
    if (!use_ozaki(m, n)) return align256(sk_gram_workspace(m, n));
    return stats_bytes(n) + align256(std::max(sk_colstats_workspace(n),
                                              std::max(sk_gram_ozaki_workspace(m, n, 0),
                                                       sk_gram_ozaki_workspace(m, n, 1))));
}

// G = X^T Y (+ rhs = X^T v) on the production engine.  On the INT8 engine the column
// scan that sets X's scales forms X^T v in the same pass (as the pipeline does).
int gram_rhs(const double *x, int64_t ldx, const double *y, int64_t ldy, int64_t m, int64_t n, const double *v,
             double *g, int64_t ldg, double *rhs, void *ws, size_t ws_bytes, cudaStream_t st) {
    if (!use_ozaki(m, n)) {
        const size_t wg = align256(sk_gram_workspace(m, n));
        int rc = sk_gram_f64(x, ldx, y, ldy, m, n, g, ldg, 0, ws, wg, st);
        if (rc != SK_OK || !v) return rc;
        return sk_gemv_t_f64(x, ldx, m, n, v, rhs, 0, static_cast<uint8_t *>(ws) + wg, ws_bytes - wg, st);
    }
    double *stats = static_cast<double *>(ws);
    void *rest = static_cast<uint8_t *>(ws) + stats_bytes(n);
    const size_t rb = ws_bytes - stats_bytes(n);
    int rc = sk_colstats_f64(x, ldx, m, n, v, stats, rest, rb, st);
    if (rc != SK_OK) return rc;
    const bool syrk = x == y && ldx == ldy;
    rc = sk_gram_ozaki_ex_f64(x, ldx, y, ldy, m, n, stats, syrk ? stats : nullptr, g, ldg, rest, rb, st);
    if (rc != SK_OK || !v) return rc;
    SK_CUDA(cudaMemcpyAsync(rhs, stats + 2 * n, (size_t)n * sizeof(double), cudaMemcpyDeviceToDevice, st));
    return SK_OK;
}
}  // namespace

extern "C" {

size_t sk_gemm_tn_workspace(int64_t m, int64_t n) {
    return gram_ws(m, n) + align256(sk_gemv_t_workspace(m, n));
}

int sk_gemm_tn_f64(const double *x, int64_t ldx, const double *y, int64_t ldy, int64_t m, int64_t n,
                   const double *v, double *g, int64_t ldg, double *rhs, void *ws, size_t ws_bytes,
                   sk_stream_t stream) {
    if (!ws || ws_bytes < sk_gemm_tn_workspace(m, n) || (v && !rhs)) {
        set_error("sk_gemm_tn_f64: bad arguments or workspace");
        return SK_ERR_ARG;
    }
    return gram_rhs(x, ldx, y, ldy, m, n, v, g, ldg, rhs, ws, ws_bytes, (cudaStream_t)stream);
}

int sk_syrk_f64(const double *x, int64_t ldx, int64_t m, int64_t n, double *g, int64_t ldg, void *ws,
                size_t ws_bytes, sk_stream_t stream) {
    if (!ws || ws_bytes < gram_ws(m, n)) {
        set_error("sk_syrk_f64: workspace too small (size it with sk_gemm_tn_workspace)");
        return SK_ERR_ARG;
    }
    return gram_rhs(x, ldx, x, ldx, m, n, nullptr, g, ldg, nullptr, ws, ws_bytes, (cudaStream_t)stream);
}

size_t sk_kappa0_workspace(int64_t m, int64_t n) {
    return align256((size_t)n * n * sizeof(double)) + std::max(gram_ws(m, n), sk_nxn_workspace(n));
}

int sk_kappa0_f64(const double *a, int64_t lda, int64_t m, int64_t n, double *kappa0_host, int *overflowed_host,
                  void *ws, size_t ws_bytes, sk_stream_t stream) {
    SK_NO_DEFER("sk_kappa0_f64");
    if (!ws || ws_bytes < sk_kappa0_workspace(m, n)) {
        set_error("sk_kappa0_f64: workspace too small");
        return SK_ERR_ARG;
    }
    double *g = static_cast<double *>(ws);
    const size_t off = align256((size_t)n * n * sizeof(double));
    void *rest = static_cast<uint8_t *>(ws) + off;
    int rc = gram_rhs(a, lda, a, lda, m, n, nullptr, g, n, nullptr, rest, ws_bytes - off, (cudaStream_t)stream);
    if (rc != SK_OK) return rc;
    return sk_kappa0_from_gram(g, n, kappa0_host, overflowed_host, rest, ws_bytes - off, stream);
}

int sk_sketch(int level, int transform, const double *a, int64_t lda, int64_t m_local, int64_t row_offset,
              int64_t m_pad, int64_t n, const double *signs, const int64_t *rows, int64_t d, double *out_partial,
              int64_t ldo, int *overflow_flag_dev, void *ws, size_t ws_bytes, sk_stream_t stream) {
    return sk_sketch_partial(level, transform, a, lda, m_local, row_offset, m_pad, n, signs, rows, d, out_partial,
                             ldo, 0, overflow_flag_dev, ws, ws_bytes, stream);
}

int sk_demote_check(const double *a, int64_t rows, int64_t cols, int64_t lda, int level, int *overflowed_host,
                    void *ws, size_t ws_bytes, sk_stream_t stream) {
    SK_NO_DEFER("sk_demote_check");
    return sk_level_overflow(a, rows, cols, lda, level, overflowed_host, ws, ws_bytes, stream);
}

int sk_residual_norms(const double *a, int64_t rows, int64_t cols, int64_t lda, const double *x, const double *b,
                      double *r, double *out_host, void *ws, size_t ws_bytes, sk_stream_t stream) {
    SK_NO_DEFER("sk_residual_norms");
    return sk_residual(a, rows, cols, lda, x, b, r, out_host, ws, ws_bytes, stream);
}

}  // extern "C"
