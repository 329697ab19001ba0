// HBM-bound passes over the tall matrix: validation + promotion + Frobenius norm,
// the level-overflow test of the demotion, and the residual r = A x - b.
//
//   _as_matrix / _check_system   src/dense.py:57-65, src/solvers.py:87-96
//   np.linalg.norm(a)            src/solvers.py:102
//   round_to_precision(...).overflowed   src/precision.py:90-103 (src/solvers.py:191-193)
//   _report: a @ x_hat - b, norms        src/solvers.py:99-117
// Each is one streaming read of A (8 m n bytes) with 16-byte vector loads and a
// grid sized to a multiple of the SM count; partial sums go to a small
// per-block buffer reduced in a fixed order (deterministic).
#include "common.cuh"

namespace sk {
namespace streamk {

constexpr int THREADS = 256;

__device__ __forceinline__ double load_as_f64(const void *p, int dtype, int64_t idx) {
    if (dtype == SK_F64) return static_cast<const double *>(p)[idx];
    if (dtype == SK_F32) return (double)static_cast<const float *>(p)[idx];
    return (double)__half2float(static_cast<const __half *>(p)[idx]);
}

// per block: [0] non-finite count, [1] sum of squares
__global__ void __launch_bounds__(THREADS)
cast_stats_kernel(const void *src, int dtype, int64_t rows, int64_t cols, int64_t lds, double *dst, int64_t ldd,
                  double *part) {
    double nf = 0.0, ss = 0.0;
    const int64_t total = rows * cols;
    if (dtype == SK_F64 && cols == lds && (dst == nullptr || cols == ldd) && (cols % 2 == 0) &&
        (reinterpret_cast<uintptr_t>(src) % 16 == 0) && (reinterpret_cast<uintptr_t>(dst) % 16 == 0)) {
        const double2 *s2 = static_cast<const double2 *>(src);
        double2 *d2 = reinterpret_cast<double2 *>(dst);
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total / 2;
             i += (int64_t)gridDim.x * blockDim.x) {
            const double2 v = s2[i];
            nf += (!isfinite(v.x)) + (!isfinite(v.y));
            ss += v.x * v.x + v.y * v.y;
            if (d2 && d2 != s2) d2[i] = v;
        }
    } else {
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
             i += (int64_t)gridDim.x * blockDim.x) {
            const int64_t r = i / cols, c = i % cols;
            const double v = load_as_f64(src, dtype, r * lds + c);
            nf += !isfinite(v);
            ss += v * v;
            if (dst) dst[r * ldd + c] = v;
        }
    }
    __shared__ double s0[THREADS / 32], s1[THREADS / 32];
    nf = warp_sum(nf);
    ss = warp_sum(ss);
    if ((threadIdx.x & 31) == 0) { s0[threadIdx.x >> 5] = nf; s1[threadIdx.x >> 5] = ss; }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0, b = 0;
        for (int k = 0; k < THREADS / 32; ++k) { a += s0[k]; b += s1[k]; }
        part[2 * blockIdx.x] = a;
        part[2 * blockIdx.x + 1] = b;
    }
}

__global__ void sum_parts(const double *part, int nblocks, int width, double *out) {
    // fixed-order reduction by one warp per output slot
    const int slot = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (slot >= width) return;
    double s = 0.0;
    for (int b = lane; b < nblocks; b += 32) s += part[(int64_t)b * width + slot];
    s = warp_sum(s);
    if (lane == 0) out[slot] = s;
}

// out[slot] += fixed-order sum of the per-block partials (streamed chunks accumulate)
__global__ void accumulate_parts(const double *part, int nblocks, int width, double *out) {
    const int slot = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (slot >= width) return;
    double s = 0.0;
    for (int b = lane; b < nblocks; b += 32) s += part[(int64_t)b * width + slot];
    s = warp_sum(s);
    if (lane == 0) out[slot] += s;
}

template <int LEVEL>
__global__ void __launch_bounds__(THREADS)
overflow_kernel(const double *a, int64_t rows, int64_t cols, int64_t lda, int *flag) {
    int over = 0;
    const int64_t total = rows * cols;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const double v = a[(i / cols) * lda + (i % cols)];
        double w;
        if (LEVEL == 16) w = (double)__half2float(__double2half(v));
        else w = (double)__double2float_rn(v);
        over |= (isinf(w) && isfinite(v));
    }
    if (__any_sync(0xffffffffu, over) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

// r = A x - b, one warp per row chunk: part[2*block] = sum r^2
__global__ void __launch_bounds__(THREADS)
residual_kernel(const double *__restrict__ a, int64_t rows, int64_t cols, int64_t lda, const double *__restrict__ x,
                const double *__restrict__ b, double *__restrict__ r, double *part) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t gw = blockIdx.x * (int64_t)(THREADS / 32) + warp;
    const int64_t nw = (int64_t)gridDim.x * (THREADS / 32);
    double ss = 0.0;
    const bool vec = ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(x)) % 16 == 0) && (lda % 2 == 0);
    for (int64_t i = gw; i < rows; i += nw) {
        const double *row = a + i * lda;
        double s = 0.0;
        if (vec) {
            // 16-byte loads, four independent chains: 2 KB of the row in flight per warp
            const double2 *r2 = reinterpret_cast<const double2 *>(row);
            const double2 *x2 = reinterpret_cast<const double2 *>(x);
            const int64_t n2 = cols / 2;
            double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
            int64_t c = lane;
            for (; c + 96 < n2; c += 128) {
                const double2 a0 = __ldcs(r2 + c), a1 = __ldcs(r2 + c + 32), a2 = __ldcs(r2 + c + 64),
                              a3 = __ldcs(r2 + c + 96);
                const double2 y0 = __ldg(x2 + c), y1 = __ldg(x2 + c + 32), y2 = __ldg(x2 + c + 64),
                              y3 = __ldg(x2 + c + 96);
                s0 = fma(a0.y, y0.y, fma(a0.x, y0.x, s0));
                s1 = fma(a1.y, y1.y, fma(a1.x, y1.x, s1));
                s2 = fma(a2.y, y2.y, fma(a2.x, y2.x, s2));
                s3 = fma(a3.y, y3.y, fma(a3.x, y3.x, s3));
            }
            for (; c < n2; c += 32) {
                const double2 a0 = __ldcs(r2 + c), y0 = __ldg(x2 + c);
                s0 = fma(a0.y, y0.y, fma(a0.x, y0.x, s0));
            }
            if ((cols & 1) && lane == 0) s1 = fma(row[cols - 1], x[cols - 1], s1);
            s = (s0 + s1) + (s2 + s3);
        } else {
            for (int64_t c = lane; c < cols; c += 32) s += row[c] * x[c];
        }
        s = warp_sum(s);
        const double ri = s - b[i];
        if (lane == 0) {
            if (r) r[i] = ri;
            ss += ri * ri;
        }
    }
    __shared__ double sh[THREADS / 32];
    if (lane == 0) sh[warp] = ss;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0;
        for (int k = 0; k < THREADS / 32; ++k) t += sh[k];
        part[2 * blockIdx.x] = t;
        part[2 * blockIdx.x + 1] = 0.0;
    }
}

__global__ void sumsq_vec(const double *x, int64_t n, double *out) {
    double s = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += x[i] * x[i];
    s = warp_sum(s);
    __shared__ double sh[32];
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0;
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t += sh[k];
        *out = t;
    }
}

static int blocks_for(int64_t elems) {
    int64_t b = (elems + THREADS * 8 - 1) / (THREADS * 8);
    const int64_t cap = (int64_t)8 * sm_count();
    if (b > cap) b = cap;
    if (b < 1) b = 1;
    return (int)b;
}

}  // namespace streamk
}  // namespace sk

using namespace sk;
using namespace sk::streamk;

extern "C" {

size_t sk_matrix_stats_workspace(int64_t rows, int64_t cols) {
    (void)rows;
    (void)cols;
    return (size_t)(8 * 1024) * 2 * sizeof(double) + 4096;
}

int sk_cast_stats(const void *src, int src_dtype, int64_t rows, int64_t cols, int64_t ld_src, double *dst,
                  int64_t ld_dst, double *stats_host, void *ws, size_t ws_bytes, sk_stream_t stream) {
    SK_NO_DEFER("sk_cast_stats");
    if (!src || !stats_host || rows < 0 || cols <= 0 || ld_src < cols || (dst && ld_dst < cols) || !ws ||
        ws_bytes < sk_matrix_stats_workspace(rows, cols) ||
        (src_dtype != SK_F16 && src_dtype != SK_F32 && src_dtype != SK_F64)) {
        set_error("sk_cast_stats: bad arguments");
        return SK_ERR_ARG;
    }
    cudaStream_t st = (cudaStream_t)stream;
    const int nb = blocks_for(rows * cols);
    double *part = static_cast<double *>(ws);
    double *out = part + 2 * 8 * 1024;
    cast_stats_kernel<<<nb, THREADS, 0, st>>>(src, src_dtype, rows, cols, ld_src, dst, ld_dst, part);
    SK_LAUNCH_CHECK("cast_stats_kernel");
    sum_parts<<<1, 64, 0, st>>>(part, nb, 2, out);
    SK_LAUNCH_CHECK("sum_parts");
    SK_CUDA(cudaMemcpyAsync(stats_host, out, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
    SK_CUDA(cudaStreamSynchronize(st));
    return SK_OK;
}

int sk_cast_stats_async(const void *src, int src_dtype, int64_t rows, int64_t cols, int64_t ld_src, double *dst,
                        int64_t ld_dst, double *stats_dev, void *ws, size_t ws_bytes, sk_stream_t stream) {
    if (!src || !stats_dev || rows < 0 || cols <= 0 || ld_src < cols || (dst && ld_dst < cols) || !ws ||
        ws_bytes < sk_matrix_stats_workspace(rows, cols) ||
        (src_dtype != SK_F16 && src_dtype != SK_F32 && src_dtype != SK_F64)) {
        set_error("sk_cast_stats_async: bad arguments");
        return SK_ERR_ARG;
    }
    if (rows == 0) return SK_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const int nb = blocks_for(rows * cols);
    double *part = static_cast<double *>(ws);
    cast_stats_kernel<<<nb, THREADS, 0, st>>>(src, src_dtype, rows, cols, ld_src, dst, ld_dst, part);
    SK_LAUNCH_CHECK("cast_stats_kernel");
    accumulate_parts<<<1, 64, 0, st>>>(part, nb, 2, stats_dev);
    SK_LAUNCH_CHECK("accumulate_parts");
    return SK_OK;
}

int sk_level_overflow(const double *a, int64_t rows, int64_t cols, int64_t lda, int level, int *overflowed_host,
                      void *ws, size_t ws_bytes, sk_stream_t stream) {
    SK_NO_DEFER("sk_level_overflow");
    if (!a || !overflowed_host || rows < 0 || cols <= 0 || lda < cols || !ws || ws_bytes < sizeof(int)) {
        set_error("sk_level_overflow: bad arguments");
        return SK_ERR_ARG;
    }
    *overflowed_host = 0;
    if (level == 64 || rows == 0) return SK_OK;   // rounding to binary64 is the identity
    cudaStream_t st = (cudaStream_t)stream;
    int *flag = static_cast<int *>(ws);
    SK_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), st));
    const int nb = blocks_for(rows * cols);
    if (level == 16) overflow_kernel<16><<<nb, THREADS, 0, st>>>(a, rows, cols, lda, flag);
    else if (level == 32) overflow_kernel<32><<<nb, THREADS, 0, st>>>(a, rows, cols, lda, flag);
    else { set_error("bad level"); return SK_ERR_ARG; }
    SK_LAUNCH_CHECK("overflow_kernel");
    SK_CUDA(cudaMemcpyAsync(overflowed_host, flag, sizeof(int), cudaMemcpyDeviceToHost, st));
    SK_CUDA(cudaStreamSynchronize(st));
    return SK_OK;
}

int sk_residual(const double *a, int64_t rows, int64_t cols, int64_t lda, const double *x, const double *b, double *r,
                double *out_host, void *ws, size_t ws_bytes, sk_stream_t stream) {
    SK_NO_DEFER("sk_residual");
    if (!a || !x || !b || !out_host || rows < 0 || cols <= 0 || lda < cols || !ws ||
        ws_bytes < sk_matrix_stats_workspace(rows, cols)) {
        set_error("sk_residual: bad arguments");
        return SK_ERR_ARG;
    }
    cudaStream_t st = (cudaStream_t)stream;
    double *part = static_cast<double *>(ws);
    double *out = part + 2 * 8 * 1024;
    int64_t nb = (rows + 7) / 8;
    const int64_t cap = (int64_t)8 * sm_count();
    if (nb > cap) nb = cap;
    if (nb < 1) nb = 1;
    residual_kernel<<<(unsigned)nb, THREADS, 0, st>>>(a, rows, cols, lda, x, b, r, part);
    SK_LAUNCH_CHECK("residual_kernel");
    sum_parts<<<1, 64, 0, st>>>(part, (int)nb, 2, out);
    SK_LAUNCH_CHECK("sum_parts");
    sumsq_vec<<<1, 256, 0, st>>>(x, cols, out + 1);
    SK_LAUNCH_CHECK("sumsq_vec");
    SK_CUDA(cudaMemcpyAsync(out_host, out, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
    SK_CUDA(cudaStreamSynchronize(st));
    return SK_OK;
}

int sk_residual_async(const double *a, int64_t rows, int64_t cols, int64_t lda, const double *x, const double *b,
                      double *r, double *out_dev, void *ws, size_t ws_bytes, sk_stream_t stream) {
    if (!a || !x || !b || !out_dev || rows < 0 || cols <= 0 || lda < cols || !ws ||
        ws_bytes < sk_matrix_stats_workspace(rows, cols)) {
        set_error("sk_residual_async: bad arguments");
        return SK_ERR_ARG;
    }
    cudaStream_t st = (cudaStream_t)stream;
    double *part = static_cast<double *>(ws);
    int64_t nb = (rows + 7) / 8;
    const int64_t cap = (int64_t)8 * sm_count();
    if (nb > cap) nb = cap;
    if (nb < 1) nb = 1;
    residual_kernel<<<(unsigned)nb, THREADS, 0, st>>>(a, rows, cols, lda, x, b, r, part);
    SK_LAUNCH_CHECK("residual_kernel");
    sum_parts<<<1, 64, 0, st>>>(part, (int)nb, 2, out_dev);
    SK_LAUNCH_CHECK("sum_parts");
    sumsq_vec<<<1, 256, 0, st>>>(x, cols, out_dev + 1);
    SK_LAUNCH_CHECK("sumsq_vec");
    return SK_OK;
}

}  // extern "C"
