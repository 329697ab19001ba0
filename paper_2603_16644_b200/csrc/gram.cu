// FP64 Gram products on the DMMA tensor pipe: G = X^T Y (GEMM-TN) and G = X^T X
// (SYRK, lower tiles + exact mirror), split-K over the tall dimension with a
// deterministic reduction; plus the memory-bound X^T v.
//
// Replaces the OpenBLAS dgemm/dsyrk calls of the reference:
//   a.T @ a            src/precision.py:230 (kappa0 Gram), src/solvers.py:137 (NE)
//   a_p.T @ a_p        src/solvers.py:230 (PNE)
//   a_p.T @ a          src/solvers.py:251 (HPNE)
//   b_matrix.T @ a     src/solvers.py:164 (NNE)
//   a_p.T @ b etc.     src/solvers.py:231, :251, :164 (gemv)
//
// Layout: X, Y row-major m x n (leading dims ldx, ldy).  Each K-step stages
// BK rows of X[:, i-tile] and Y[:, j-tile] in shared memory with cp.async
// (STAGES-deep ring); warps issue mma.sync m8n8k4 f64 (DMMA) from fragments read
// with a conflict-free padded layout (row pitch = 4 mod 16 doubles).
#include "common.cuh"

namespace sk {

namespace gram {

// Tile configuration, measured on B200 with tools/ab_gram.sh at 1M x 2048 (SYRK / GEMM
// TFLOP/s): 64x64 tiles, 4 warps of 32x32, BK 16, 4 stages, 3 CTAs per SM: 33.3 / 34.2
// (96% of cuBLAS DGEMM); 128x128 / 8 warps / BK 32 x 3: 30.4 / 32.7; BK 16 x 4: 30.1 /
// 32.5; 64x64 BK 8 x 6: 32.4 / 33.3.  More resident CTAs hide the DMMA / barrier
// latencies that one 8-warp CTA per SM could not.
#ifndef SK_GRAM_BK
#define SK_GRAM_BK 16
#endif
#ifndef SK_GRAM_STAGES
#define SK_GRAM_STAGES 4
#endif
#ifndef SK_GRAM_BM
#define SK_GRAM_BM 64
#define SK_GRAM_WM 32
#define SK_GRAM_WN 32
#define SK_GRAM_THREADS 128
#define SK_GRAM_MINB 3
#endif
constexpr int BM = SK_GRAM_BM, BN = SK_GRAM_BM, BK = SK_GRAM_BK, WM = SK_GRAM_WM, WN = SK_GRAM_WN,
              STAGES = SK_GRAM_STAGES;
constexpr int THREADS = SK_GRAM_THREADS;
constexpr int PITCH = BM + 4;  // doubles; 132 = 4 (mod 16) -> conflict-free fragment loads
constexpr size_t SMEM = size_t(STAGES) * BK * PITCH * 2 * sizeof(double);

template <bool VEC16>
__device__ __forceinline__ void load_stage(double *xs, double *ys, const double *__restrict__ x,
                                           int64_t ldx, const double *__restrict__ y, int64_t ldy,
                                           int64_t k0, int64_t kend, int i0, int j0, int n) {
    const int tid = threadIdx.x;
    if (VEC16) {
        // BK rows x BM/2 16-byte chunks per operand
        constexpr int CH = BK * (BM / 2);
#pragma unroll
        for (int c = tid; c < CH; c += THREADS) {
            const int r = c / (BM / 2);
            const int cc = (c % (BM / 2)) * 2;
            const int64_t k = k0 + r;
            const bool krow = k < kend;
            {
                const int col = i0 + cc;
                int bytes = krow ? (n - col) * 8 : 0;
                bytes = bytes < 0 ? 0 : (bytes > 16 ? 16 : bytes);
                const double *src = bytes ? x + k * ldx + col : x;
                cp_async16(xs + r * PITCH + cc, src, bytes);
            }
            {
                const int col = j0 + cc;
                int bytes = krow ? (n - col) * 8 : 0;
                bytes = bytes < 0 ? 0 : (bytes > 16 ? 16 : bytes);
                const double *src = bytes ? y + k * ldy + col : y;
                cp_async16(ys + r * PITCH + cc, src, bytes);
            }
        }
    } else {
        constexpr int CH = BK * BM;
        for (int c = tid; c < CH; c += THREADS) {
            const int r = c / BM;
            const int cc = c % BM;
            const int64_t k = k0 + r;
            const bool krow = k < kend;
            {
                const int col = i0 + cc;
                const int bytes = (krow && col < n) ? 8 : 0;
                cp_async8(xs + r * PITCH + cc, bytes ? x + k * ldx + col : x, bytes);
            }
            {
                const int col = j0 + cc;
                const int bytes = (krow && col < n) ? 8 : 0;
                cp_async8(ys + r * PITCH + cc, bytes ? y + k * ldy + col : y, bytes);
            }
        }
    }
}

// One work unit = (tile, split).  unit = split * ntiles + tile so that CTAs that
// are resident together share a K range (L2 reuse of the X/Y row block).
template <bool VEC16, bool SYRK>
__global__ void __launch_bounds__(THREADS, SK_GRAM_MINB)
gram_tn_kernel(const double *__restrict__ x, int64_t ldx, const double *__restrict__ y, int64_t ldy,
               int64_t m, int n, int ntn, int ntiles, int64_t kchunk, double *__restrict__ part, const int *gate) {
    if (gate && *gate == 0) return;   // gated fallback (deferred verdicts): run only when flagged
    extern __shared__ __align__(16) double smem[];
    double *xs_base = smem;
    double *ys_base = smem + STAGES * BK * PITCH;

    const int unit = blockIdx.x;
    const int tile = unit % ntiles;
    const int split = unit / ntiles;
    int ti, tj;
    if (SYRK) {  // lower-triangular tile index -> (ti, tj), tj <= ti
        ti = (int)((sqrt(8.0 * tile + 1.0) - 1.0) * 0.5);
        while ((ti + 1) * (ti + 2) / 2 <= tile) ++ti;
        while (ti * (ti + 1) / 2 > tile) --ti;
        tj = tile - ti * (ti + 1) / 2;
    } else {
        ti = tile / ntn;
        tj = tile % ntn;
    }
    const int i0 = ti * BM, j0 = tj * BN;
    const int64_t kbeg = split * kchunk;
    const int64_t kend = min(m, kbeg + kchunk);
    const int nk = kend > kbeg ? (int)((kend - kbeg + BK - 1) / BK) : 0;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    const int wm = warp % (BM / WM), wn = warp / (BM / WM);

    double acc[WM / 8][WN / 8][2];
#pragma unroll
    for (int a = 0; a < WM / 8; ++a)
#pragma unroll
        for (int b = 0; b < WN / 8; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

    // prologue
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
        if (s < nk)
            load_stage<VEC16>(xs_base + s * BK * PITCH, ys_base + s * BK * PITCH, x, ldx, y, ldy,
                              kbeg + (int64_t)s * BK, kend, i0, j0, n);
        cp_async_commit();
    }

    for (int kt = 0; kt < nk; ++kt) {
        cp_async_wait<STAGES - 2>();
        __syncthreads();
        {
            const int nxt = kt + STAGES - 1;
            if (nxt < nk) {
                const int s = nxt % STAGES;
                load_stage<VEC16>(xs_base + s * BK * PITCH, ys_base + s * BK * PITCH, x, ldx, y,
                                  ldy, kbeg + (int64_t)nxt * BK, kend, i0, j0, n);
            }
            cp_async_commit();
        }
        const double *xs = xs_base + (kt % STAGES) * BK * PITCH;
        const double *ys = ys_base + (kt % STAGES) * BK * PITCH;
#pragma unroll
        for (int kk = 0; kk < BK; kk += 4) {
            double af[WM / 8], bf[WN / 8];
            const double *xr = xs + (kk + t) * PITCH + wm * WM + g;
            const double *yr = ys + (kk + t) * PITCH + wn * WN + g;
#pragma unroll
            for (int a = 0; a < WM / 8; ++a) af[a] = xr[a * 8];
#pragma unroll
            for (int b = 0; b < WN / 8; ++b) bf[b] = yr[b * 8];
#pragma unroll
            for (int a = 0; a < WM / 8; ++a)
#pragma unroll
                for (int b = 0; b < WN / 8; ++b) dmma884(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
        }
    }
    cp_async_wait<0>();

    double *out = part + ((size_t)split * ntiles + tile) * (BM * BN);
#pragma unroll
    for (int a = 0; a < WM / 8; ++a)
#pragma unroll
        for (int b = 0; b < WN / 8; ++b) {
            const int r = wm * WM + a * 8 + g;
            const int c = wn * WN + b * 8 + 2 * t;
            *reinterpret_cast<double2 *>(out + r * BN + c) = make_double2(acc[a][b][0], acc[a][b][1]);
        }
}

// G[i][j] (+)= sum_s part[s][tile(i,j)][li][lj]; SYRK reads the lower tile for both
// halves so the result is exactly symmetric.
template <bool SYRK>
__global__ void gram_reduce_kernel(const double *__restrict__ part, int splits, int ntiles, int ntn,
                                   int n, double *__restrict__ gout, int64_t ldg, int accumulate, const int *gate) {
    if (gate && *gate == 0) return;
    const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= (int64_t)n * n) return;
    int i = (int)(idx / n), j = (int)(idx % n);
    int si = i, sj = j;
    if (SYRK && j > i) { si = j; sj = i; }
    const int ti = si / BM, tj = sj / BN;
    const int tile = SYRK ? ti * (ti + 1) / 2 + tj : ti * ntn + tj;
    const double *p = part + (size_t)tile * (BM * BN) + (si % BM) * BN + (sj % BN);
    double s = 0.0;
    for (int k = 0; k < splits; ++k) s += p[(size_t)k * ntiles * (BM * BN)];
    double *o = gout + (int64_t)i * ldg + j;
    *o = accumulate ? *o + s : s;
}

struct Plan {
    int ntn, ntiles, splits;
    int64_t kchunk;
};

static Plan make_plan(int64_t m, int64_t n, bool syrk) {
    Plan p;
    p.ntn = (int)((n + BN - 1) / BN);
    p.ntiles = syrk ? p.ntn * (p.ntn + 1) / 2 : p.ntn * p.ntn;
    const int sms = sm_count();
    // rows per split: GEMM-TN >= 128 (8 BK steps), so a short m still spreads over the SMs
    // (config 1's A_p^T A: 54 -> 9 us); SYRK >= 1024 (its summation order is what the
    // NotPositiveDefinite cases of the reference's tests were pinned with)
    const int64_t min_chunk = syrk ? 1024 : 128;
    int64_t smax = (m + min_chunk - 1) / min_chunk;
    if (smax < 1) smax = 1;
    // ~16 waves of resident CTAs; among nearby split counts pick the one whose last
    // wave is fullest (units = tiles x splits spread over sms x SK_GRAM_MINB slots)
    const int64_t slots = (int64_t)sms * SK_GRAM_MINB;
    int64_t target = 16 * slots / p.ntiles;
    if (target < 1) target = 1;
    if (target > smax) target = smax;
    int64_t best = target;
    double best_fill = -1.0;
    for (int64_t s = std::max<int64_t>(1, target / 2); s <= std::min<int64_t>(smax, 2 * target); ++s) {
        const int64_t units = (int64_t)p.ntiles * s;
        const int64_t waves = (units + slots - 1) / slots;
        const double fill = (double)units / (double)(waves * slots);
        if (fill > best_fill + 1e-9 || (fill > best_fill - 1e-9 && s > best)) { best_fill = fill; best = s; }
    }
    p.splits = (int)best;
    p.kchunk = (m + p.splits - 1) / p.splits;
    p.kchunk = (p.kchunk + BK - 1) / BK * BK;
    p.splits = (int)((m + p.kchunk - 1) / p.kchunk);
    if (p.splits < 1) p.splits = 1;
    return p;
}

static size_t ws_bytes_for(int64_t m, int64_t n, bool syrk) {
    Plan p = make_plan(m, n, syrk);
    return (size_t)p.splits * p.ntiles * BM * BN * sizeof(double);
}

}  // namespace gram

// ---------------------------------------------------------------- GEMV-T ---
namespace gemvt {
constexpr int THREADS = 256;
__global__ void __launch_bounds__(THREADS)
gemv_t_kernel(const double *__restrict__ x, int64_t ldx, int64_t m, int n, const double *__restrict__ v,
              int64_t kchunk, double *__restrict__ part) {
    const int j = blockIdx.x * THREADS + threadIdx.x;
    const int split = blockIdx.y;
    const int64_t k0 = split * kchunk, k1 = min(m, k0 + kchunk);
    double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
    if (j < n) {
        int64_t k = k0;
        for (; k + 4 <= k1; k += 4) {
            s0 += x[k * ldx + j] * v[k];
            s1 += x[(k + 1) * ldx + j] * v[k + 1];
            s2 += x[(k + 2) * ldx + j] * v[k + 2];
            s3 += x[(k + 3) * ldx + j] * v[k + 3];
        }
        for (; k < k1; ++k) s0 += x[k * ldx + j] * v[k];
        part[(size_t)split * n + j] = (s0 + s1) + (s2 + s3);
    }
}
__global__ void gemv_t_reduce(const double *__restrict__ part, int splits, int n, double *out, int accumulate) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    double s = 0;
    for (int k = 0; k < splits; ++k) s += part[(size_t)k * n + j];
    out[j] = accumulate ? out[j] + s : s;
}
static int splits_for(int64_t m, int64_t n) {
    const int cols = (int)((n + THREADS - 1) / THREADS);
    int64_t s = (int64_t)4 * sm_count() / cols;
    int64_t smax = (m + 4095) / 4096;
    if (smax < 16) smax = std::min<int64_t>(16, (m + 63) / 64);   // short m: >= 64 rows per split, not one CTA
    if (s > smax) s = smax;
    if (s < 1) s = 1;
    return (int)s;
}
}  // namespace gemvt

}  // namespace sk

using namespace sk;

namespace sk {
namespace gram {
int gram_f64_gated(const double *x, int64_t ldx, const double *y, int64_t ldy, int64_t m, int64_t n, double *g,
                   int64_t ldg, int accumulate, void *ws, size_t ws_bytes, sk_stream_t stream, const int *gate);
}  // namespace gram
}  // namespace sk

extern "C" {

size_t sk_gram_workspace(int64_t m, int64_t n) {
    size_t a = gram::ws_bytes_for(m, n, false), b = gram::ws_bytes_for(m, n, true);
    return a > b ? a : b;
}

int sk_gram_f64(const double *x, int64_t ldx, const double *y, int64_t ldy, int64_t m, int64_t n,
                double *g, int64_t ldg, int accumulate, void *ws, size_t ws_bytes, sk_stream_t stream) {
    return sk::gram::gram_f64_gated(x, ldx, y, ldy, m, n, g, ldg, accumulate, ws, ws_bytes, stream, nullptr);
}

}  // extern "C"

namespace sk {
namespace gram {
// sk_gram_f64 whose kernels run only when *gate != 0 (gate == nullptr: always): the
// stream-ordered DMMA fallback of the INT8 Gram under deferred verdicts
int gram_f64_gated(const double *x, int64_t ldx, const double *y, int64_t ldy, int64_t m, int64_t n, double *g,
                   int64_t ldg, int accumulate, void *ws, size_t ws_bytes, sk_stream_t stream, const int *gate) {
    if (!x || !y || !g || m < 0 || n <= 0 || ldx < n || ldy < n || ldg < n || n > (1 << 20)) {
        set_error("sk_gram_f64: bad arguments");
        return SK_ERR_ARG;
    }
    const bool syrk = (x == y) && (ldx == ldy);
    gram::Plan p = gram::make_plan(m, n, syrk);
    const size_t need = (size_t)p.splits * p.ntiles * gram::BM * gram::BN * sizeof(double);
    if (ws_bytes < need || !ws) {
        set_error("sk_gram_f64: workspace %zu < %zu", ws_bytes, need);
        return SK_ERR_ARG;
    }
    cudaStream_t st = (cudaStream_t)stream;
    const bool vec = ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) % 16 == 0) &&
                     (ldx % 2 == 0) && (ldy % 2 == 0);
    double *part = static_cast<double *>(ws);
    const int units = p.ntiles * p.splits;
    if (m == 0) {
        SK_CUDA(cudaMemsetAsync(part, 0, (size_t)p.ntiles * gram::BM * gram::BN * sizeof(double), st));
        p.splits = 1;
    } else {
#define SK_GRAM_LAUNCH(V, S)                                                                       \
    do {                                                                                           \
        auto kfn = gram::gram_tn_kernel<V, S>;                                                     \
        SK_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gram::SMEM)); \
        kfn<<<units, gram::THREADS, gram::SMEM, st>>>(x, ldx, y, ldy, m, (int)n, p.ntn, p.ntiles, \
                                                      p.kchunk, part, gate);                       \
    } while (0)
        if (vec && syrk) SK_GRAM_LAUNCH(true, true);
        else if (vec) SK_GRAM_LAUNCH(true, false);
        else if (syrk) SK_GRAM_LAUNCH(false, true);
        else SK_GRAM_LAUNCH(false, false);
#undef SK_GRAM_LAUNCH
        SK_LAUNCH_CHECK("gram_tn_kernel");
    }
    const int64_t total = n * n;
    const int rb = 256;
    const unsigned rg = (unsigned)((total + rb - 1) / rb);
    if (syrk)
        gram::gram_reduce_kernel<true><<<rg, rb, 0, st>>>(part, p.splits, p.ntiles, p.ntn, (int)n, g, ldg, accumulate,
                                                            gate);
    else
        gram::gram_reduce_kernel<false><<<rg, rb, 0, st>>>(part, p.splits, p.ntiles, p.ntn, (int)n, g, ldg, accumulate,
                                                             gate);
    SK_LAUNCH_CHECK("gram_reduce_kernel");
    return SK_OK;
}
}  // namespace gram
}  // namespace sk

extern "C" {

size_t sk_gemv_t_workspace(int64_t m, int64_t n) {
    return (size_t)gemvt::splits_for(m, n) * (size_t)n * sizeof(double);
}

int sk_gemv_t_f64(const double *x, int64_t ldx, int64_t m, int64_t n, const double *v, double *out,
                  int accumulate, void *ws, size_t ws_bytes, sk_stream_t stream) {
    if (!x || !v || !out || m < 0 || n <= 0 || ldx < n) {
        set_error("sk_gemv_t_f64: bad arguments");
        return SK_ERR_ARG;
    }
    const int splits = gemvt::splits_for(m, n);
    if (ws_bytes < (size_t)splits * n * sizeof(double) || !ws) {
        set_error("sk_gemv_t_f64: workspace too small");
        return SK_ERR_ARG;
    }
    cudaStream_t st = (cudaStream_t)stream;
    double *part = static_cast<double *>(ws);
    const int64_t kchunk = (m + splits - 1) / splits;
    dim3 grid((unsigned)((n + gemvt::THREADS - 1) / gemvt::THREADS), (unsigned)splits);
    gemvt::gemv_t_kernel<<<grid, gemvt::THREADS, 0, st>>>(x, ldx, m, (int)n, v, kchunk > 0 ? kchunk : 1, part);
    SK_LAUNCH_CHECK("gemv_t_kernel");
    gemvt::gemv_t_reduce<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(part, splits, (int)n, out, accumulate);
    SK_LAUNCH_CHECK("gemv_t_reduce");
    return SK_OK;
}

}  // extern "C"
