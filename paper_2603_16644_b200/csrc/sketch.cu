// SRTT sketch  A_s = sqrt(m_pad/d) * S F D * A_level  (src/sketch.py:138-169).
//
// The reference demotes A to the level (src/solvers.py:191-193), flips row signs,
// runs a full length-m orthonormal DCT-II (pocketfft) or Walsh-Hadamard transform
// along the rows, keeps the d sampled output rows and scales them.  Only d of the
// m transform outputs are ever used, so here the sampled rows of the transform
// are formed directly as a GEMM against the closed-form operator
//     F_dct[r, j] = c_r cos(pi r (2j+1) / (2M)),   F_wht[r, j] = (-1)^popc(r & j) / sqrt(M)
// generated on the fly in shared memory, with the signs folded into the demoted
// A tile.  This v1 kernel runs on the FP64 DMMA pipe for every level (the exact
// product is then rounded to the level in sk_sketch_finalize, matching the
// reference's "transform in working precision, round" to within the level's
// unit roundoff).  Row shards pass their global row_offset, so partial sketches
// of contiguous row blocks sum (NCCL allreduce) to the global sketch.
//
// DCT phases are exact: p = r (2j+1) mod 4M in integer arithmetic, then
// sincospi(p / 2M); within a 16-wide K block the angle advances by a per-row
// rotation e^{i t pi r / M} computed the same way, so every Omega entry is a
// product of two correctly-reduced unit complex numbers (~2 ulp).
#include "common.cuh"

namespace sk {
namespace sketch {

constexpr int BM = 128, BN = 128, BK = 16, THREADS = 512, WM = 32, WN = 32;   // 16 warps of 32 x 32
#ifndef SK_OMEGA_ANCHOR
#define SK_OMEGA_ANCHOR 16   // k-steps between exact operator phases (1: exact every step)
#endif
constexpr int APITCH = BK + 4;   // Omega tile [i][k], 20 = 4 (mod 16)
constexpr int BPITCH = BN + 4;   // A tile [k][c], 132 = 4 (mod 16)
constexpr size_t SMEM = sizeof(double) * (2 * BM * APITCH + 2 * BK * BPITCH + 2 * BM * BK);

template <int LEVEL>
__device__ __forceinline__ double demote(double v, int &over) {
    double w;
    if (LEVEL == 16) w = (double)__half2float(__double2half(v));
    else if (LEVEL == 32) w = (double)__double2float_rn(v);
    else w = v;
    over |= (isinf(w) && isfinite(v)) ? 1 : 0;
    return w;
}

template <int LEVEL, int TRANSFORM>
__global__ void __launch_bounds__(THREADS, 1)
sketch_kernel(const double *__restrict__ a, int64_t lda, int64_t m_local, int64_t row_offset,
              int64_t mpad, int n, const double *__restrict__ signs, const int64_t *__restrict__ rows,
              int d, int ntn, int ntiles, int64_t kchunk, double *__restrict__ part, int *overflow_flag) {
    extern __shared__ __align__(16) double smem[];
    double *om = smem;                          // [2][BM][APITCH]
    double *bt = om + 2 * BM * APITCH;          // [2][BK][BPITCH]
    double *rot = bt + 2 * BK * BPITCH;         // [BM][BK] (cos) + [BM][BK] (sin) -> per-row step rotations

    const int unit = blockIdx.x;
    const int tile = unit % ntiles, split = unit / ntiles;
    const int ti = tile / ntn, tj = tile % ntn;
    const int i0 = ti * BM, c0 = tj * BN;
    const int64_t kbeg = split * kchunk;
    const int64_t kend = min(m_local, kbeg + kchunk);
    const int nk = kend > kbeg ? (int)((kend - kbeg + BK - 1) / BK) : 0;

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
    const int wm = warp % (BM / WM), wn = warp / (BM / WM);

    // Omega generator role: thread -> (row gi = tid/4, k quarter = tid%4 -> 4 columns)
    constexpr int GC = BM * BK / THREADS;   // generated columns per thread (4)
    const int gi = tid / (BK / GC), gh = tid % (BK / GC);
    const bool grow_ok = (i0 + gi) < d;
    const int64_t rr = grow_ok ? rows[i0 + gi] : 0;
    const double M = (double)mpad;
    const int64_t fourM = 4 * mpad;
    const double cr = (rr == 0) ? sqrt(1.0 / M) : sqrt(2.0 / M);
    double rc[GC], rs[GC];   // e^{i (gh*GC + u) pi r / M}, u < GC, relative to the block base
    if (TRANSFORM == SK_DCT2) {
#pragma unroll
        for (int u = 0; u < GC; ++u) {
            const int64_t q = (int64_t)(((uint64_t)rr * (uint64_t)(2 * u)) % (uint64_t)fourM);
            sincospi((double)q / (2.0 * M), &rs[u], &rc[u]);
        }
    }
    (void)rot;
    int over = 0;
    // block base phase e^{i pi p / 2M}, p = rr (2 jg0 + 1) mod 4M: exact (sincospi of the
    // exactly reduced integer phase) every SK_OMEGA_ANCHOR k-steps, advanced in between by
    // the fixed rotation of one k-step (p += 2 BK rr): the per-step 64-bit modular products
    // and FP64 sincospi dominated the kernel's instruction stream (ncu: DMMA 17% of the
    // instructions at config-2 shape); the rotation adds <= SK_OMEGA_ANCHOR roundings
    const uint64_t f1 = (uint64_t)rr % (uint64_t)fourM;
    const uint64_t dstep = (f1 * (uint64_t)(2 * BK)) % (uint64_t)fourM;
    double c_step = 1.0, s_step = 0.0;
    if (TRANSFORM == SK_DCT2) sincospi((double)dstep / (2.0 * M), &s_step, &c_step);
    double cb_cur = 1.0, sb_cur = 0.0;
    int gen_count = 0;

    auto gen_omega = [&](double *dst, int64_t kb) {
        // columns kb + gh*8 + u (local rows of A), global jg = row_offset + local
        const int64_t jl0 = kb + gh * GC;
        if (TRANSFORM == SK_DCT2) {
            double sb, cb;
            if (gen_count % SK_OMEGA_ANCHOR == 0) {
                const int64_t jg0 = row_offset + jl0;
                // both factors < 4M < 2^32, so the product fits in 64 bits
                const uint64_t f2 = (uint64_t)(2 * jg0 + 1) % (uint64_t)fourM;
                const int64_t p = (int64_t)((f1 * f2) % (uint64_t)fourM);
                sincospi((double)p / (2.0 * M), &sb, &cb);
            } else {
                cb = cb_cur * c_step - sb_cur * s_step;
                sb = sb_cur * c_step + cb_cur * s_step;
            }
            cb_cur = cb;
            sb_cur = sb;
            ++gen_count;
#pragma unroll
            for (int u = 0; u < GC; ++u) {
                double v = cr * (cb * rc[u] - sb * rs[u]);
                if (!grow_ok || jl0 + u >= kend) v = 0.0;
                dst[gi * APITCH + gh * GC + u] = v;
            }
        } else {
            const double inv = 1.0 / sqrt(M);
#pragma unroll
            for (int u = 0; u < GC; ++u) {
                const int64_t jg = row_offset + jl0 + u;
                double v = (__popcll((unsigned long long)(rr & jg)) & 1) ? -inv : inv;
                if (!grow_ok || jl0 + u >= kend) v = 0.0;
                dst[gi * APITCH + gh * GC + u] = v;
            }
        }
    };
    // A tile loader role: thread -> (k row, LC consecutive columns)
    constexpr int LC = BK * BN / THREADS;   // 4
    const int lk = tid / (BN / LC), lc = (tid % (BN / LC)) * LC;
    double areg[LC];
    auto load_a = [&](int64_t kb) {
        const int64_t k = kb + lk;
#pragma unroll
        for (int u = 0; u < LC; ++u) {
            const int c = c0 + lc + u;
            areg[u] = (k < kend && c < n) ? a[k * lda + c] : 0.0;
        }
    };
    auto store_a = [&](double *dst, int64_t kb) {
        const int64_t k = kb + lk;
        const double s = (k < kend) ? signs[row_offset + k] : 0.0;
#pragma unroll
        for (int u = 0; u < LC; ++u) dst[lk * BPITCH + lc + u] = s * demote<LEVEL>(areg[u], over);
    };

    double acc[WM / 8][WN / 8][2];
#pragma unroll
    for (int x = 0; x < WM / 8; ++x)
#pragma unroll
        for (int y = 0; y < WN / 8; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;

    if (nk > 0) {
        load_a(kbeg);
        gen_omega(om, kbeg);
        store_a(bt, kbeg);
    }
    __syncthreads();
    for (int kt = 0; kt < nk; ++kt) {
        const int cur = kt & 1;
        const bool more = kt + 1 < nk;
        const int64_t kb_next = kbeg + (int64_t)(kt + 1) * BK;
        if (more) load_a(kb_next);
        const double *os = om + cur * BM * APITCH;
        const double *bs = bt + cur * BK * BPITCH;
#pragma unroll
        for (int kk = 0; kk < BK; kk += 4) {
            double af[WM / 8], bf[WN / 8];
#pragma unroll
            for (int x = 0; x < WM / 8; ++x) af[x] = os[(wm * WM + x * 8 + g) * APITCH + kk + t];
#pragma unroll
            for (int y = 0; y < WN / 8; ++y) bf[y] = bs[(kk + t) * BPITCH + wn * WN + y * 8 + g];
#pragma unroll
            for (int x = 0; x < WM / 8; ++x)
#pragma unroll
                for (int y = 0; y < WN / 8; ++y) dmma884(acc[x][y][0], acc[x][y][1], af[x], bf[y]);
        }
        if (more) {
            gen_omega(om + (cur ^ 1) * BM * APITCH, kb_next);
            store_a(bt + (cur ^ 1) * BK * BPITCH, kb_next);
        }
        __syncthreads();
    }
    if (over) atomicOr(overflow_flag, 1);

    double *out = part + ((size_t)split * ntiles + tile) * (BM * BN);
#pragma unroll
    for (int x = 0; x < WM / 8; ++x)
#pragma unroll
        for (int y = 0; y < WN / 8; ++y) {
            const int r = wm * WM + x * 8 + g, c = wn * WN + y * 8 + 2 * t;
            *reinterpret_cast<double2 *>(out + r * BN + c) = make_double2(acc[x][y][0], acc[x][y][1]);
        }
}

// out (col-major d x n, ldo) (+)= sum over splits
__global__ void sketch_reduce(const double *__restrict__ part, int splits, int ntiles, int ntn, int d, int n,
                              double *__restrict__ out, int64_t ldo, int accumulate) {
    const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= (int64_t)d * n) return;
    const int c = (int)(idx / d), i = (int)(idx % d);   // consecutive threads -> consecutive i (col-major)
    const int tile = (i / BM) * ntn + (c / BN);
    const double *p = part + (size_t)tile * (BM * BN) + (i % BM) * BN + (c % BN);
    double s = 0.0;
    for (int k = 0; k < splits; ++k) s += p[(size_t)k * ntiles * (BM * BN)];
    double *o = out + (int64_t)c * ldo + i;
    *o = accumulate ? *o + s : s;
}

template <int LEVEL>
__global__ void sketch_finalize_kernel(const double *__restrict__ sum, int64_t ldsum, int d, int n,
                                       double scale64, void *a_s, double *out_f64) {
    const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= (int64_t)d * n) return;
    const int c = (int)(idx / d), i = (int)(idx % d);
    const double v = sum[(int64_t)c * ldsum + i];
    double promoted;
    if (LEVEL == 16) {
        // transform computed in binary32 then rounded to binary16 (src/sketch.py:163-165),
        // then the binary16 product with binary16(sqrt(m_pad/d)) (src/sketch.py:168-169)
        const __half h = __float2half_rn(__double2float_rn(v));
        const __half s = __float2half_rn(__double2float_rn(scale64));
        const __half o = __float2half_rn(__fmul_rn(__half2float(h), __half2float(s)));
        static_cast<__half *>(a_s)[idx] = o;
        promoted = (double)__half2float(o);
    } else if (LEVEL == 32) {
        const float o = __fmul_rn(__double2float_rn(v), __double2float_rn(scale64));
        static_cast<float *>(a_s)[idx] = o;
        promoted = (double)o;
    } else {
        const double o = __dmul_rn(v, scale64);
        static_cast<double *>(a_s)[idx] = o;
        promoted = o;
    }
    if (out_f64) out_f64[(int64_t)i * n + c] = promoted;
}

struct Plan {
    int ntm, ntn, ntiles, splits;
    int64_t kchunk;
};
static Plan make_plan(int64_t m_local, int64_t n, int64_t d) {
    Plan p;
    p.ntm = (int)((d + BM - 1) / BM);
    p.ntn = (int)((n + BN - 1) / BN);
    p.ntiles = p.ntm * p.ntn;
    const int sms = sm_count();
    int64_t smax = (m_local + 63) / 64;   // >= 64 rows per split (small m: more CTAs, shorter K loops)
    if (smax < 1) smax = 1;
    int64_t target = (int64_t)32 * sms / p.ntiles;
    if (target < 1) target = 1;
    if (target > smax) target = smax;
    int64_t best = target;
    for (int64_t s = target; s >= (target * 4) / 5 && s >= 1; --s)
        if (((int64_t)p.ntiles * s) % sms == 0) { best = s; break; }
    p.kchunk = (m_local + best - 1) / best;
    p.kchunk = (p.kchunk + BK - 1) / BK * BK;
    if (p.kchunk < BK) p.kchunk = BK;
    p.splits = (int)((m_local + p.kchunk - 1) / p.kchunk);
    if (p.splits < 1) p.splits = 1;
    return p;
}

}  // namespace sketch
}  // namespace sk

using namespace sk;

namespace sk {
bool sketch_fft_supported(int64_t m_pad);
size_t sketch_fft_workspace(int64_t m_pad, int64_t n, int64_t d);
int sketch_fft_run(int level, const double *a, int64_t lda, int64_t m_local, int64_t row_offset, int64_t m_pad,
                   int64_t n, const double *signs, const int64_t *rows, int64_t d, double *out, int64_t ldo,
                   int accumulate, int *overflow_flag_dev, void *ws, size_t ws_bytes, cudaStream_t st);
size_t sketch_tc_workspace(int64_t m_local, int64_t n, int64_t d);
int sketch_tc_run(int transform, const double *a, int64_t lda, int64_t m_local, int64_t row_offset, int64_t m_pad,
                  int64_t n, const double *signs, const int64_t *rows, int64_t d, double *out, int64_t ldo,
                  int accumulate, int *overflow_flag_dev, void *ws, size_t ws_bytes, cudaStream_t st);
}

extern "C" {

static size_t dmma_sketch_ws(int64_t m_local, int64_t n, int64_t d) {
    sketch::Plan p = sketch::make_plan(m_local, n, d);
    return (size_t)p.splits * p.ntiles * sketch::BM * sketch::BN * sizeof(double);
}

size_t sk_sketch_workspace(int level, int64_t m_local, int64_t n, int64_t d) {
    (void)level;
    // independent of the row shard's size for the FFT path, so callers pass m_pad
    // as m_local to size it; take the max over engines
    const size_t a = dmma_sketch_ws(m_local, n, d);
    const size_t b = sk::sketch_tc_workspace(m_local, n, d);
    const size_t c = sk::sketch_fft_workspace(m_local, n, d);
    return std::max(a, std::max(b, c));
}

size_t sk_sketch_workspace_ex(int level, int transform, int64_t m_local, int64_t m_pad, int64_t n, int64_t d) {
    size_t w = dmma_sketch_ws(m_local, n, d);
    if (level == 16) w = std::max(w, sk::sketch_tc_workspace(m_local, n, d));
    if (transform == SK_DCT2) w = std::max(w, sk::sketch_fft_workspace(m_pad, n, d));
    return w;
}

int sk_sketch_partial_ex(int level, int transform, const double *a, int64_t lda, int64_t m_local,
                         int64_t row_offset, int64_t m_pad, int64_t n, const double *signs, const int64_t *rows,
                         int64_t d, double *out, int64_t ldo, int accumulate, int *overflow_flag_dev, void *ws,
                         size_t ws_bytes, sk_stream_t stream, int algo);

// binary16 engine under SK_SKETCH_AUTO: the FFT transform costs O(M log M) for the WHOLE
// operator height M, the tcgen05 GEMM O(d m_local) for the rows this call holds.  The
// FFT wins for the whole matrix; row shards / streamed chunks keep the GEMM.
// SK_SKETCH16=tc|fft overrides.
// Whole matrix at 4M x 2048: FFT (binary32 transform, whole-sector Y) 88 ms vs the
// tcgen05 GEMM 100 ms (profiles/r2s2_sketch_engines.json).
constexpr bool FFT16_DEFAULT = true;
static bool fft16_preferred(bool fft_ok, int64_t m_local, int64_t m_pad) {
    static const char *env = getenv("SK_SKETCH16");
    if (env && strcmp(env, "tc") == 0) return false;
    if (env && strcmp(env, "fft") == 0) return fft_ok;
    return fft_ok && m_local == m_pad && FFT16_DEFAULT;
}

int sk_sketch_partial(int level, int transform, const double *a, int64_t lda, int64_t m_local,
                      int64_t row_offset, int64_t m_pad, int64_t n, const double *signs,
                      const int64_t *rows, int64_t d, double *out, int64_t ldo, int accumulate,
                      int *overflow_flag_dev, void *ws, size_t ws_bytes, sk_stream_t stream) {
    return sk_sketch_partial_ex(level, transform, a, lda, m_local, row_offset, m_pad, n, signs, rows, d, out, ldo,
                                accumulate, overflow_flag_dev, ws, ws_bytes, stream, SK_SKETCH_AUTO);
}

int sk_sketch_partial_ex(int level, int transform, const double *a, int64_t lda, int64_t m_local,
                         int64_t row_offset, int64_t m_pad, int64_t n, const double *signs, const int64_t *rows,
                         int64_t d, double *out, int64_t ldo, int accumulate, int *overflow_flag_dev, void *ws,
                         size_t ws_bytes, sk_stream_t stream, int algo) {
    if (!a || !signs || !rows || !out || !overflow_flag_dev || m_local < 0 || n <= 0 || d <= 0 ||
        lda < n || ldo < d || m_pad <= 0 || row_offset < 0 || row_offset + m_local > m_pad ||
        (level != 16 && level != 32 && level != 64) || (transform != SK_DCT2 && transform != SK_WHT) ||
        m_pad >= (int64_t(1) << 30) || algo < SK_SKETCH_AUTO || algo > SK_SKETCH_FFT) {
        set_error("sk_sketch_partial: bad arguments");
        return SK_ERR_ARG;
    }
    const bool fft_ok = transform == SK_DCT2 && sk::sketch_fft_supported(m_pad);
    if (level == 16 && (algo == SK_SKETCH_TC || (algo == SK_SKETCH_AUTO && !fft16_preferred(fft_ok, m_local, m_pad))))
        return sk::sketch_tc_run(transform, a, lda, m_local, row_offset, m_pad, n, signs, rows, d, out, ldo,
                                 accumulate, overflow_flag_dev, ws, ws_bytes, (cudaStream_t)stream);
    if (algo == SK_SKETCH_TC) {
        set_error("sk_sketch_partial: the tensor-core path exists for binary16 only");
        return SK_ERR_ARG;
    }
    if (algo == SK_SKETCH_FFT || (algo == SK_SKETCH_AUTO && fft_ok)) {
        if (!fft_ok) {
            set_error("sk_sketch_partial: the FFT path needs DCT-II and m_pad %% 2048 == 0");
            return SK_ERR_ARG;
        }
        return sk::sketch_fft_run(level, a, lda, m_local, row_offset, m_pad, n, signs, rows, d, out, ldo, accumulate,
                                  overflow_flag_dev, ws, ws_bytes, (cudaStream_t)stream);
    }
    sketch::Plan p = sketch::make_plan(m_local, n, d);
    const size_t need = (size_t)p.splits * p.ntiles * sketch::BM * sketch::BN * sizeof(double);
    if (!ws || ws_bytes < need) {
        set_error("sk_sketch_partial: workspace %zu < %zu", ws_bytes, need);
        return SK_ERR_ARG;
    }
    cudaStream_t st = (cudaStream_t)stream;
    double *part = static_cast<double *>(ws);
    const unsigned units = (unsigned)(p.ntiles * p.splits);
#define SK_SKETCH(L, T)                                                                            \
    do {                                                                                           \
        auto kfn = sketch::sketch_kernel<L, T>;                                                    \
        SK_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sketch::SMEM)); \
        kfn<<<units, sketch::THREADS, sketch::SMEM, st>>>(a, lda, m_local, row_offset, m_pad, (int)n, signs, \
                                                          rows, (int)d, p.ntn, p.ntiles, p.kchunk, part,    \
                                                          overflow_flag_dev);                      \
    } while (0)
    if (transform == SK_DCT2) {
        if (level == 16) SK_SKETCH(16, SK_DCT2);
        else if (level == 32) SK_SKETCH(32, SK_DCT2);
        else SK_SKETCH(64, SK_DCT2);
    } else {
        if (level == 16) SK_SKETCH(16, SK_WHT);
        else if (level == 32) SK_SKETCH(32, SK_WHT);
        else SK_SKETCH(64, SK_WHT);
    }
#undef SK_SKETCH
    SK_LAUNCH_CHECK("sketch_kernel");
    const int64_t total = d * n;
    sketch::sketch_reduce<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(part, p.splits, p.ntiles, p.ntn,
                                                                           (int)d, (int)n, out, ldo, accumulate);
    SK_LAUNCH_CHECK("sketch_reduce");
    return SK_OK;
}

int sk_sketch_finalize(int level, const double *sum, int64_t ldsum, int64_t d, int64_t n, int64_t m_pad,
                       void *a_s_level, double *out_f64, sk_stream_t stream) {
    if (!sum || !a_s_level || d <= 0 || n <= 0 || ldsum < d || m_pad <= 0) {
        set_error("sk_sketch_finalize: bad arguments");
        return SK_ERR_ARG;
    }
    const double scale = sqrt((double)m_pad / (double)d);   // math.sqrt(op.m_pad / op.d)
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t total = d * n;
    const unsigned grid = (unsigned)((total + 255) / 256);
    if (level == 16) sketch::sketch_finalize_kernel<16><<<grid, 256, 0, st>>>(sum, ldsum, (int)d, (int)n, scale, a_s_level, out_f64);
    else if (level == 32) sketch::sketch_finalize_kernel<32><<<grid, 256, 0, st>>>(sum, ldsum, (int)d, (int)n, scale, a_s_level, out_f64);
    else if (level == 64) sketch::sketch_finalize_kernel<64><<<grid, 256, 0, st>>>(sum, ldsum, (int)d, (int)n, scale, a_s_level, out_f64);
    else { set_error("bad level"); return SK_ERR_ARG; }
    SK_LAUNCH_CHECK("sketch_finalize_kernel");
    return SK_OK;
}

}  // extern "C"

namespace sk {
namespace sketch {
// numpy's Philox (Philox4x64, 10 rounds): one thread per 4-word output block.
__global__ void __launch_bounds__(256)
signs_kernel(uint64_t k0, uint64_t k1, int64_t count, double *__restrict__ signs) {
    const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (b * 8 >= count) return;
    uint64_t c0 = (uint64_t)b + 1, c1 = 0, c2 = 0, c3 = 0, ka = k0, kb = k1;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint64_t lo0 = 0xD2E7470EE14C6C93ull * c0, hi0 = __umul64hi(0xD2E7470EE14C6C93ull, c0);
        const uint64_t lo1 = 0xCA5A826395121157ull * c2, hi1 = __umul64hi(0xCA5A826395121157ull, c2);
        const uint64_t n0 = hi1 ^ c1 ^ ka, n2 = hi0 ^ c3 ^ kb;
        c0 = n0;
        c1 = lo1;
        c2 = n2;
        c3 = lo0;
        ka += 0x9E3779B97F4A7C15ull;
        kb += 0xBB67AE8584CAA73Bull;
    }
    const uint64_t w[4] = {c0, c1, c2, c3};
    double s[8];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        s[2 * q] = (w[q] & 0x80000000ull) ? 1.0 : -1.0;              // low 32-bit draw
        s[2 * q + 1] = (w[q] & 0x8000000000000000ull) ? 1.0 : -1.0;  // high 32-bit draw
    }
    const int64_t j0 = b * 8;
    if (j0 + 8 <= count) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
            reinterpret_cast<double2 *>(signs + j0)[q] = make_double2(s[2 * q], s[2 * q + 1]);
    } else {
        for (int q = 0; q < 8 && j0 + q < count; ++q) signs[j0 + q] = s[q];
    }
}
}  // namespace sketch
}  // namespace sk

extern "C" int sk_sketch_signs(uint64_t key_lo, uint64_t key_hi, int64_t count, double *signs, sk_stream_t stream) {
    if (count < 0 || (count > 0 && (!signs || (reinterpret_cast<uintptr_t>(signs) & 15)))) {
        set_error("sk_sketch_signs: bad arguments (signs must be 16-byte aligned)");
        return SK_ERR_ARG;
    }
    if (count == 0) return SK_OK;
    const int64_t blocks = (count + 7) / 8;
    sketch::signs_kernel<<<(unsigned)((blocks + 255) / 256), 256, 0, (cudaStream_t)stream>>>(key_lo, key_hi, count,
                                                                                           signs);
    SK_LAUNCH_CHECK("signs_kernel");
    return SK_OK;
}
