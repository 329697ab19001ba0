// FP64 fast sampled DCT-II sketch (binary64 / binary32 levels).
//
// The reference applies the sketch as a full length-M orthonormal DCT-II
// (pocketfft, src/sketch.py:163-167) and keeps d rows.  A dense GEMM against the
// sampled operator costs 2 d M n flops (2.8 s in FP64 at 4M x 2048); the transform
// costs O(M log M n).  Here the DCT is computed through Makhoul's reordering and a
// four-step FFT whose second step is pruned to the sampled outputs:
//
//   v_j = x_{2j} (j < M/2),  v_{M-1-j} = x_{2j+1};   X_k = Re(e^{-i pi k / 2M} V_k),
//   V_k = DFT_M(v)_k,  j = j1 + M1 j2 (j2 < M2 = 2048),  k = k2 + M2 k1:
//   pass A  for every j1 and column pair (c, c'): the M2-point FFT over j2 of
//           z = v_c + i v_c' (two real columns per complex FFT), times the twiddle
//           e^{-2 pi i j1 k2 / M}  ->  Y[pair][k2][j1]             (in shared memory,
//           mixed-radix 16 x 16 x 8 Stockham, table twiddles)
//   pass B  for every sampled k and its mirror M-k: Z = sum_j1 e^{-2 pi i j1 k1 / M1}
//           Y[pair][k2][j1], requests grouped by k2 so each Y row is read once
//   final   V_c = (Z_k + conj Z_{M-k}) / 2, V_c' = (Z_k - conj Z_{M-k}) / 2i,
//           out[k, c] = c_k Re(e^{-i pi k / 2M} V_c)    (unscaled operator F D)
//
// HBM traffic ~ 8Mn (A) + 2 x 8Mn (Y written and read), in column blocks so Y stays
// a few GB.  Arithmetic is FP64 throughout; the result is rounded to the level in
// sk_sketch_finalize (binary32: more accurate than the reference's binary32 FFT).
#include <vector>

#include "common.cuh"

namespace sk {
namespace skfft {

constexpr int N2 = 1024;          // M2: FFT length of pass A
constexpr int A_THREADS = 512;    // 4 FFTs per CTA (2 j1 x 2 column pairs)
constexpr int B_THREADS = 256;
constexpr int B_PAIRS = 4;        // column pairs per pass-B CTA

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 mul_mi(double2 a) { return make_double2(a.y, -a.x); }   // a * (-i)

// forward 4-point DFT (W4 = -i)
__device__ __forceinline__ void dft4(double2 &x0, double2 &x1, double2 &x2, double2 &x3) {
    const double2 a = cadd(x0, x2), b = csub(x0, x2), c = cadd(x1, x3), d = mul_mi(csub(x1, x3));
    x0 = cadd(a, c);
    x2 = csub(a, c);
    x1 = cadd(b, d);
    x3 = csub(b, d);
}

// forward R-point DFT in registers, R = 16 (4 x 4) or 8 (4 x 2); tw = e^{-2 pi i t / N2} table
template <int R>
__device__ __forceinline__ void dft_small(double2 (&v)[R], const double2 *tw) {
    if constexpr (R == 4) {
        dft4(v[0], v[1], v[2], v[3]);
    } else if constexpr (R == 16) {
        // n = 4 n1 + n2: 4-point over n1, twiddle W16^{n2 k1}, 4-point over n2
#pragma unroll
        for (int n2 = 0; n2 < 4; ++n2) dft4(v[n2], v[4 + n2], v[8 + n2], v[12 + n2]);
        // now v[4 k1 + n2] = A[n2][k1]
#pragma unroll
        for (int n2 = 1; n2 < 4; ++n2)
#pragma unroll
            for (int k1 = 1; k1 < 4; ++k1) v[4 * k1 + n2] = cmul(v[4 * k1 + n2], tw[(n2 * k1) * (N2 / 16)]);
#pragma unroll
        for (int k1 = 0; k1 < 4; ++k1) dft4(v[4 * k1], v[4 * k1 + 1], v[4 * k1 + 2], v[4 * k1 + 3]);
        // v[4 k1 + k2] = X[k1 + 4 k2] -> reorder
        double2 t[16];
#pragma unroll
        for (int k1 = 0; k1 < 4; ++k1)
#pragma unroll
            for (int k2 = 0; k2 < 4; ++k2) t[k1 + 4 * k2] = v[4 * k1 + k2];
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = t[i];
    } else {
        static_assert(R == 8, "radix");
        // n = 2 n1 + n2: 4-point over n1, twiddle W8^{n2 k1}, 2-point over n2
        dft4(v[0], v[2], v[4], v[6]);
        dft4(v[1], v[3], v[5], v[7]);
        // v[2 k1 + n2] = A[n2][k1]
#pragma unroll
        for (int k1 = 1; k1 < 4; ++k1) v[2 * k1 + 1] = cmul(v[2 * k1 + 1], tw[k1 * (N2 / 8)]);
        double2 t[8];
#pragma unroll
        for (int k1 = 0; k1 < 4; ++k1) {
            t[k1] = cadd(v[2 * k1], v[2 * k1 + 1]);
            t[k1 + 4] = csub(v[2 * k1], v[2 * k1 + 1]);
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = t[i];
    }
}

// One Stockham stage (radix R, Ns = product of earlier radices) over `nfft` in-place
// FFTs of length N2 stored back to back in x; threads stride over butterflies.
// PER = butterflies per thread (compile-time: nfft * N2 / R == PER * blockDim.x).
template <int R, int PER>
__device__ __forceinline__ void stockham_stage(double2 *x, int Ns, const double2 *tw) {
    constexpr int NB = N2 / R;
    double2 v[PER][R];
#pragma unroll
    for (int c = 0; c < PER; ++c) {
        const int b = threadIdx.x + c * blockDim.x;
        const int f = b / NB, j = b % NB;
        const double2 *xf = x + f * N2;
#pragma unroll
        for (int r = 0; r < R; ++r) v[c][r] = xf[j + r * NB];
        const int jm = j % Ns;
        // stage twiddle e^{-2 pi i jm r / (Ns R)} = tw[jm r N2 / (Ns R)]
        const int step = jm * (N2 / (Ns * R));
#pragma unroll
        for (int r = 1; r < R; ++r) v[c][r] = cmul(v[c][r], tw[(r * step) & (N2 - 1)]);
        dft_small<R>(v[c], tw);
    }
    __syncthreads();
#pragma unroll
    for (int c = 0; c < PER; ++c) {
        const int b = threadIdx.x + c * blockDim.x;
        const int f = b / NB, j = b % NB, jm = j % Ns;
        double2 *xf = x + f * N2;
        const int base = (j / Ns) * Ns * R + jm;
#pragma unroll
        for (int r = 0; r < R; ++r) xf[base + r * Ns] = v[c][r];
    }
    __syncthreads();
}

struct PassAParams {
    const double *a;
    int64_t lda, m_local, row_offset, M, M1;
    const double *signs;
    int c0, ncols;          // column block [c0, c0 + ncols), ncols multiple of 4 (pairs padded)
    int n;
    double2 *y;             // [pair][k2][j1], pairs of this block
    int level;              // 32: demote A to binary32 on load (overflow -> *overflow = 1); 64: as is
    int *overflow;
    const double2 *tw_n2;   // e^{-2 pi i t / N2}, t < N2 (precomputed once per call)
};

// e^{-2 pi i t / len}, t < len (one table per call instead of one per CTA)
__global__ void twiddle_table(double2 *tw, int64_t len) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < len; t += (int64_t)gridDim.x * blockDim.x) {
        double s, c;
        sincospi(-2.0 * (double)t / (double)len, &s, &c);
        tw[t] = make_double2(c, s);
    }
}

// grid: (M1/2, ncols/8).  A CTA owns j1 in {2 a2, 2 a2 + 1} and 8 columns (4 complex
// pairs): every gathered row segment is a full 64-byte line, every Y store 32 bytes.
__global__ void __launch_bounds__(A_THREADS) fft_pass_a(const PassAParams p) {
    extern __shared__ __align__(16) double2 fa_smem[];
    double2 *tw = fa_smem;                  // N2 twiddles
    double2 *x = fa_smem + N2;              // 8 FFTs: f = jj * 4 + pp
    double2 *otw = x + 8 * N2;              // [jj][hi 32 | lo 32]: e^{-2 pi i j1 (32 h + l) / M}
    const int a2 = blockIdx.x;
    const int q = blockIdx.y;               // column octet
    for (int t = threadIdx.x; t < N2; t += blockDim.x) tw[t] = p.tw_n2[t];
    if (threadIdx.x < 128) {
        // output twiddles e^{-2 pi i j1 k2 / M} = hi[k2 / 32] * lo[k2 % 32] (j1 k2 < M, exact phases)
        const int jj = threadIdx.x >> 6, h = (threadIdx.x >> 5) & 1, t = threadIdx.x & 31;
        const int64_t j1 = 2 * (int64_t)a2 + jj;
        const int64_t ph = j1 * (int64_t)(h ? t : 32 * t);
        double s, c;
        sincospi(-2.0 * (double)ph / (double)p.M, &s, &c);
        otw[jj * 64 + (h ? 32 : 0) + t] = make_double2(c, s);
    }
    // ---- gather: v_{j1 + M1 j2} for the two j1 and eight columns
    const int cbase = p.c0 + 8 * q;
    for (int e = threadIdx.x; e < 2 * N2; e += blockDim.x) {
        const int jj = e / N2, j2 = e % N2;
        const int64_t j1 = 2 * (int64_t)a2 + jj;
        const int64_t row = (j2 < N2 / 2) ? (2 * j1 + 2 * p.M1 * (int64_t)j2)
                                          : (2 * p.M - 1 - 2 * j1 - 2 * p.M1 * (int64_t)j2);
        const int64_t lr = row - p.row_offset;
        double v[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        if (lr >= 0 && lr < p.m_local) {
            const double sg = p.signs[row];
            const double *src = p.a + lr * p.lda + cbase;
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (cbase + u < p.n) {
                    double w = src[u];
                    if (p.level == 32) {   // round_to_precision(A, binary32) (src/precision.py:90-103)
                        const double r = (double)__double2float_rn(w);
                        if (isinf(r) && isfinite(w)) *p.overflow = 1;
                        w = r;
                    }
                    v[u] = sg * w;
                }
        }
#pragma unroll
        for (int pp = 0; pp < 4; ++pp) x[(jj * 4 + pp) * N2 + j2] = make_double2(v[2 * pp], v[2 * pp + 1]);
    }
    __syncthreads();
    // 8 FFTs x 1024 points: radix-16 stages have 512 butterflies (1 per thread),
    // the radix-4 stage 2048 (4 per thread)
    stockham_stage<16, 1>(x, 1, tw);
    stockham_stage<16, 1>(x, 16, tw);
    stockham_stage<4, 4>(x, 256, tw);
    // ---- twiddle e^{-2 pi i j1 k2 / M} and store Y[pair][k2][j1 pair]
    const int pair0 = 4 * q;                // pair index within the block
    for (int e = threadIdx.x; e < 4 * N2; e += blockDim.x) {
        const int pp = e / N2, k2 = e % N2;
        double2 out[2];
#pragma unroll
        for (int jj = 0; jj < 2; ++jj) {
            const double2 w = cmul(otw[jj * 64 + (k2 >> 5)], otw[jj * 64 + 32 + (k2 & 31)]);
            out[jj] = cmul(x[(jj * 4 + pp) * N2 + k2], w);
        }
        double2 *dst = p.y + ((size_t)(pair0 + pp) * N2 + k2) * p.M1 + 2 * a2;
        *reinterpret_cast<double4 *>(dst) = make_double4(out[0].x, out[0].y, out[1].x, out[1].y);
    }
}

struct PassBParams {
    const double2 *y;
    int64_t M1;
    const int *req_ptr;     // CSR over k2: requests [req_ptr[k2], req_ptr[k2+1])
    const int *req_s;       // sample index
    const int *req_which;   // 0: target k, 1: target M-k
    const int64_t *req_k1;  // k1 of the target
    int npairs;             // pairs in this block
    double2 *zbuf;          // [s][which][pair] (pairs of this block), ldz = npairs
    int d;
    const double2 *tw_m1;   // e^{-2 pi i t / M1}, t < M1 (precomputed once per call)
};

// grid: (N2 k2 values, ceil(npairs / B_PAIRS))
__global__ void __launch_bounds__(B_THREADS) fft_pass_b(const PassBParams p) {
    extern __shared__ __align__(16) double2 fb_smem[];
    const int k2 = blockIdx.x;
    const int r0 = p.req_ptr[k2], r1 = p.req_ptr[k2 + 1];
    if (r0 == r1) return;
    const int M1 = (int)p.M1;
    double2 *tw = fb_smem;                  // e^{-2 pi i t / M1}
    const int pbase = blockIdx.y * B_PAIRS;
    const int np = min(B_PAIRS, p.npairs - pbase);
    for (int t = threadIdx.x; t < M1; t += blockDim.x) tw[t] = p.tw_m1[t];
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const int tasks = (r1 - r0) * np;
    for (int t = warp; t < tasks; t += nw) {
        const int rq = r0 + t / np, pp = t % np;
        const int64_t k1 = p.req_k1[rq];
        double2 acc = make_double2(0.0, 0.0);
        const double2 *yrow = p.y + ((size_t)(pbase + pp) * N2 + k2) * M1;   // reused by the k2's requests (L1/L2)
        // twiddle index (j1 k1) mod M1, advanced incrementally (no 64-bit modulo per term)
        int idx = (int)(((int64_t)lane * k1) % M1);
        const int step = (int)((32 * k1) % M1);
        for (int j1 = lane; j1 < M1; j1 += 32) {
            const double2 w = tw[idx];
            idx += step;
            if (idx >= M1) idx -= M1;
            const double2 yv = yrow[j1];
            acc.x += w.x * yv.x - w.y * yv.y;
            acc.y += w.x * yv.y + w.y * yv.x;
        }
        acc.x = warp_sum(acc.x);
        acc.y = warp_sum(acc.y);
        if (lane == 0) p.zbuf[((size_t)p.req_s[rq] * 2 + p.req_which[rq]) * p.npairs + pbase + pp] = acc;
    }
}

// out (col-major d x n, ldo) (+)= c_k Re(e^{-i pi k / 2M} V) for the block's columns
__global__ void fft_finalize(const double2 *zbuf, int npairs, const int64_t *rows, int d, int64_t M, int c0,
                             int ncols_real, double *out, int64_t ldo, int accumulate) {
    const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= (int64_t)d * npairs) return;
    const int pp = (int)(idx / d), s = (int)(idx % d);
    const double2 zk = zbuf[((size_t)s * 2 + 0) * npairs + pp];
    const double2 zm = zbuf[((size_t)s * 2 + 1) * npairs + pp];
    // V_a = (Zk + conj Zm)/2, V_b = (Zk - conj Zm)/(2i)
    const double2 va = make_double2(0.5 * (zk.x + zm.x), 0.5 * (zk.y - zm.y));
    const double2 vb = make_double2(0.5 * (zk.y + zm.y), -0.5 * (zk.x - zm.x));
    const int64_t k = rows[s];
    double sn, cs;
    sincospi(-(double)k / (2.0 * (double)M), &sn, &cs);
    const double ck = (k == 0) ? sqrt(1.0 / (double)M) : sqrt(2.0 / (double)M);
    const double xa = ck * (va.x * cs - va.y * sn);
    const double xb = ck * (vb.x * cs - vb.y * sn);
    const int ca = c0 + 2 * pp, cb = ca + 1;
    if (ca < ncols_real) {
        double *o = out + (int64_t)ca * ldo + s;
        *o = accumulate ? *o + xa : xa;
    }
    if (cb < ncols_real) {
        double *o = out + (int64_t)cb * ldo + s;
        *o = accumulate ? *o + xb : xb;
    }
}

constexpr int COLBLOCK = 256;   // columns per block: Y = 8 M COLBLOCK bytes

}  // namespace skfft

bool sketch_fft_supported(int64_t m_pad) { return m_pad >= 2 * skfft::N2 && m_pad % (2 * skfft::N2) == 0; }

size_t sketch_fft_workspace(int64_t m_pad, int64_t n, int64_t d) {
    using namespace skfft;
    if (!sketch_fft_supported(m_pad)) return 0;
    const int64_t cb = std::min<int64_t>(COLBLOCK, (n + 7) / 8 * 8);
    const size_t ybytes = (size_t)(cb / 2) * m_pad * sizeof(double2);
    const size_t zbytes = (size_t)d * 2 * (cb / 2) * sizeof(double2);
    const size_t req = (size_t)(N2 + 1) * sizeof(int) + (size_t)2 * d * (2 * sizeof(int) + sizeof(int64_t));
    const size_t tables = (size_t)(N2 + m_pad / N2) * sizeof(double2);
    return align_up(ybytes, 256) + align_up(zbytes, 256) + align_up(req, 256) + align_up(tables, 256) + 1024;
}

int sketch_fft_run(int level, const double *a, int64_t lda, int64_t m_local, int64_t row_offset, int64_t m_pad,
                   int64_t n, const double *signs, const int64_t *rows, int64_t d, double *out, int64_t ldo,
                   int accumulate, int *overflow_flag_dev, void *ws, size_t ws_bytes, cudaStream_t st) {
    using namespace skfft;
    if (!sketch_fft_supported(m_pad)) { set_error("sketch_fft: M must be a multiple of 4096"); return SK_ERR_ARG; }
    if (ws_bytes < sketch_fft_workspace(m_pad, n, d)) { set_error("sketch_fft: workspace too small"); return SK_ERR_ARG; }
    const int64_t M = m_pad, M1 = M / N2;
    const int64_t cb = std::min<int64_t>(COLBLOCK, (n + 7) / 8 * 8);
    uint8_t *p = static_cast<uint8_t *>(ws);
    double2 *y = reinterpret_cast<double2 *>(p);
    p += align_up((size_t)(cb / 2) * M * sizeof(double2), 256);
    double2 *zbuf = reinterpret_cast<double2 *>(p);
    p += align_up((size_t)d * 2 * (cb / 2) * sizeof(double2), 256);
    int *d_ptr = reinterpret_cast<int *>(p);
    int *d_s = d_ptr + (N2 + 1);
    int *d_w = d_s + 2 * d;
    int64_t *d_k1 = reinterpret_cast<int64_t *>(align_up(reinterpret_cast<uintptr_t>(d_w + 2 * d), 8));
    p += align_up((size_t)(N2 + 1) * sizeof(int) + (size_t)2 * d * (2 * sizeof(int) + sizeof(int64_t)), 256);
    double2 *tw_n2 = reinterpret_cast<double2 *>(p);
    double2 *tw_m1 = tw_n2 + N2;
    twiddle_table<<<4, 256, 0, st>>>(tw_n2, N2);
    twiddle_table<<<(unsigned)std::min<int64_t>((M1 + 255) / 256, 1024), 256, 0, st>>>(tw_m1, M1);
    SK_LAUNCH_CHECK("twiddle_table");
    // ---- request lists grouped by k2 (host; d entries)
    std::vector<int64_t> hrows((size_t)d);
    SK_CUDA(cudaMemcpyAsync(hrows.data(), rows, (size_t)d * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    SK_CUDA(cudaStreamSynchronize(st));
    std::vector<int> cnt(N2 + 1, 0), hs(2 * d), hw(2 * d);
    std::vector<int64_t> hk1(2 * d);
    for (int64_t s = 0; s < d; ++s)
        for (int w = 0; w < 2; ++w) {
            const int64_t t = (w == 0) ? hrows[s] : (M - hrows[s]) % M;
            cnt[(t % N2) + 1]++;
        }
    for (int i = 0; i < N2; ++i) cnt[i + 1] += cnt[i];
    std::vector<int> fill(cnt.begin(), cnt.end() - 1);
    for (int64_t s = 0; s < d; ++s)
        for (int w = 0; w < 2; ++w) {
            const int64_t t = (w == 0) ? hrows[s] : (M - hrows[s]) % M;
            const int at = fill[t % N2]++;
            hs[at] = (int)s;
            hw[at] = w;
            hk1[at] = t / N2;
        }
    SK_CUDA(cudaMemcpyAsync(d_ptr, cnt.data(), (size_t)(N2 + 1) * sizeof(int), cudaMemcpyHostToDevice, st));
    SK_CUDA(cudaMemcpyAsync(d_s, hs.data(), (size_t)2 * d * sizeof(int), cudaMemcpyHostToDevice, st));
    SK_CUDA(cudaMemcpyAsync(d_w, hw.data(), (size_t)2 * d * sizeof(int), cudaMemcpyHostToDevice, st));
    SK_CUDA(cudaMemcpyAsync(d_k1, hk1.data(), (size_t)2 * d * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    const size_t smem_a = (size_t)(N2 + 8 * N2 + 128) * sizeof(double2);
    const size_t smem_b = (size_t)M1 * sizeof(double2);
    if (smem_b > 200 * 1024) { set_error("sketch_fft: M too large for pass B (M1 %lld)", (long long)M1); return SK_ERR_ARG; }
    SK_CUDA(cudaFuncSetAttribute(fft_pass_a, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_a));
    SK_CUDA(cudaFuncSetAttribute(fft_pass_b, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_b));
    for (int64_t c0 = 0; c0 < n; c0 += cb) {
        const int ncols = (int)std::min<int64_t>(cb, (n - c0 + 7) / 8 * 8);
        const int npairs = ncols / 2;
        PassAParams pa{a,     lda,          m_local, row_offset, M, M1, signs, (int)c0, ncols, (int)n, y,
                       level, overflow_flag_dev, tw_n2};
        fft_pass_a<<<dim3((unsigned)(M1 / 2), (unsigned)(ncols / 8)), A_THREADS, smem_a, st>>>(pa);
        SK_LAUNCH_CHECK("fft_pass_a");
        PassBParams pb{y, M1, d_ptr, d_s, d_w, d_k1, npairs, zbuf, (int)d, tw_m1};
        fft_pass_b<<<dim3((unsigned)N2, (unsigned)((npairs + B_PAIRS - 1) / B_PAIRS)), B_THREADS, smem_b, st>>>(pb);
        SK_LAUNCH_CHECK("fft_pass_b");
        const int64_t total = d * (int64_t)npairs;
        fft_finalize<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(zbuf, npairs, rows, (int)d, M, (int)c0,
                                                                     (int)n, out, ldo, accumulate);
        SK_LAUNCH_CHECK("fft_finalize");
    }
    return SK_OK;
}

}  // namespace sk
