// FP64 Gram products G = X^T Y on the INT8 tensor cores (tcgen05 kind::i8):
// Ozaki scheme II, i.e. exact integer products modulo up to 16 coprime moduli and a
// Chinese-remainder reconstruction.
//
// Same call sites as gram.cu (`a.T @ a` src/precision.py:230, `a_p.T @ a_p`
// src/solvers.py:230, `a_p.T @ a` :251, `b_matrix.T @ a` :164).  B200 has ~3.1 POPS
// of dense INT8 against 35 TFLOP/s of FP64 DMMA; 14-16 INT8 products replace one FP64
// product.
//
//   1. column scales: e_i with max_k |X[k,i]| < 2^e_i (one pass over X and Y)
//   2. per K-chunk of rows: X'[k,i] = rint(X[k,i] 2^(t - e_i)), |X'| <= 2^t, an exact
//      integer; its residues modulo p_1..p_nm (odd, pairwise coprime, <= 255) as
//      signed bytes in [-127, 127], nm planes per operand, row-major like X
//   3. per (modulus, K split <= 131072 rows, 256x256 output tile): one tcgen05 INT8
//      GEMM with int32 accumulation in TMEM (|sum| < 131072 * 127^2 < 2^31: exact);
//      both operands MN-major, TMA-staged with 128-byte swizzle
//   4. residues of the int32 partials summed modulo p
//   5. Garner mixed-radix reconstruction of C' = X'^T Y' (|C'| < M/2, M = prod p) in
//      128-bit integers, G = C' 2^(e_i + f_j - 2t).
//
// Error: only step 2 rounds (|X' - X 2^(t-e)| <= 1/2), so |G - X^T Y|_ij <=
// 2^-t (2^e_i sum_k |Y_kj| + 2^f_j sum_k |X_ki|) / 2 (+ the final rounding).  nm and t
// come from gram_moduli: the worst case stays 2^8 under the FP64 GEMM's gamma_K bound
// (m = 4M rows: nm = 15, t = 47).  The SYRK path computes lower tiles only; C' is
// exactly symmetric, so G is too.
#include <math_constants.h>

#include <vector>

#include "tc.cuh"

namespace sk {
namespace oz {

constexpr int NMOD = 16;
// the moduli as a constexpr function (folds to immediates inside unrolled loops)
__host__ __device__ constexpr int pm(int k) {
    return k == 0 ? 255 : k == 1 ? 253 : k == 2 ? 251 : k == 3 ? 247 : k == 4 ? 241 : k == 5 ? 239 : k == 6 ? 233
         : k == 7 ? 229 : k == 8 ? 227 : k == 9 ? 223 : k == 10 ? 217 : k == 11 ? 211 : k == 12 ? 199
         : k == 13 ? 197 : k == 14 ? 193 : 191;
}

__host__ __device__ constexpr uint32_t c1_of(int k) { return (uint32_t)((1ull << 17) % (uint64_t)pm(k)); }
__host__ __device__ constexpr uint32_t c2_of(int k) { return (uint32_t)((1ull << 34) % (uint64_t)pm(k)); }
__host__ __device__ constexpr uint32_t magic_of(int k) {
    return (uint32_t)(((1ull << 32) + pm(k) - 1) / (uint64_t)pm(k));
}
constexpr int inv_mod(int a, int p) {
    int t = 0, nt = 1, r = p, nr = a % p;
    while (nr != 0) {
        const int q = r / nr, tt = t - q * nt, rr = r - q * nr;
        t = nt; nt = tt; r = nr; nr = rr;
    }
    return t < 0 ? t + p : t;
}
// (p_0 ... p_{k-1})^{-1} mod p_k for Garner's mixed radix
constexpr int garner_of(int k) {
    int prod = 1;
    for (int j = 0; j < k; ++j) prod = (int)(((int64_t)prod * pm(j)) % pm(k));
    return inv_mod(prod, pm(k));
}

constexpr int BM = 256, UMMA_M = 128, BN = 256, BK = 128, STAGES = 3, UMMA_K = 32;
constexpr int THREADS = 384, EPI_WARP0 = 4;                 // warps 4..11 drain TMEM
constexpr uint32_t BOX_BYTES = 128 * BK;                     // one 128-col x BK-row int8 box
constexpr uint32_t A_BYTES = 2 * BOX_BYTES, B_BYTES = 2 * BOX_BYTES;
constexpr size_t SMEM = 1024 + STAGES * (A_BYTES + B_BYTES) + 256;
constexpr int64_t KSPLIT_MAX = 131072;                       // int32-exact accumulation length

// ---------------------------------------------------------- column scales ---
// Column statistics in one pass, deterministic: a fixed grid of STAT_BLOCKS row
// blocks writes per-block (max |x|, sum x^2) partials, reduced in block order.
// max feeds the scales; max^2 m / sum x^2 is the guard (below).  fmax propagates a NaN
// only from its second operand, so non-finite entries are kept sticky explicitly.
// With v != NULL the same pass also forms X^T v (the PNE/HPNE right-hand side A_p^T b),
// so the Gram's column scan doubles as its GEMV.
constexpr int STAT_BLOCKS = 512;
__global__ void __launch_bounds__(256) colstats_kernel(const double *__restrict__ x, int64_t ldx, int64_t m, int n,
                                                       const double *__restrict__ v, double *__restrict__ part) {
    const int c = blockIdx.y * 256 + threadIdx.x;
    if (c >= n) return;
    double mx = 0.0, ss = 0.0, dt = 0.0;
    const int64_t g = gridDim.x;
    int64_t r = blockIdx.x;
    for (; r + 3 * g < m; r += 4 * g) {   // four independent loads in flight
        const double a0 = x[r * ldx + c], a1 = x[(r + g) * ldx + c], a2 = x[(r + 2 * g) * ldx + c],
                     a3 = x[(r + 3 * g) * ldx + c];
        mx = fmax(fmax(mx, fmax(fabs(a0), fabs(a1))), fmax(fabs(a2), fabs(a3)));
        ss += (a0 * a0 + a1 * a1) + (a2 * a2 + a3 * a3);
        if (v) dt += (a0 * v[r] + a1 * v[r + g]) + (a2 * v[r + 2 * g] + a3 * v[r + 3 * g]);
        if (!isfinite(a0) || !isfinite(a1) || !isfinite(a2) || !isfinite(a3)) mx = CUDART_INF;
    }
    for (; r < m; r += g) {
        const double a = x[r * ldx + c];
        mx = isfinite(a) ? fmax(mx, fabs(a)) : CUDART_INF;
        ss += a * a;
        if (v) dt += a * v[r];
    }
    part[(size_t)blockIdx.x * n + c] = mx;
    part[((size_t)STAT_BLOCKS + blockIdx.x) * n + c] = ss;
    if (v) part[((size_t)2 * STAT_BLOCKS + blockIdx.x) * n + c] = dt;
}

__global__ void colstats_finalize(const double *__restrict__ part, int nblk, int n, int with_dot,
                                  double *__restrict__ stats) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n) return;
    double mx = 0.0, ss = 0.0, dt = 0.0;
    for (int b = 0; b < nblk; ++b) {
        const double v = part[(size_t)b * n + c];
        mx = (isfinite(v) && isfinite(mx)) ? fmax(mx, v) : CUDART_INF;
        ss += part[((size_t)STAT_BLOCKS + b) * n + c];
        if (with_dot) dt += part[((size_t)2 * STAT_BLOCKS + b) * n + c];
    }
    stats[c] = mx;
    stats[n + c] = ss;
    if (with_dot) stats[2 * n + c] = dt;
}

// max bits of the scales input (non-negative doubles order like their bit patterns)
__global__ void stats_to_bits(const double *__restrict__ stats, int n, unsigned long long *__restrict__ bits) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c < n) bits[c] = (unsigned long long)__double_as_longlong(stats[c]);
}

// Guard: the INT8 product's error bound 2^(1-t) (2^e_i sum|Y_j| + 2^f_j sum|X_i|) is
// within a factor 2 F of 2^-t ||X_i|| ||Y_j|| when max|X_i| sqrt(m) <= F ||X_i|| (sum|x|
// <= sqrt(m) ||x||, 2^e <= 2 max).  F = 64: at t = 51 the bound is 2^-43 ||X_i|| ||Y_j||,
// the size of an FP64 GEMM's typical error.  Columns spikier than that, or non-finite
// input, take the FP64 DMMA path.
constexpr double GUARD_F2 = 64.0 * 64.0;
__global__ void guard_kernel(const double *__restrict__ sx, const double *__restrict__ sy, int n, int64_t m,
                             int *flag) {
    __shared__ int bad;
    if (threadIdx.x == 0) bad = 0;
    __syncthreads();
    int b = 0;
    for (int c = threadIdx.x; c < n; c += blockDim.x) {
        const double *s[2] = {sx, sy};
        for (int o = 0; o < 2; ++o) {
            const double mx = s[o][c], ss = s[o][n + c];
            if (!isfinite(mx) || !isfinite(ss)) b = 1;
            else if (mx > 0.0 && mx * mx * (double)m > GUARD_F2 * ss) b = 1;
        }
    }
    if (b) atomicOr(&bad, 1);
    __syncthreads();
    if (threadIdx.x == 0) *reinterpret_cast<volatile int *>(flag) = bad;
}

// e = exponent with max < 2^e; scale = 2^(t - e) (inputs), out_exp for the product
__global__ void scales_kernel(const unsigned long long *__restrict__ bits, int n, int t, double *__restrict__ scale,
                              int *__restrict__ expo) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n) return;
    const double mx = __longlong_as_double((long long)bits[c]);
    int e = 0;
    if (mx > 0.0) {
        frexp(mx, &e);            // mx = f 2^e, f in [0.5, 1) -> mx < 2^e
    }
    expo[c] = e;
    scale[c] = ldexp(1.0, t - e);
}

// ------------------------------------------------------------- residues -----
// X' = h3 2^39 + h2 2^26 + h1 2^13 + h0 with balanced 13-bit limbs |h| <= 2^12 (exact
// FP64 splitting), so X' mod p = (h3 c3 + h2 c2 + h1 c1 + h0) mod p with centred
// c_j = 2^(13 j) mod p in [-127, 127]: |v| <= 1.56e6, exact in FP32.  q = round(v / p)
// by the 1.5 2^23 magic (v inv_p is within 5e-4 of v / p, and v / p is at least 1/510
// from a half-integer since p is odd), r = v - q p exact and already centred.
__host__ __device__ constexpr int centred_pow2_mod(int e, int k) {
    const int r = (int)((1ull << e) % (uint64_t)pm(k));
    return r > (pm(k) - 1) / 2 ? r - pm(k) : r;
}
constexpr float FMAGIC = 12582912.0f;   // 1.5 * 2^23

__device__ __forceinline__ uint32_t residue_byte(float h0, float h1, float h2, float h3, int k) {
    const float v = fmaf(h3, (float)centred_pow2_mod(39, k),
                         fmaf(h2, (float)centred_pow2_mod(26, k), fmaf(h1, (float)centred_pow2_mod(13, k), h0)));
    const float q = fmaf(v, 1.0f / (float)pm(k), FMAGIC) - FMAGIC;
    const float r = fmaf(-q, (float)pm(k), v);
    return __float_as_uint(r + FMAGIC);     // low byte = r as a two's-complement int8
}

// The same for two elements at once on the packed FP32x2 pipe (FFMA2 / FADD2, sm_100).
__device__ __forceinline__ uint64_t f2pack(float a, float b) {
    return (uint64_t)__float_as_uint(a) | ((uint64_t)__float_as_uint(b) << 32);
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
    uint64_t d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
// returns the two residue bytes in bits 0-7 and 32-39
__device__ __forceinline__ uint64_t residue_pair(uint64_t h0, uint64_t h1, uint64_t h2, uint64_t h3, int k) {
    const float c1 = (float)centred_pow2_mod(13, k), c2 = (float)centred_pow2_mod(26, k),
                c3 = (float)centred_pow2_mod(39, k), p = (float)pm(k), ip = 1.0f / (float)pm(k);
    const uint64_t v = ffma2(h3, f2pack(c3, c3), ffma2(h2, f2pack(c2, c2), ffma2(h1, f2pack(c1, c1), h0)));
    const uint64_t q = fadd2(ffma2(v, f2pack(ip, ip), f2pack(FMAGIC, FMAGIC)), f2pack(-FMAGIC, -FMAGIC));
    const uint64_t r = ffma2(q, f2pack(-p, -p), v);
    return fadd2(r, f2pack(FMAGIC, FMAGIC));
}

// 8 consecutive columns of one row per thread -> 16 planes of 8 bytes.  Rows are
// walked grid-stride; a block covers 256 column groups (one row of n = 2048, or
// several rows of narrower matrices), so no 64-bit division per item.
constexpr int RV = 8;
#ifndef SK_OZ_RES_MINB
#define SK_OZ_RES_MINB 4   // <= 64 registers, no spills
#endif
__global__ void __launch_bounds__(256, SK_OZ_RES_MINB)
residues_kernel(const double *__restrict__ x, int64_t ldx, int64_t rows, int n, const double *__restrict__ scale,
                int8_t *__restrict__ out, int64_t ldr, int64_t plane, int vec, int nm) {
    const int cpr = (n + RV - 1) / RV;
    const int rpi = cpr >= 256 ? 1 : 256 / cpr;
    const int sub = cpr >= 256 ? 0 : threadIdx.x / cpr;
    const int cfirst = cpr >= 256 ? threadIdx.x : threadIdx.x % cpr;
    const int cstep = cpr >= 256 ? 256 : cpr;
    for (int64_t r0 = (int64_t)blockIdx.x * rpi; r0 < rows; r0 += (int64_t)gridDim.x * rpi) {
        const int64_t r = r0 + sub;
        if (sub >= rpi || r >= rows) continue;
        for (int ch = cfirst; ch < cpr; ch += cstep) {
            const int c0 = ch * RV;
            const double *src = x + r * ldx + c0;
            double v[RV];
            if (vec && c0 + RV <= n) {
#pragma unroll
                for (int q = 0; q < RV / 2; ++q) {
                    const double2 d = __ldcs(reinterpret_cast<const double2 *>(src) + q);
                    v[2 * q] = d.x;
                    v[2 * q + 1] = d.y;
                }
            } else {
#pragma unroll
                for (int q = 0; q < RV; ++q) v[q] = c0 + q < n ? src[q] : 0.0;
            }
            float h0[RV], h1[RV], h2[RV], h3[RV];
#pragma unroll
            for (int q = 0; q < RV; ++q) {
                const double s = c0 + q < n ? __ldg(scale + c0 + q) : 0.0;
                const double xs = rint(v[q] * s);                 // |xs| <= 2^t <= 2^51, exact
                const double a3 = rint(xs * 0x1p-39);
                const double r3 = fma(-a3, 0x1p39, xs);
                const double a2 = rint(r3 * 0x1p-26);
                const double r2 = fma(-a2, 0x1p26, r3);
                const double a1 = rint(r2 * 0x1p-13);
                h3[q] = (float)a3;
                h2[q] = (float)a2;
                h1[q] = (float)a1;
                h0[q] = (float)fma(-a1, 0x1p13, r2);
            }
            int8_t *dst = out + r * ldr + c0;
            uint64_t p0[RV / 2], p1[RV / 2], p2[RV / 2], p3[RV / 2];
#pragma unroll
            for (int q = 0; q < RV / 2; ++q) {
                p0[q] = f2pack(h0[2 * q], h0[2 * q + 1]);
                p1[q] = f2pack(h1[2 * q], h1[2 * q + 1]);
                p2[q] = f2pack(h2[2 * q], h2[2 * q + 1]);
                p3[q] = f2pack(h3[2 * q], h3[2 * q + 1]);
            }
#pragma unroll
            for (int k = 0; k < NMOD; ++k) {
                if (k >= nm) break;   // the first nm moduli (uniform)
                uint32_t w[2];
#pragma unroll
                for (int q4 = 0; q4 < 2; ++q4) {
                    uint32_t b[4];
#pragma unroll
                    for (int bb = 0; bb < 2; ++bb) {
                        const int q2 = 2 * q4 + bb;
                        const uint64_t rr = residue_pair(p0[q2], p1[q2], p2[q2], p3[q2], k);
                        b[2 * bb] = (uint32_t)rr;
                        b[2 * bb + 1] = (uint32_t)(rr >> 32);
                    }
                    w[q4] = __byte_perm(__byte_perm(b[0], b[1], 0x0040), __byte_perm(b[2], b[3], 0x0040), 0x5410);
                }
                *reinterpret_cast<uint2 *>(dst + k * plane) = make_uint2(w[0], w[1]);
            }
        }
    }
}

// ---------------------------------------------------------------- GEMM ------
struct GemmParams {
    int ntn, ntiles, splits, units, syrk, n;
    int64_t rows, kchunk;
    int32_t *acc;               // [mod][n][n] residues in [0, p)
    // product mode (blocked TRSM update): C = P Q, P K-major [mod][mrows][K], Q MN-major
    // [mod][K][nout]; residues of C stored as int8 planes out[mod][mrows][ldo]
    int64_t mrows, ldo, oplane;
    int nout;
    int8_t *out;
};

// lower-triangular tile list for SYRK: tile index -> (tm, tn) with tm >= tn
__device__ __forceinline__ void tile_coords(const GemmParams &p, int tile, int &tm, int &tn) {
    if (!p.syrk) {
        tm = tile / p.ntn;
        tn = tile % p.ntn;
    } else {
        int r = (int)((sqrtf(8.0f * tile + 1.0f) - 1.0f) * 0.5f);
        while ((r + 1) * (r + 2) / 2 <= tile) ++r;
        while (r * (r + 1) / 2 > tile) --r;
        tm = r;
        tn = tile - r * (r + 1) / 2;
    }
}

__device__ __forceinline__ void tma_load_3d(void *smem_dst, const CUtensorMap *map, uint64_t *bar, int x, int y,
                                            int z) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];\n" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
}

// int32 product value -> a residue modulo p in [-127, 127] (as a byte in bits 0-7).
// v = a 2^13 + b, t = a c13 + b with c13 = centred 2^13 mod p: |t| < 2^21 for |v| < 2^27
// (K <= 8192), so round(t / p) in FP32 is off by at most 2^-9.6 < 1 / (2p), r = t - q p.
__device__ __forceinline__ uint32_t i32_residue(int v, float fp, float fip, int c13) {
    const int t = (v >> 13) * c13 + (v & 8191);
    const float tf = (float)t;
    const float q = fmaf(tf, fip, FMAGIC) - FMAGIC;
    return __float_as_uint(fmaf(-q, fp, tf) + FMAGIC);
}

template <bool PROD>
__global__ void __launch_bounds__(PROD ? 640 : THREADS, 1)
gemm_kernel(const __grid_constant__ CUtensorMap tmap_x, const __grid_constant__ CUtensorMap tmap_y,
            const GemmParams p) {
    constexpr int NTHR = PROD ? 640 : THREADS;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *sa = smem;
    uint8_t *sb = smem + STAGES * A_BYTES;
    uint64_t *full = reinterpret_cast<uint64_t *>(sb + STAGES * B_BYTES);
    uint64_t *empty = full + STAGES;
    uint64_t *tfull = empty + STAGES;
    uint64_t *tempty = tfull + 1;                                   // [2] in product mode
    uint32_t *tslot = reinterpret_cast<uint32_t *>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int NEPI = (NTHR / 32) - EPI_WARP0;
    if (warp == 0 && lane == 0) {
        for (int s = 0; s < STAGES; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&empty[s], 1);
        }
        tc::mbar_init(tfull, 1);
        tc::mbar_init(tempty, NEPI);
        tc::mbar_init(tempty + 1, NEPI);
        tc::mbar_fence_init();
        tc::tma_prefetch_desc(&tmap_x);
        tc::tma_prefetch_desc(&tmap_y);
    }
    if (warp == 2) tc::tmem_alloc<512>(tslot);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = *tslot;

    auto unit_coords = [&](int u, int &mod, int &split, int &tile, int64_t &k0, int &nkb) {
        tile = u % p.ntiles;
        const int rest = u / p.ntiles;
        split = rest % p.splits;
        mod = rest / p.splits;
        k0 = (int64_t)split * p.kchunk;
        const int64_t k1 = min(p.rows, k0 + p.kchunk);
        nkb = (int)((k1 - k0 + BK - 1) / BK);
    };

    if (warp == 0) {
        if (lane == 0) {   // ------------------------------------------ TMA producer
            int stage = 0;
            unsigned phase = 0;
            for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
                int mod, split, tile, nkb, tm, tn;
                int64_t k0;
                unit_coords(u, mod, split, tile, k0, nkb);
                tile_coords(p, tile, tm, tn);
                for (int kb = 0; kb < nkb; ++kb) {
                    tc::mbar_wait(&empty[stage], phase ^ 1);
                    tc::mbar_arrive_expect_tx(&full[stage], A_BYTES + B_BYTES);
                    const int krow = (int)(k0 + (int64_t)kb * BK);
                    uint8_t *a_dst = sa + stage * A_BYTES, *b_dst = sb + stage * B_BYTES;
                    if constexpr (PROD) {   // K-major P: box = 128 K bytes x 128 rows
                        tma_load_3d(a_dst, &tmap_x, &full[stage], krow, tm * BM, mod);
                        tma_load_3d(a_dst + BOX_BYTES, &tmap_x, &full[stage], krow, tm * BM + 128, mod);
                    } else {
                        tma_load_3d(a_dst, &tmap_x, &full[stage], tm * BM, krow, mod);
                        tma_load_3d(a_dst + BOX_BYTES, &tmap_x, &full[stage], tm * BM + 128, krow, mod);
                    }
                    tma_load_3d(b_dst, &tmap_y, &full[stage], tn * BN, krow, mod);
                    tma_load_3d(b_dst + BOX_BYTES, &tmap_y, &full[stage], tn * BN + 128, krow, mod);
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {   // --------------------------------------------- MMA issuer
            constexpr uint32_t idesc = tc::idesc_s32acc_s8(UMMA_M, BN, PROD ? 0 : 1, 1);
            int stage = 0;
            unsigned phase = 0, tphase = 0;
            for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
                int mod, split, tile, nkb;
                int64_t k0;
                unit_coords(u, mod, split, tile, k0, nkb);
                if constexpr (PROD) {
                    // Accumulator 0 is released by the epilogue before accumulator 1: issue
                    // accumulator 0's MMAs for the first (resident) stages as soon as it is
                    // free, then accumulator 1's for the same stages once that is free too,
                    // so the tile's main loop starts under the previous tile's epilogue.
                    const int pre = nkb < STAGES ? nkb : STAGES;
                    const int st0 = stage;
                    const unsigned ph0 = phase;
                    tc::mbar_wait(tempty, tphase ^ 1);
                    tc::tc_fence_after();
                    for (int kb = 0; kb < pre; ++kb) {
                        tc::mbar_wait(&full[stage], phase);
                        tc::tc_fence_after();
                        const uint64_t ad0 = tc::desc_kmajor_sw128(smem_u32(sa + stage * A_BYTES));
                        const uint64_t bd = tc::desc_mnmajor_sw128(smem_u32(sb + stage * B_BYTES), BOX_BYTES, 1024);
#pragma unroll
                        for (int k = 0; k < BK / UMMA_K; ++k)
                            tc::mma_i8_ss(tmem, ad0 + (uint64_t)(UMMA_K >> 4) * k,
                                          bd + (uint64_t)((UMMA_K * 128) >> 4) * k, idesc, (kb | k) ? 1u : 0u);
                        if (++stage == STAGES) { stage = 0; phase ^= 1; }
                    }
                    tc::mbar_wait(tempty + 1, tphase ^ 1);
                    tc::tc_fence_after();
                    stage = st0;
                    phase = ph0;
                    for (int kb = 0; kb < pre; ++kb) {
                        const uint64_t ad1 = tc::desc_kmajor_sw128(smem_u32(sa + stage * A_BYTES) + BOX_BYTES);
                        const uint64_t bd = tc::desc_mnmajor_sw128(smem_u32(sb + stage * B_BYTES), BOX_BYTES, 1024);
#pragma unroll
                        for (int k = 0; k < BK / UMMA_K; ++k)
                            tc::mma_i8_ss(tmem + BN, ad1 + (uint64_t)(UMMA_K >> 4) * k,
                                          bd + (uint64_t)((UMMA_K * 128) >> 4) * k, idesc, (kb | k) ? 1u : 0u);
                        tc::mma_commit(&empty[stage]);
                        if (++stage == STAGES) { stage = 0; phase ^= 1; }
                    }
                } else {
                    tc::mbar_wait(tempty, tphase ^ 1);
                    tc::tc_fence_after();
                }
                for (int kb = PROD ? (nkb < STAGES ? nkb : STAGES) : 0; kb < nkb; ++kb) {
                    tc::mbar_wait(&full[stage], phase);
                    tc::tc_fence_after();
                    const uint32_t a0 = smem_u32(sa + stage * A_BYTES), b0 = smem_u32(sb + stage * B_BYTES);
                    // MN-major SW128: 128-element MN blocks BOX_BYTES apart, 8-row K groups 1 KB apart
                    // K-major SW128 (product mode): 128-B K rows, advance 32 B per K step
                    const uint64_t ad0 = PROD ? tc::desc_kmajor_sw128(a0) : tc::desc_mnmajor_sw128(a0, BOX_BYTES, 1024);
                    const uint64_t ad1 = PROD ? tc::desc_kmajor_sw128(a0 + BOX_BYTES)
                                              : tc::desc_mnmajor_sw128(a0 + BOX_BYTES, BOX_BYTES, 1024);
                    const uint64_t bd = tc::desc_mnmajor_sw128(b0, BOX_BYTES, 1024);
#pragma unroll
                    for (int k = 0; k < BK / UMMA_K; ++k) {   // +32 K rows = 4 KB per step
                        const uint64_t adv = (uint64_t)((UMMA_K * 128) >> 4) * k;
                        const uint64_t aadv = PROD ? (uint64_t)(UMMA_K >> 4) * k : adv;
                        tc::mma_i8_ss(tmem, ad0 + aadv, bd + adv, idesc, (kb | k) ? 1u : 0u);
                        tc::mma_i8_ss(tmem + BN, ad1 + aadv, bd + adv, idesc, (kb | k) ? 1u : 0u);
                    }
                    tc::mma_commit(&empty[stage]);
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
                tc::mma_commit(tfull);
                tphase ^= 1;
            }
        }
    } else if (warp >= EPI_WARP0) {
        // ------------------------------------------------------------- epilogue
        // warp w drains TMEM lanes 32*(w%4); warps 4-7 accumulator 0, 8-11 accumulator 1
        const int lg = warp & 3, acc = ((warp - EPI_WARP0) >> 2) & 1;
        unsigned tphase = 0;
        for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
            int mod, split, tile, nkb;
            int64_t k0;
            unit_coords(u, mod, split, tile, k0, nkb);
            tc::mbar_wait(tfull, tphase);
            tc::tc_fence_after();
            tphase ^= 1;
            if constexpr (PROD) {
                // 16 warps = (lane quadrant, 64-column quarter); all of them drain
                // accumulator 0 first and release it (tempty[0]), then accumulator 1
                // (tempty[1]), so the next tile's MMAs start under this epilogue
                int tm, tn;
                tile_coords(p, tile, tm, tn);
                const int cq = (warp - EPI_WARP0) >> 2;
                const int pmod = pm(mod);
                const float fp = (float)pmod, fip = 1.0f / fp;
                const int c13 = (int)((8192 % pmod) > (pmod - 1) / 2 ? (8192 % pmod) - pmod : 8192 % pmod);
#pragma unroll 1
              for (int acc2 = 0; acc2 < 2; ++acc2) {
                const int64_t row = (int64_t)tm * BM + acc2 * UMMA_M + lg * 32 + lane;
                int8_t *dst_row = p.out + (size_t)mod * p.oplane + (size_t)row * p.ldo;
#pragma unroll 1
                for (int cb = cq * 2; cb < cq * 2 + 2; ++cb) {
                    uint32_t v[32];
                    tc::tmem_ld_32x32b_x32(tmem + ((uint32_t)(lg * 32) << 16) + (uint32_t)(acc2 * BN + cb * 32), v);
                    tc::tmem_ld_wait();
                    const int col0 = tn * BN + cb * 32;
                    if (row < p.mrows && col0 < p.nout) {
                        uint32_t w[8];
                        if (p.rows <= 1024) {
                            // |v| <= 1024 * 127^2 < 2^24: exact in FP32; two rounding steps on
                            // FFMA2 (the first quotient may be off by one) leave |r| <= p/2
                            const uint64_t ip2 = f2pack(fip, fip), mp2 = f2pack(-fp, -fp),
                                           mg = f2pack(FMAGIC, FMAGIC), nmg = f2pack(-FMAGIC, -FMAGIC);
#pragma unroll
                            for (int q4 = 0; q4 < 8; ++q4) {
                                uint32_t b[4];
#pragma unroll
                                for (int hh = 0; hh < 2; ++hh) {
                                    const uint64_t f = f2pack((float)(int)v[4 * q4 + 2 * hh],
                                                              (float)(int)v[4 * q4 + 2 * hh + 1]);
                                    const uint64_t r1 = ffma2(fadd2(ffma2(f, ip2, mg), nmg), mp2, f);
                                    const uint64_t r2 = ffma2(fadd2(ffma2(r1, ip2, mg), nmg), mp2, r1);
                                    const uint64_t rb = fadd2(r2, mg);
                                    b[2 * hh] = (uint32_t)rb;
                                    b[2 * hh + 1] = (uint32_t)(rb >> 32);
                                }
                                w[q4] = __byte_perm(__byte_perm(b[0], b[1], 0x0040), __byte_perm(b[2], b[3], 0x0040),
                                                    0x5410);
                            }
                        } else {
#pragma unroll
                            for (int q4 = 0; q4 < 8; ++q4) {
                                const uint32_t b0 = i32_residue((int)v[4 * q4], fp, fip, c13),
                                               b1 = i32_residue((int)v[4 * q4 + 1], fp, fip, c13),
                                               b2 = i32_residue((int)v[4 * q4 + 2], fp, fip, c13),
                                               b3 = i32_residue((int)v[4 * q4 + 3], fp, fip, c13);
                                w[q4] = __byte_perm(__byte_perm(b0, b1, 0x0040), __byte_perm(b2, b3, 0x0040),
                                                    0x5410);
                            }
                        }
                        int8_t *dst = dst_row + col0;
                        if (col0 + 32 <= p.nout) {
                            reinterpret_cast<uint4 *>(dst)[0] = make_uint4(w[0], w[1], w[2], w[3]);
                            reinterpret_cast<uint4 *>(dst)[1] = make_uint4(w[4], w[5], w[6], w[7]);
                        } else {
                            for (int q = 0; q < p.nout - col0; ++q) dst[q] = (int8_t)(w[q >> 2] >> (8 * (q & 3)));
                        }
                    }
                }
                tc::tc_fence_before();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(tempty + acc2);
              }
                continue;
            }
            // acc[mod][row][col] = (acc + C_partial) mod p, in [0, p): one unit per
            // (modulus, tile) per launch, so no two CTAs touch the same entries
            int tm, tn;
            tile_coords(p, tile, tm, tn);
            const int pmod = pm(mod);
            const int row = tm * BM + acc * UMMA_M + lg * 32 + lane;
            int32_t *dst_row = p.acc + (size_t)mod * p.n * p.n + (size_t)row * p.n + (size_t)tn * BN;
#pragma unroll 1
            for (int cb = 0; cb < BN / 32; ++cb) {
                uint32_t v[32];
                tc::tmem_ld_32x32b_x32(tmem + ((uint32_t)(lg * 32) << 16) + (uint32_t)(acc * BN + cb * 32), v);
                tc::tmem_ld_wait();
                if (row < p.n) {
                    int32_t *dst = dst_row + cb * 32;
                    const int cols = min(32, p.n - (tn * BN + cb * 32));
                    if (cols == 32 && (p.n & 3) == 0) {
#pragma unroll
                        for (int q4 = 0; q4 < 8; ++q4) {
                            int4 o = reinterpret_cast<int4 *>(dst)[q4];
                            int *oo = reinterpret_cast<int *>(&o);
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                int s = (int)v[4 * q4 + e] % pmod + oo[e];
                                s += s < 0 ? pmod : 0;
                                s -= s >= pmod ? pmod : 0;
                                oo[e] = s;
                            }
                            reinterpret_cast<int4 *>(dst)[q4] = o;
                        }
                    } else {
#pragma unroll
                        for (int q = 0; q < 32; ++q) {
                            if (q >= cols) break;
                            int s = (int)v[q] % pmod + dst[q];
                            s += s < 0 ? pmod : 0;
                            s -= s >= pmod ? pmod : 0;
                            dst[q] = s;
                        }
                    }
                }
            }
            tc::tc_fence_before();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(tempty);
        }
    }
    tc::tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc::tc_fence_after();
        tc::tmem_dealloc<512>(tmem);
    }
}

// ------------------------------------------------------ modular reduction ----
// acc[mod][i][j] = (acc + sum_split part) mod p, in [0, p); SYRK: lower tiles only
__global__ void reduce_kernel(const int32_t *__restrict__ part, int splits, int ntiles, int ntn, int syrk, int n,
                              int32_t *__restrict__ acc) {
    const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t nn = (int64_t)n * n;
    if (idx >= nn * NMOD) return;
    const int mod = (int)(idx / nn);
    const int64_t e = idx - (int64_t)mod * nn;
    const int i = (int)(e / n), j = (int)(e % n);
    const int tm = i / BM, tn = j / BN;
    if (syrk && tm < tn) return;
    const int tile = syrk ? tm * (tm + 1) / 2 + tn : tm * ntn + tn;
    const int32_t *pp = part + ((size_t)mod * splits * ntiles + tile) * (size_t)(BM * BN) + (size_t)(j % BN) * BM +
                        (i % BM);
    int64_t s = acc[idx];
    for (int k = 0; k < splits; ++k) s += pp[(size_t)k * ntiles * (BM * BN)];
    int32_t p = 0;
#pragma unroll
    for (int k = 0; k < NMOD; ++k)
        if (k == mod) p = pm(k);
    int32_t r = (int32_t)(s % p);
    acc[idx] = r < 0 ? r + p : r;
}

// ------------------------------------------------------- reconstruction -----
__global__ void crt_kernel(const int32_t *__restrict__ acc, int n, int syrk, const int *__restrict__ ex,
                           const int *__restrict__ ey, int t, double *__restrict__ g, int64_t ldg, int nm,
                           int accumulate) {
    const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t nn = (int64_t)n * n;
    if (idx >= nn) return;
    const int i = (int)(idx / n), j = (int)(idx % n);
    const int64_t src = (syrk && (i / BM) < (j / BN)) ? (int64_t)j * n + i : idx;   // mirror: C' symmetric
    int r[NMOD];
#pragma unroll
    for (int k = 0; k < NMOD; ++k) r[k] = k < nm ? acc[(int64_t)k * nn + src] : 0;
    // Garner over the first nm moduli: x = v0 + v1 p0 + v2 p0 p1 + ...
    int v[NMOD];
#pragma unroll
    for (int k = 0; k < NMOD; ++k) {
        if (k >= nm) { v[k] = 0; continue; }
        // x_{k} mod p_k from the digits so far (Horner, mod p_k)
        int acc_k = 0;
#pragma unroll
        for (int j2 = k - 1; j2 >= 0; --j2) acc_k = (acc_k * pm(j2) + v[j2]) % pm(k);
        int d = (r[k] - acc_k) % pm(k);
        d = d < 0 ? d + pm(k) : d;
        v[k] = (int)(((int64_t)d * garner_of(k)) % pm(k));
    }
    unsigned __int128 x = 0;
#pragma unroll
    for (int k = NMOD - 1; k >= 0; --k)
        if (k < nm) x = x * (unsigned)pm(k) + (unsigned)v[k];
    unsigned __int128 mprod = 1;
#pragma unroll
    for (int k = 0; k < NMOD; ++k)
        if (k < nm) mprod *= (unsigned)pm(k);
    const bool neg = x > (mprod >> 1);
    const unsigned __int128 mag = neg ? mprod - x : x;
    const double hi = (double)(unsigned long long)(mag >> 64), lo = (double)(unsigned long long)mag;
    double val = fma(hi, 18446744073709551616.0, lo);
    val = neg ? -val : val;
    const double out = ldexp(val, ex[i] + ey[j] - 2 * t);
    double *dst = g + (int64_t)i * ldg + j;
    *dst = accumulate ? *dst + out : out;   // row-chunked callers sum per-chunk Grams in FP64
}

// ================================================ blocked TRSM update (product) ==
// A_p[:, h:] = (A[:, h:] - A_p[:, :h] R[:h, h:]) R[h:, h:]^-1: the off-diagonal update
// C = P Q (P = A_p[:, :h] rows, Q = R[:h, h:]) on the INT8 engine.  Row scales for P
// (its rows are the output rows), column scales for Q, so the error is again
// 2^-t (2^e_r sum_k |Q_kj| + 2^f_j sum_k |P_rk|) / 2 per entry.

// P' = rint(P 2^(t - e_r)) with max_k |P[r, k]| < 2^e_r found in the same pass: 16
// K-major planes [mod][rows][ldk].  k % 256 == 0, so each row is whole warps.  Rows
// whose max^2 k > F^2 sum^2 (spiky) or with non-finite entries raise *flag.
__global__ void __launch_bounds__(256, SK_OZ_RES_MINB)
rowres_kernel(const double *__restrict__ x, int64_t ldx, int64_t rows, int k, int t, int8_t *__restrict__ out,
              int64_t ldk, int64_t plane, int *__restrict__ expo, int *flag, int nm) {
    __shared__ double smx[8], sss[8];
    const int cpr = k / RV, rpi = 256 / cpr, wpr = cpr / 32;
    const int sub = threadIdx.x / cpr, c0 = (threadIdx.x % cpr) * RV;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int64_t r0 = (int64_t)blockIdx.x * rpi; r0 < rows; r0 += (int64_t)gridDim.x * rpi) {
        const int64_t r = r0 + sub;
        const bool live = sub < rpi && r < rows;   // cpr need not divide 256 (h = 768)
        double v[RV];
        if (live) {
            const double *src = x + r * ldx + c0;
#pragma unroll
            for (int q = 0; q < RV / 2; ++q) {
                const double2 d = __ldcs(reinterpret_cast<const double2 *>(src) + q);
                v[2 * q] = d.x;
                v[2 * q + 1] = d.y;
            }
        } else {
#pragma unroll
            for (int q = 0; q < RV; ++q) v[q] = 0.0;
        }
        double mx = 0.0, ss = 0.0;
        bool bad = false;
#pragma unroll
        for (int q = 0; q < RV; ++q) {
            bad |= !isfinite(v[q]);
            mx = fmax(mx, fabs(v[q]));
            ss = fma(v[q], v[q], ss);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            ss += __shfl_xor_sync(0xffffffffu, ss, o);
        }
        bad = __any_sync(0xffffffffu, bad);
        if (lane == 0) {
            smx[warp] = bad ? CUDART_INF : mx;
            sss[warp] = ss;
        }
        __syncthreads();
        double rmx = 0.0, rss = 0.0;
        for (int w2 = sub * wpr; live && w2 < (sub + 1) * wpr; ++w2) {
            const double a = smx[w2];
            rmx = (isfinite(a) && isfinite(rmx)) ? fmax(rmx, a) : CUDART_INF;
            rss += sss[w2];
        }
        __syncthreads();
        if (!live) continue;
        int e = 0;
        const bool ok = isfinite(rmx) && isfinite(rss);
        if (ok && rmx > 0.0) frexp(rmx, &e);
        if (threadIdx.x % cpr == 0) {
            expo[r] = e;
            if (!ok || (rmx > 0.0 && rmx * rmx * (double)k > GUARD_F2 * rss)) atomicOr(flag, 1);
        }
        const double s = ldexp(1.0, t - e);
        float h0[RV], h1[RV], h2[RV], h3[RV];
#pragma unroll
        for (int q = 0; q < RV; ++q) {
            const double xs = ok ? rint(v[q] * s) : 0.0;
            const double a3 = rint(xs * 0x1p-39);
            const double r3 = fma(-a3, 0x1p39, xs);
            const double a2 = rint(r3 * 0x1p-26);
            const double r2 = fma(-a2, 0x1p26, r3);
            const double a1 = rint(r2 * 0x1p-13);
            h3[q] = (float)a3;
            h2[q] = (float)a2;
            h1[q] = (float)a1;
            h0[q] = (float)fma(-a1, 0x1p13, r2);
        }
        int8_t *dst = out + r * ldk + c0;
        uint64_t p0[RV / 2], p1[RV / 2], p2[RV / 2], p3[RV / 2];
#pragma unroll
        for (int q = 0; q < RV / 2; ++q) {
            p0[q] = f2pack(h0[2 * q], h0[2 * q + 1]);
            p1[q] = f2pack(h1[2 * q], h1[2 * q + 1]);
            p2[q] = f2pack(h2[2 * q], h2[2 * q + 1]);
            p3[q] = f2pack(h3[2 * q], h3[2 * q + 1]);
        }
#pragma unroll
        for (int kk = 0; kk < NMOD; ++kk) {
            if (kk >= nm) break;   // the first nm moduli (uniform)
            uint32_t w[2];
#pragma unroll
            for (int q4 = 0; q4 < 2; ++q4) {
                uint32_t b[4];
#pragma unroll
                for (int bb = 0; bb < 2; ++bb) {
                    const int q2 = 2 * q4 + bb;
                    const uint64_t rr = residue_pair(p0[q2], p1[q2], p2[q2], p3[q2], kk);
                    b[2 * bb] = (uint32_t)rr;
                    b[2 * bb + 1] = (uint32_t)(rr >> 32);
                }
                w[q4] = __byte_perm(__byte_perm(b[0], b[1], 0x0040), __byte_perm(b[2], b[3], 0x0040), 0x5410);
            }
            *reinterpret_cast<uint2 *>(dst + kk * plane) = make_uint2(w[0], w[1]);
        }
    }
}

// column guard of Q (same test as guard_kernel), OR-ed into *flag
__global__ void colguard_or_kernel(const double *__restrict__ s, int n, int64_t m, int *flag) {
    int b = 0;
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
        const double mx = s[c], ss = s[n + c];
        if (!isfinite(mx) || !isfinite(ss)) b = 1;
        else if (mx > 0.0 && mx * mx * (double)m > GUARD_F2 * ss) b = 1;
    }
    if (b) atomicOr(flag, 1);
}

// (M / p_k)^-1 mod p_k: literals (folded to immediates), checked against the definition
__host__ __device__ constexpr int crt_q(int k) {
    return k == 0 ? 124 : k == 1 ? 215 : k == 2 ? 217 : k == 3 ? 18 : k == 4 ? 119 : k == 5 ? 134 : k == 6 ? 223
         : k == 7 ? 51 : k == 8 ? 120 : k == 9 ? 174 : k == 10 ? 5 : k == 11 ? 6 : k == 12 ? 152 : k == 13 ? 117
         : k == 14 ? 13 : 135;
}
constexpr int crt_q_def(int k) {
    int prod = 1;
    for (int j = 0; j < NMOD; ++j)
        if (j != k) prod = (int)(((int64_t)prod * pm(j)) % pm(k));
    return inv_mod(prod, pm(k));
}
constexpr bool crt_q_ok() {
    for (int k = 0; k < NMOD; ++k)
        if (crt_q(k) != crt_q_def(k)) return false;
    return true;
}
static_assert(crt_q_ok(), "CRT inverse table");

// Reconstruction by the CRT sum: C' = sum_k y_k W_k - q M with W_k = M / p_k and
// y_k = r_k crt_q(k) - p_k round(r_k crt_q(k) / p_k) (any integer quotient gives a
// residue; |y_k| <= p_k / 2 + 1).  W_k = wa 2^76 + wr: sum y wa is exact in FP64
// (|sum| <= 16 M / 2^77 < 2^53), sum y wr (< 2^87) carries < 2^35 of rounding, far
// below the 2^(t+5) truncation error of C' itself; q = round(sum / M) is exact since
// |C'| < M / 2^12.  The residue arithmetic runs two columns at a time on FFMA2.
struct CrtSub {
    double wa[NMOD], wr[NMOD];
    float qf[NMOD], qip[NMOD];   // (M / p_k)^-1 mod p_k and that / p_k
    double ma, mr, rm;
    int nm;                      // moduli in use (the first nm): M = p_0 ... p_{nm-1}
};

__device__ __forceinline__ uint64_t fmul2(uint64_t a, uint64_t b) {
    uint64_t d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}

template <int NM>
__global__ void __launch_bounds__(256)
crt_sub_kernel(const int8_t *__restrict__ planes, int64_t plane, int64_t ldo, int64_t rows, int w,
               const int *__restrict__ er, const int *__restrict__ fq, int t, const double *__restrict__ a,
               int64_t lda, double *__restrict__ out, int64_t ldout, const CrtSub c) {
    constexpr float BIAS = 8388736.0f;   // 2^23 + 128: byte (r + 128) in a float's mantissa
    const int gpr = (w + 3) / 4;
    for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
        const int erow = er[r] - 2 * t;
        for (int g = threadIdx.x; g < gpr; g += blockDim.x) {
            const int j0 = g * 4;
            const int nc = min(4, w - j0);
            uint32_t pk[NMOD];
            const int8_t *src = planes + r * ldo + j0;
            const double *ar = a + r * lda + j0;
            double av[4];
            int ev[4];
            if (nc == 4) {
#pragma unroll
                for (int k = 0; k < NMOD; ++k)
                    pk[k] = k < NM ? __ldcs(reinterpret_cast<const uint32_t *>(src + k * plane)) : 0x80808080u;
                // A and the exponents in flight during the reconstruction (rows 32-byte aligned)
                const double2 a01 = __ldcs(reinterpret_cast<const double2 *>(ar)),
                              a23 = __ldcs(reinterpret_cast<const double2 *>(ar) + 1);
                av[0] = a01.x; av[1] = a01.y; av[2] = a23.x; av[3] = a23.y;
                const int4 f4 = __ldg(reinterpret_cast<const int4 *>(fq + j0));
                ev[0] = f4.x; ev[1] = f4.y; ev[2] = f4.z; ev[3] = f4.w;
            } else {
#pragma unroll
                for (int k = 0; k < NMOD; ++k) {
                    uint32_t x = 0;
                    for (int q = 0; q < nc && k < NM; ++q) x |= (uint32_t)(uint8_t)src[k * plane + q] << (8 * q);
                    pk[k] = x;
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    av[q] = q < nc ? ar[q] : 0.0;
                    ev[q] = q < nc ? fq[j0 + q] : 0;
                }
            }
            double s1[4] = {0.0, 0.0, 0.0, 0.0}, s2[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
            for (int k = 0; k < NMOD; ++k) {
                if (k >= NM) break;
                const uint32_t u = pk[k] ^ 0x80808080u;   // signed byte r -> r + 128
                const float p = (float)pm(k), q = c.qf[k], qip = c.qip[k];
#pragma unroll
                for (int h2 = 0; h2 < 2; ++h2) {
                    const uint64_t rr = fadd2(f2pack(__uint_as_float(__byte_perm(u, 0x4B000000u, 0x7540 + 2 * h2)),
                                                     __uint_as_float(__byte_perm(u, 0x4B000000u, 0x7541 + 2 * h2))),
                                              f2pack(-BIAS, -BIAS));
                    const uint64_t qq = fadd2(ffma2(rr, f2pack(qip, qip), f2pack(FMAGIC, FMAGIC)),
                                              f2pack(-FMAGIC, -FMAGIC));
                    const uint64_t y = ffma2(qq, f2pack(-p, -p), fmul2(rr, f2pack(q, q)));
                    const double y0 = (double)__uint_as_float((uint32_t)y), y1 = (double)__uint_as_float((uint32_t)(y >> 32));
                    s1[2 * h2] = fma(y0, c.wa[k], s1[2 * h2]);
                    s2[2 * h2] = fma(y0, c.wr[k], s2[2 * h2]);
                    s1[2 * h2 + 1] = fma(y1, c.wa[k], s1[2 * h2 + 1]);
                    s2[2 * h2 + 1] = fma(y1, c.wr[k], s2[2 * h2 + 1]);
                }
            }
            double res[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const double qq = rint(fma(s1[q], 0x1p76, s2[q]) * c.rm);
                const double v = fma(fma(-qq, c.ma, s1[q]), 0x1p76, fma(-qq, c.mr, s2[q]));
                const int e = erow + ev[q];
                // 2^e from its bits (|e| < 1000 always in practice; ldexp otherwise)
                const double sc = __longlong_as_double((long long)(e + 1023) << 52);
                res[q] = av[q] - ((e > -1000 && e < 1000) ? v * sc : ldexp(v, e));
            }
            double *orow = out + r * ldout + j0;
            if (nc == 4) {
                reinterpret_cast<double2 *>(orow)[0] = make_double2(res[0], res[1]);
                reinterpret_cast<double2 *>(orow)[1] = make_double2(res[2], res[3]);
            } else {
                for (int q = 0; q < nc; ++q) orow[q] = res[q];
            }
        }
    }
}

// -------------------------------------------------------------- planning ----
struct Plan {
    int ntm, ntn, ntiles, t, nm;
    int64_t chunk, kchunk, ldr;
    int splits;
    size_t res_bytes, part_bytes, acc_bytes, aux_bytes;
};

// Gram moduli: the fewest leading moduli with t >= 68 - log2 K (capped at 51), i.e. the
// INT8 product's worst-case bound 2^(7-t) ||X_i|| ||Y_j|| (guarded columns) stays 2^8
// below the FP64 GEMM's gamma_K ~ K u, and its typical error ~2^-t K^-1/2 ||X_i|| ||Y_j||
// under the blocked DMMA Gram's.  K = 2M-4M rows: 15 moduli, t = 47; K <= 2^17: 16, t = 51.
// (t = 43 with 14 moduli was measured: HPNE error 9.5e-15 against 2.7e-15 at kappa 10.)
int gram_moduli(int64_t m, int *t_out) {
    const double L = log2((double)std::max<int64_t>(m, 1));
    const int tmin = std::min(51, (int)ceil(68.0 - L));
    double lg = 0.0;
    for (int k = 0; k < NMOD; ++k) {
        lg += log2((double)pm(k));
        const int t = std::min(51, (int)floor((lg - 1.0 - L - 0.01) / 2.0));
        if (t >= tmin || k == NMOD - 1) {
            *t_out = t;
            return k + 1;
        }
    }
    *t_out = 51;
    return NMOD;
}

int choose_t(int64_t m) {
    double lg = 0.0;
    for (int k = 0; k < NMOD; ++k) lg += log2((double)pm(k));
    // |C'| <= m 2^(2t) must stay below M/2
    const int t = (int)floor((lg - 1.0 - log2((double)std::max<int64_t>(m, 1)) - 0.01) / 2.0);
    return std::min(t, 51);
}

Plan make_plan(int64_t m, int64_t n, bool syrk) {
    Plan p;
    p.ntm = (int)((n + BM - 1) / BM);
    p.ntn = p.ntm;
    p.ntiles = syrk ? p.ntm * (p.ntm + 1) / 2 : p.ntm * p.ntn;
    p.nm = gram_moduli(m, &p.t);
    p.ldr = (n + 15) / 16 * 16;
    p.kchunk = KSPLIT_MAX;
    p.chunk = std::min<int64_t>((m + BK - 1) / BK * BK, KSPLIT_MAX);
    p.splits = (int)((p.chunk + p.kchunk - 1) / p.kchunk);
    const int ops = syrk ? 1 : 2;
    p.res_bytes = (size_t)2 * ops * NMOD * p.chunk * p.ldr;   // double-buffered chunks
    p.part_bytes = 0;   // the GEMM epilogue accumulates modulo p straight into acc
    p.acc_bytes = (size_t)NMOD * n * n * sizeof(int32_t);
    // bits / scales / exponents (6n words), column stats of X and Y (4n), stats partials
    p.aux_bytes = (size_t)(10 * n + 3 * STAT_BLOCKS * n) * 8 + 8192;
    return p;
}

size_t align_up256(size_t b) { return (b + 255) & ~size_t(255); }

// per (host thread, device) side stream + events of the residue/GEMM pipeline
struct SidePipe {
    bool ok = false;
    cudaStream_t side = nullptr, hi = nullptr;   // residues (lowest priority), GEMMs (highest)
    cudaEvent_t start = nullptr, end = nullptr, res_done[2] = {nullptr, nullptr}, gemm_done[2] = {nullptr, nullptr};
};

SidePipe &side_pipe() {
    thread_local SidePipe pipes[64];
    int dev = 0;
    cudaGetDevice(&dev);
    SidePipe &sp = pipes[dev & 63];
    if (!sp.ok) {
        int least = 0, greatest = 0;
        cudaDeviceGetStreamPriorityRange(&least, &greatest);
        bool ok = cudaStreamCreateWithPriority(&sp.side, cudaStreamNonBlocking, least) == cudaSuccess;
        ok = ok && cudaStreamCreateWithPriority(&sp.hi, cudaStreamNonBlocking, greatest) == cudaSuccess;
        ok = ok && cudaEventCreateWithFlags(&sp.start, cudaEventDisableTiming) == cudaSuccess;
        ok = ok && cudaEventCreateWithFlags(&sp.end, cudaEventDisableTiming) == cudaSuccess;
        for (int i = 0; i < 2; ++i) {
            ok = ok && cudaEventCreateWithFlags(&sp.res_done[i], cudaEventDisableTiming) == cudaSuccess;
            ok = ok && cudaEventCreateWithFlags(&sp.gemm_done[i], cudaEventDisableTiming) == cudaSuccess;
        }
        sp.ok = ok;
    }
    return sp;
}

// ----------------------------------------------------- blocked TRSM plan -----
// update depth h: rowres_kernel spreads one row of P over its 256 threads x RV = 2048
// columns (and |int32 partials| < 2^27 needs h <= 8192), so h is capped at 2048; wider
// solves recurse on the right part with more updates
constexpr int64_t TRSM_KMAX = 2048;
// rows per update chunk (residue planes: 15 x chunk x (h + w) bytes); SK_TRSM_CHUNK overrides
int64_t trsm_chunk() {
    static const int64_t c = [] {
        const char *e = getenv("SK_TRSM_CHUNK");
        const int64_t v = e ? atoll(e) : 0;
        return v >= 256 ? v / 256 * 256 : (int64_t)65536;
    }();
    return c;
}

int64_t trsm_split(int64_t n) { return std::min<int64_t>((n / 2 + 255) / 256 * 256, TRSM_KMAX); }

struct TrsmPlan {
    int64_t chunk, hmax, wmax, ldw;
    size_t pres, ores, qres, aux;
};

TrsmPlan trsm_plan(int64_t m, int64_t n) {
    TrsmPlan p;
    p.hmax = trsm_split(n);            // the top level has the largest h and w
    p.wmax = n - p.hmax;
    p.ldw = (p.wmax + 15) / 16 * 16;
    p.chunk = std::min<int64_t>((std::max<int64_t>(m, 1) + 255) / 256 * 256, trsm_chunk());
    p.pres = (size_t)NMOD * p.chunk * p.hmax;
    p.ores = (size_t)NMOD * p.chunk * p.ldw;
    p.qres = (size_t)NMOD * p.hmax * p.ldw;
    // Q stats (2w) + bits (w) + scales (w) + exps (w ints) + P row exps (chunk ints) + partials
    p.aux = (size_t)(5 * p.wmax + p.chunk) * 8 + 3 * STAT_BLOCKS * (size_t)p.wmax * 8 + 8192;
    return p;
}

CrtSub make_crt_sub(int nm) {
    CrtSub c{};
    c.nm = nm;
    unsigned __int128 M = 1;
    for (int k = 0; k < nm; ++k) M *= (unsigned)pm(k);
    const unsigned __int128 low = (((unsigned __int128)1) << 76) - 1;
    auto dbl = [](unsigned __int128 v) {
        return (double)(uint64_t)(v >> 64) * 18446744073709551616.0 + (double)(uint64_t)v;
    };
    for (int k = 0; k < nm; ++k) {
        const unsigned __int128 W = M / (unsigned)pm(k);
        c.wa[k] = dbl(W >> 76);
        c.wr[k] = dbl(W & low);
        const int q = inv_mod((int)(W % (unsigned)pm(k)), pm(k));
        c.qf[k] = (float)q;
        c.qip[k] = (float)q / (float)pm(k);
    }
    c.ma = dbl(M >> 76);
    c.mr = dbl(M & low);
    c.rm = 1.0 / dbl(M);
    return c;
}

// fewest leading moduli whose product exceeds 2 K 2^(2t) (|C'| < M / 2 with margin)
int moduli_needed(int64_t K, int t) {
    double lg = 0.0;
    for (int k = 0; k < NMOD; ++k) {
        lg += log2((double)pm(k));
        if (lg - 1.0 - 0.01 >= 2.0 * t + log2((double)std::max<int64_t>(K, 1))) return k + 1;
    }
    return NMOD;
}

struct TrsmWs {
    int8_t *pres, *ores, *qres;
    double *qstats, *qscale;
    unsigned long long *bits;
    int *qexp, *pexp, *flag;
    void *statws;
    size_t statws_bytes;
    TrsmPlan plan;
    int64_t base;
};

}  // namespace oz

namespace gram {
int gram_f64_gated(const double *x, int64_t ldx, const double *y, int64_t ldy, int64_t m, int64_t n, double *g,
                   int64_t ldg, int accumulate, void *ws, size_t ws_bytes, sk_stream_t stream, const int *gate);
}  // namespace gram

namespace trsm {
int launch(const double *a, int64_t lda, int64_t m, int n, const double *r, int64_t ldr, double *ap, int64_t ldap,
           cudaStream_t st, const int *gate = nullptr);
int first_zero_diagonal(const double *r, int64_t ldr, int n, cudaStream_t st, int *out);
}  // namespace trsm

namespace oz {
// A_p[:, :n] = A R^-1 by recursive column halving: solve the left part, subtract its
// INT8 product with R[:h, h:] from the right part, solve the right part in place.
// Leaves of width <= base are the FP64 DMMA kernel.
// SK_TRSM_OZ_PROFILE=1: per-phase CUDA-event times to stderr (leaf solves, Q prep,
// row residues, INT8 products, reconstruction)
struct TrsmProf {
    std::vector<std::pair<int, cudaEvent_t>> ev;
    void mark(int phase, cudaStream_t st) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, st);
        ev.emplace_back(phase, e);
    }
    void report() {
        if (ev.empty()) return;
        cudaEventSynchronize(ev.back().second);
        static const char *names[] = {"leaf", "qprep", "rowres", "product", "crt"};
        float acc[5] = {0, 0, 0, 0, 0}, tot = 0, t;
        for (size_t i = 1; i < ev.size(); ++i) {
            cudaEventElapsedTime(&t, ev[i - 1].second, ev[i].second);
            if (ev[i].first >= 0) acc[ev[i].first] += t;
            tot += t;
        }
        fprintf(stderr, "trsm_ozaki: total %.2f ms", tot);
        for (int k = 0; k < 5; ++k) fprintf(stderr, ", %s %.2f", names[k], acc[k]);
        fprintf(stderr, "\n");
        for (auto &p : ev) cudaEventDestroy(p.second);
        ev.clear();
    }
};
TrsmProf *trsm_prof() {
    static const bool on = getenv("SK_TRSM_OZ_PROFILE") != nullptr;
    thread_local TrsmProf p;
    return on ? &p : nullptr;
}

int trsm_rec(const double *a, int64_t lda, double *ap, int64_t ldap, int64_t m, int64_t n, const double *r,
             int64_t ldr, const TrsmWs &W, cudaStream_t st) {
    TrsmProf *prof = trsm_prof();
    if (n <= W.base) {
        const int rc0 = trsm::launch(a, lda, m, (int)n, r, ldr, ap, ldap, st);
        if (prof) prof->mark(0, st);
        return rc0;
    }
    const int64_t h = trsm_split(n), w = n - h;
    int rc = trsm_rec(a, lda, ap, ldap, m, h, r, ldr, W, st);
    if (rc) return rc;
    const int sms = sm_count();
    const int t = choose_t(h);
    const int nm = std::max(15, moduli_needed(h, t));   // 15 at h = 1024, t = 51
    const CrtSub crt = make_crt_sub(nm);
    // Q = R[:h, h:]: column scales, guard, residues (MN-major B planes [mod][h][ldw])
    const double *q = r + h;
    rc = sk_colstats_f64(q, ldr, h, w, nullptr, W.qstats, W.statws, W.statws_bytes, st);
    if (rc) return rc;
    const unsigned wg = (unsigned)((w + 255) / 256);
    colguard_or_kernel<<<wg, 256, 0, st>>>(W.qstats, (int)w, h, W.flag);
    stats_to_bits<<<wg, 256, 0, st>>>(W.qstats, (int)w, W.bits);
    scales_kernel<<<wg, 256, 0, st>>>(W.bits, (int)w, t, W.qscale, W.qexp);
    const int64_t ldw = W.plan.ldw, qplane = h * ldw;
    {
        const int cpr = (int)((w + RV - 1) / RV);
        const int rpi = cpr >= 256 ? 1 : 256 / cpr;
        const int vq = ((reinterpret_cast<uintptr_t>(q) & 15) == 0) && (ldr % 2 == 0);
        residues_kernel<<<(unsigned)((h + rpi - 1) / rpi), 256, 0, st>>>(q, ldr, h, (int)w, W.qscale, W.qres, ldw,
                                                                          qplane, vq, nm);
        SK_LAUNCH_CHECK("oz trsm q residues");
    }
    if (prof) prof->mark(1, st);
    CUtensorMap tq;
    rc = make_tmap_3d(&tq, CU_TENSOR_MAP_DATA_TYPE_UINT8, W.qres, (uint64_t)w, (uint64_t)h, NMOD, (uint64_t)ldw,
                      (uint64_t)qplane, 128, BK, CU_TENSOR_MAP_SWIZZLE_128B);
    if (rc) return rc;
    const int64_t chunk = W.plan.chunk, pplane = chunk * h, oplane = chunk * ldw;
    SK_CUDA(cudaFuncSetAttribute(gemm_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM));
    for (int64_t r0 = 0; r0 < m; r0 += chunk) {
        const int64_t rows = std::min(chunk, m - r0);
        const int rpi = (int)(256 / (h / RV));
        rowres_kernel<<<(unsigned)std::min<int64_t>((rows + rpi - 1) / rpi, (int64_t)sms * 16), 256, 0, st>>>(
            ap + r0 * ldap, ldap, rows, (int)h, t, W.pres, h, pplane, W.pexp, W.flag, nm);
        SK_LAUNCH_CHECK("oz trsm row residues");
        if (prof) prof->mark(2, st);
        CUtensorMap tp;
        rc = make_tmap_3d(&tp, CU_TENSOR_MAP_DATA_TYPE_UINT8, W.pres, (uint64_t)h, (uint64_t)rows, NMOD, (uint64_t)h,
                          (uint64_t)pplane, BK, 128, CU_TENSOR_MAP_SWIZZLE_128B);
        if (rc) return rc;
        GemmParams gp{};
        gp.ntn = (int)((w + BN - 1) / BN);
        gp.ntiles = (int)((rows + BM - 1) / BM) * gp.ntn;
        gp.splits = 1;
        gp.units = nm * gp.ntiles;
        gp.syrk = 0;
        gp.rows = h;
        gp.kchunk = h;
        gp.mrows = rows;
        gp.ldo = ldw;
        gp.oplane = oplane;
        gp.nout = (int)w;
        gp.out = W.ores;
        gemm_kernel<true><<<std::min(gp.units, sms), 640, SMEM, st>>>(tp, tq, gp);
        SK_LAUNCH_CHECK("oz trsm product");
        if (prof) prof->mark(3, st);
        auto crt_fn = nm == 15 ? crt_sub_kernel<15> : crt_sub_kernel<16>;
        crt_fn<<<(unsigned)std::min<int64_t>(rows, (int64_t)sms * 8), 256, 0, st>>>(
            W.ores, oplane, ldw, rows, (int)w, W.pexp, W.qexp, t, a + r0 * lda + h, lda, ap + r0 * ldap + h, ldap,
            crt);
        SK_LAUNCH_CHECK("oz trsm reconstruction");
        if (prof) prof->mark(4, st);
    }
    return trsm_rec(ap + h, ldap, ap + h, ldap, m, w, r + h * ldr + h, ldr, W, st);
}

}  // namespace oz
}  // namespace sk

using namespace sk;

namespace {
thread_local int g_trsm_oz_fell_back = 0;
int *trsm_guard_slot() {   // mapped pinned flag: read on the host after one synchronize
    thread_local int *slot = nullptr;
    if (!slot) {
        void *p = nullptr;
        if (cudaHostAlloc(&p, sizeof(int), cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess) return nullptr;
        slot = static_cast<int *>(p);
    }
    return slot;
}
}  // namespace

extern "C" {

size_t sk_trsm_ozaki_workspace(int64_t m, int64_t n) {
    if (n < 2) return 256;
    oz::TrsmPlan p = oz::trsm_plan(m, n);
    return oz::align_up256(p.pres) + oz::align_up256(p.ores) + oz::align_up256(p.qres) + oz::align_up256(p.aux) +
           1024;
}

int sk_trsm_ozaki_fell_back(void) { return g_trsm_oz_fell_back; }

int sk_trsm_ozaki_f64(const double *a, int64_t lda, int64_t m, int64_t n, const double *r, int64_t ldr, double *ap,
                      int64_t ldap, sk_status *status, void *ws, size_t ws_bytes, sk_stream_t stream) {
    if (!a || !r || !ap || m < 0 || n <= 0 || lda < n || ldr < n || ldap < n || n > (1 << 20) || a == ap) {
        set_error("sk_trsm_ozaki_f64: bad arguments (a and a_p must be distinct)");
        return SK_ERR_ARG;
    }
    if (!ws || ws_bytes < sk_trsm_ozaki_workspace(m, n)) {
        set_error("sk_trsm_ozaki_f64: workspace %zu < %zu", ws_bytes, sk_trsm_ozaki_workspace(m, n));
        return SK_ERR_ARG;
    }
    cudaStream_t st = (cudaStream_t)stream;
    // deferred verdicts: zero diagonal recorded on the device; the spiky / non-finite
    // guard flag on the device past the workspace, the DMMA re-solve gated on it
    const bool defer = deferred_status() != nullptr;
    const size_t flag_off = sk_trsm_ozaki_workspace(m, n);
    int rc = SK_OK;
    if (defer) {
        if (ws_bytes < flag_off + 256) {
            set_error("sk_trsm_ozaki_f64: under deferred verdicts needs %zu workspace bytes", flag_off + 256);
            return SK_ERR_ARG;
        }
        rc = note_zero_diagonal(r, ldr, n, SK_SINGULAR_TRIANGULAR, st);
        if (rc) return rc;
    } else {
        int first_zero = 0;
        rc = trsm::first_zero_diagonal(r, ldr, (int)n, st, &first_zero);
        if (rc) return rc;
        if (first_zero != INT32_MAX) {
            set_error("zero diagonal entry at index %d", first_zero);
            return fill_status(status, SK_SINGULAR_TRIANGULAR, first_zero, 0.0, 0.0);
        }
    }
    g_trsm_oz_fell_back = 0;
    static const int64_t base = getenv("SK_TRSM_OZ_BASE") ? atoll(getenv("SK_TRSM_OZ_BASE")) : 1024;
    const bool aligned = ((reinterpret_cast<uintptr_t>(ap) | reinterpret_cast<uintptr_t>(r) |
                           reinterpret_cast<uintptr_t>(a)) % 16 == 0) &&
                         (ldap % 2 == 0) && (ldr % 2 == 0) && (lda % 2 == 0);
    if (m == 0 || n <= std::max<int64_t>(base, 256) || !aligned) {
        rc = trsm::launch(a, lda, m, (int)n, r, ldr, ap, ldap, st);
        if (rc) return rc;
        return fill_status(status, SK_OK, -1, 0, 0);
    }
    int *flag = defer ? reinterpret_cast<int *>(static_cast<uint8_t *>(ws) + flag_off) : trsm_guard_slot();
    if (!flag) {
        set_error("sk_trsm_ozaki_f64: pinned guard slot unavailable");
        return SK_ERR_CUDA;
    }
    if (defer) SK_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), st));
    else *reinterpret_cast<volatile int *>(flag) = 0;   // the stream is idle (synchronized above)
    oz::TrsmWs W;
    W.plan = oz::trsm_plan(m, n);
    uint8_t *w = static_cast<uint8_t *>(ws);
    W.pres = reinterpret_cast<int8_t *>(w);
    w += oz::align_up256(W.plan.pres);
    W.ores = reinterpret_cast<int8_t *>(w);
    w += oz::align_up256(W.plan.ores);
    W.qres = reinterpret_cast<int8_t *>(w);
    w += oz::align_up256(W.plan.qres);
    const int64_t wm = W.plan.wmax;
    W.qstats = reinterpret_cast<double *>(w);                  // 2 wmax
    W.qscale = W.qstats + 2 * wm;                              // wmax
    W.bits = reinterpret_cast<unsigned long long *>(W.qscale + wm);   // wmax
    W.qexp = reinterpret_cast<int *>(W.bits + wm);             // wmax ints (in a wmax-double slot)
    W.pexp = W.qexp + 2 * wm;                                  // chunk ints
    W.statws = reinterpret_cast<uint8_t *>(W.pexp + 2 * W.plan.chunk);
    W.statws = reinterpret_cast<void *>((reinterpret_cast<uintptr_t>(W.statws) + 255) & ~uintptr_t(255));
    W.statws_bytes = sk_colstats_workspace(wm);
    W.flag = flag;
    W.base = std::max<int64_t>(base, 256);
    if (oz::TrsmProf *prof = oz::trsm_prof()) prof->mark(-1, st);
    rc = oz::trsm_rec(a, lda, ap, ldap, m, n, r, ldr, W, st);
    if (rc) return rc;
    if (oz::TrsmProf *prof = oz::trsm_prof()) prof->report();
    if (defer) {   // spiky rows of A_p / columns of R, or non-finite values: the DMMA solve, gated
        rc = trsm::launch(a, lda, m, (int)n, r, ldr, ap, ldap, st, flag);
        if (rc) return rc;
        return fill_status(status, SK_OK, -1, 0, 0);
    }
    SK_CUDA(cudaStreamSynchronize(st));
    if (*reinterpret_cast<volatile int *>(flag)) {
        // spiky rows of A_p / columns of R, or non-finite values: redo on the DMMA path
        g_trsm_oz_fell_back = 1;
        rc = trsm::launch(a, lda, m, (int)n, r, ldr, ap, ldap, st);
        if (rc) return rc;
    }
    return fill_status(status, SK_OK, -1, 0, 0);
}

size_t sk_gram_ozaki_workspace(int64_t m, int64_t n, int syrk) {
    oz::Plan p = oz::make_plan(m, n, syrk != 0);
    return oz::align_up256(p.res_bytes) + oz::align_up256(p.part_bytes) + oz::align_up256(p.acc_bytes) +
           oz::align_up256(p.aux_bytes) + 1024;
}

size_t sk_colstats_workspace(int64_t n) { return (size_t)3 * oz::STAT_BLOCKS * n * sizeof(double) + 256; }

int sk_colstats_f64(const double *x, int64_t ldx, int64_t m, int64_t n, const double *v, double *stats, void *ws,
                    size_t ws_bytes, sk_stream_t stream) {
    if (!x || !stats || m < 0 || n <= 0 || ldx < n || !ws || ws_bytes < sk_colstats_workspace(n)) {
        set_error("sk_colstats_f64: bad arguments or workspace");
        return SK_ERR_ARG;
    }
    cudaStream_t st = (cudaStream_t)stream;
    if (m == 0) {
        SK_CUDA(cudaMemsetAsync(stats, 0, (size_t)(v ? 3 : 2) * n * sizeof(double), st));
        return SK_OK;
    }
    const int nblk = (int)std::min<int64_t>(m, oz::STAT_BLOCKS);
    double *part = static_cast<double *>(ws);
    oz::colstats_kernel<<<dim3((unsigned)nblk, (unsigned)((n + 255) / 256)), 256, 0, st>>>(x, ldx, m, (int)n, v,
                                                                                         part);
    SK_LAUNCH_CHECK("oz colstats");
    oz::colstats_finalize<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(part, nblk, (int)n, v != nullptr, stats);
    SK_LAUNCH_CHECK("oz colstats finalize");
    return SK_OK;
}

namespace {
thread_local int g_oz_fell_back = 0;
int *guard_slot() {
    thread_local int *slot = nullptr;
    if (!slot) {
        void *p = nullptr;
        if (cudaHostAlloc(&p, sizeof(int), cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess) return nullptr;
        slot = static_cast<int *>(p);
    }
    return slot;
}
}  // namespace

int sk_gram_ozaki_fell_back(void) { return g_oz_fell_back; }

int sk_gram_ozaki_f64(const double *x, int64_t ldx, const double *y, int64_t ldy, int64_t m, int64_t n, double *g,
                      int64_t ldg, void *ws, size_t ws_bytes, sk_stream_t stream) {
    return sk_gram_ozaki_ex_f64(x, ldx, y, ldy, m, n, nullptr, nullptr, g, ldg, ws, ws_bytes, stream);
}

int sk_gram_ozaki_ex_f64(const double *x, int64_t ldx, const double *y, int64_t ldy, int64_t m, int64_t n,
                         const double *xstats, const double *ystats, double *g, int64_t ldg, void *ws,
                         size_t ws_bytes, sk_stream_t stream) {
    return sk_gram_ozaki_acc_f64(x, ldx, y, ldy, m, n, xstats, ystats, g, ldg, 0, ws, ws_bytes, stream);
}

int sk_gram_ozaki_acc_f64(const double *x, int64_t ldx, const double *y, int64_t ldy, int64_t m, int64_t n,
                          const double *xstats, const double *ystats, double *g, int64_t ldg, int accumulate,
                          void *ws, size_t ws_bytes, sk_stream_t stream) {
    if (!x || !y || !g || m < 0 || n <= 0 || ldx < n || ldy < n || ldg < n || n > 65536) {
        set_error("sk_gram_ozaki_f64: bad arguments");
        return SK_ERR_ARG;
    }
    const bool syrk = (x == y) && (ldx == ldy);
    if (!ws || ws_bytes < sk_gram_ozaki_workspace(m, n, syrk)) {
        set_error("sk_gram_ozaki_f64: workspace %zu < %zu", ws_bytes, sk_gram_ozaki_workspace(m, n, syrk));
        return SK_ERR_ARG;
    }
    cudaStream_t st = (cudaStream_t)stream;
    oz::Plan p = oz::make_plan(m, n, syrk);
    uint8_t *w = static_cast<uint8_t *>(ws);
    int8_t *res = reinterpret_cast<int8_t *>(w);
    w += oz::align_up256(p.res_bytes);
    w += oz::align_up256(p.part_bytes);
    int32_t *acc = reinterpret_cast<int32_t *>(w);
    w += oz::align_up256(p.acc_bytes);
    unsigned long long *bits = reinterpret_cast<unsigned long long *>(w);   // 2n
    double *scale = reinterpret_cast<double *>(bits + 2 * n);                // 2n
    int *expo = reinterpret_cast<int *>(scale + 2 * n);                      // 2n (+ pad)
    double *stats = reinterpret_cast<double *>(w + oz::align_up256((size_t)6 * n * 8));   // 4n: x, y
    void *stat_ws = w + oz::align_up256((size_t)10 * n * 8);

    g_oz_fell_back = 0;
    const int sms = sm_count();
    const unsigned sgrid = (unsigned)((n + 255) / 256);
    // column statistics: given by the caller (sk_colstats_f64 of the same matrix) or a pass here
    const double *sx = xstats, *sy = syrk ? xstats : ystats;
    if (!sx) {
        int rc = sk_colstats_f64(x, ldx, m, n, nullptr, stats, stat_ws, sk_colstats_workspace(n), stream);
        if (rc) return rc;
        sx = stats;
        if (syrk) sy = stats;
    }
    if (!sy) {
        int rc = sk_colstats_f64(y, ldy, m, n, nullptr, stats + 2 * n, stat_ws, sk_colstats_workspace(n), stream);
        if (rc) return rc;
        sy = stats + 2 * n;
    }
    // deferred verdicts: the guard flag lives on the device, past both engines' workspace,
    // and the DMMA fallback runs gated on it after the INT8 product (which then computed
    // garbage that the fallback overwrites); no host read
    const bool defer = deferred_status() != nullptr;
    const size_t flag_off = std::max(sk_gram_ozaki_workspace(m, n, syrk), sk_gram_workspace(m, n));
    if (defer && (accumulate || ws_bytes < flag_off + 256)) {
        set_error("sk_gram_ozaki_f64: under deferred verdicts needs accumulate = 0 and %zu workspace bytes",
                  flag_off + 256);
        return SK_ERR_ARG;
    }
    int *flag = defer ? reinterpret_cast<int *>(static_cast<uint8_t *>(ws) + flag_off) : guard_slot();
    if (!flag) {
        set_error("sk_gram_ozaki_f64: pinned guard slot unavailable");
        return SK_ERR_CUDA;
    }
    oz::guard_kernel<<<1, 1024, 0, st>>>(sx, sy, (int)n, m, flag);
    SK_LAUNCH_CHECK("oz guard");
    if (!defer) SK_CUDA(cudaStreamSynchronize(st));
    if (!defer && *reinterpret_cast<volatile int *>(flag)) {
        // spiky columns or non-finite input: the FP64 DMMA Gram (same workspace)
        g_oz_fell_back = 1;
        if (ws_bytes < sk_gram_workspace(m, n)) {
            set_error("sk_gram_ozaki_f64: workspace too small for the DMMA fallback");
            return SK_ERR_ARG;
        }
        return sk_gram_f64(x, ldx, y, ldy, m, n, g, ldg, accumulate, ws, ws_bytes, stream);
    }
    oz::stats_to_bits<<<sgrid, 256, 0, st>>>(sx, (int)n, bits);
    oz::stats_to_bits<<<sgrid, 256, 0, st>>>(sy, (int)n, bits + n);
    SK_CUDA(cudaMemsetAsync(acc, 0, p.acc_bytes, st));
    oz::scales_kernel<<<sgrid, 256, 0, st>>>(bits, (int)n, p.t, scale, expo);
    oz::scales_kernel<<<sgrid, 256, 0, st>>>(bits + n, (int)n, p.t, scale + n, expo + n);
    SK_LAUNCH_CHECK("oz scales");

    const int vx = ((reinterpret_cast<uintptr_t>(x) & 15) == 0) && (ldx % 2 == 0);
    const int vy = ((reinterpret_cast<uintptr_t>(y) & 15) == 0) && (ldy % 2 == 0);
    const int64_t plane = p.chunk * p.ldr;
    const size_t buf_bytes = (size_t)(syrk ? 1 : 2) * oz::NMOD * plane;
    SK_CUDA(cudaFuncSetAttribute(oz::gemm_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)oz::SMEM));
    // Two-stream pipeline: the residues of chunk c+1 (ALU-bound, side stream) run
    // while the INT8 GEMM of chunk c (tensor-bound, caller's stream) runs; chunks
    // alternate between two residue buffers.
    oz::SidePipe &sp = oz::side_pipe();
    if (!sp.ok) {
        set_error("sk_gram_ozaki_f64: side stream unavailable");
        return SK_ERR_CUDA;
    }
    // Default: one stream.  SK_OZ_PIPELINE=1 runs residues (lowest priority) beside the
    // GEMMs (highest priority); measured no faster at config 3 (a GEMM CTA leaves room
    // for one or two residue blocks per SM, and both then compete for HBM and power).
    static const bool serial = getenv("SK_OZ_PIPELINE") == nullptr || getenv("SK_OZ_PROFILE") != nullptr;
    static const bool prof = getenv("SK_OZ_PROFILE") != nullptr;   // phase timing to stderr (serial mode)
    cudaStream_t rs = serial ? st : sp.side;   // residues: lowest priority
    cudaStream_t gs = serial ? st : sp.hi;     // GEMMs + reconstruction: highest priority
    std::vector<cudaEvent_t> pe;
    int npe = 0;
    if (prof) {
        pe.resize(2 * (size_t)((m + p.chunk - 1) / p.chunk) + 4);
        for (auto &e : pe) cudaEventCreate(&e);
        SK_CUDA(cudaEventRecord(pe[npe++], st));   // NB: recorded after colmax (launched above)
    }
    if (!serial) {
        SK_CUDA(cudaEventRecord(sp.start, st));
        SK_CUDA(cudaStreamWaitEvent(sp.side, sp.start, 0));
        SK_CUDA(cudaStreamWaitEvent(sp.hi, sp.start, 0));
    }
    int chunk_idx = 0;
    for (int64_t r0 = 0; r0 < m; r0 += p.chunk, ++chunk_idx) {
        const int buf = chunk_idx & 1;
        int8_t *res_x = res + buf * buf_bytes;
        int8_t *res_y = syrk ? res_x : res_x + (size_t)oz::NMOD * plane;
        const int64_t rows = std::min(p.chunk, m - r0);
        const int cpr = (int)((n + oz::RV - 1) / oz::RV);
        const int rpi = cpr >= 256 ? 1 : 256 / cpr;
        const unsigned rgrid = (unsigned)std::min<int64_t>((rows + rpi - 1) / rpi, (int64_t)sms * 16);
        if (prof) SK_CUDA(cudaEventRecord(pe[npe++], st));
        if (!serial && chunk_idx >= 2) SK_CUDA(cudaStreamWaitEvent(sp.side, sp.gemm_done[buf], 0));
        oz::residues_kernel<<<rgrid, 256, 0, rs>>>(x + r0 * ldx, ldx, rows, (int)n, scale, res_x, p.ldr, plane, vx,
                                                   p.nm);
        SK_LAUNCH_CHECK("oz residues");
        if (!syrk) {
            oz::residues_kernel<<<rgrid, 256, 0, rs>>>(y + r0 * ldy, ldy, rows, (int)n, scale + n, res_y, p.ldr,
                                                       plane, vy, p.nm);
            SK_LAUNCH_CHECK("oz residues");
        }
        if (!serial) {
            SK_CUDA(cudaEventRecord(sp.res_done[buf], sp.side));
            SK_CUDA(cudaStreamWaitEvent(sp.hi, sp.res_done[buf], 0));
        }
        if (prof) SK_CUDA(cudaEventRecord(pe[npe++], st));
        CUtensorMap tx, ty;
        int rc = make_tmap_3d(&tx, CU_TENSOR_MAP_DATA_TYPE_UINT8, res_x, (uint64_t)n, (uint64_t)rows, oz::NMOD,
                              (uint64_t)p.ldr, (uint64_t)plane, 128, oz::BK, CU_TENSOR_MAP_SWIZZLE_128B);
        if (rc) return rc;
        rc = make_tmap_3d(&ty, CU_TENSOR_MAP_DATA_TYPE_UINT8, res_y, (uint64_t)n, (uint64_t)rows, oz::NMOD,
                          (uint64_t)p.ldr, (uint64_t)plane, 128, oz::BK, CU_TENSOR_MAP_SWIZZLE_128B);
        if (rc) return rc;
        oz::GemmParams gp;
        gp.ntn = p.ntn;
        gp.ntiles = p.ntiles;
        gp.splits = (int)((rows + p.kchunk - 1) / p.kchunk);
        gp.units = p.nm * gp.splits * p.ntiles;
        gp.syrk = syrk;
        gp.rows = rows;
        gp.kchunk = p.kchunk;
        gp.acc = acc;
        gp.n = (int)n;
        oz::gemm_kernel<false><<<std::min(gp.units, sms), oz::THREADS, oz::SMEM, gs>>>(tx, ty, gp);
        SK_LAUNCH_CHECK("oz gemm");
        if (!serial) SK_CUDA(cudaEventRecord(sp.gemm_done[buf], gs));
    }
    const int64_t nn = n * n;
    if (prof) SK_CUDA(cudaEventRecord(pe[npe++], st));
    oz::crt_kernel<<<(unsigned)((nn + 255) / 256), 256, 0, gs>>>(acc, (int)n, syrk, expo, expo + n, p.t, g, ldg,
                                                                 p.nm, accumulate);
    SK_LAUNCH_CHECK("oz crt");
    if (!serial) {   // the caller's stream resumes after the reconstruction
        SK_CUDA(cudaEventRecord(sp.end, sp.hi));
        SK_CUDA(cudaStreamWaitEvent(st, sp.end, 0));
    }
    if (prof) {
        SK_CUDA(cudaEventRecord(pe[npe++], st));
        SK_CUDA(cudaEventSynchronize(pe[npe - 1]));
        float tot = 0, res_ms = 0, gemm_ms = 0, pre_ms = 0, t;
        cudaEventElapsedTime(&pre_ms, pe[0], pe[1]);
        for (int i = 1; i + 2 < npe; i += 2) {
            cudaEventElapsedTime(&t, pe[i], pe[i + 1]);
            res_ms += t;
            cudaEventElapsedTime(&t, pe[i + 1], pe[i + 2]);
            gemm_ms += t;
        }
        cudaEventElapsedTime(&tot, pe[0], pe[npe - 1]);
        fprintf(stderr, "ozaki %s m=%lld: total %.2f ms, colmax+scales %.2f, residues %.2f, gemm %.2f, other %.2f\n",
                syrk ? "syrk" : "gemm", (long long)m, tot, pre_ms, res_ms, gemm_ms, tot - pre_ms - res_ms - gemm_ms);
        for (int i = 0; i < npe; ++i) cudaEventDestroy(pe[i]);
    }
    if (defer)   // spiky or non-finite columns: the FP64 DMMA Gram, gated on the device flag
        return gram::gram_f64_gated(x, ldx, y, ldy, m, n, g, ldg, 0, ws, ws_bytes, stream, flag);
    return SK_OK;
}

}  // extern "C"
