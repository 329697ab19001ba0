// binary16 SRTT sketch on the 5th-generation tensor cores (tcgen05 + TMEM + TMA).
//
//   A_s(partial) = F_sampled * (D A16)      M = d sampled rows, N = n, K = m rows
//
// Reference semantics (src/sketch.py:138-169 at binary16, src/solvers.py:191-195):
// A is demoted to binary16, signs flipped (exact), the orthonormal DCT-II / WHT is
// taken along the rows (pocketfft in binary32 for the DCT, per-op binary16 for
// the WHT), the d sampled rows are kept, rounded to binary16 and scaled.  Here
// the d sampled rows of the transform are a tensor-core GEMM:
//
//   prep kernel   : A16[j][c] = sign_j * fp16(A[j][c])     (one streaming HBM pass in A's
//                   own row order, overflow of the demotion -> flag); the tensor cores
//                   read it as an MN-major B operand
//   main kernel   : persistent, warp-specialised, 1 CTA / SM; CTA b keeps sampled-row
//                   tile b % ntm and walks (column tile, K split) groups with the other
//                   ntm - 1 CTAs of its slot, so B chunks are shared through L2
//       warp 0      TMA producer: B tile A16[k-block 64][n-tile 256] as four 64 x 64
//                   SWIZZLE_128B boxes
//       warp 1      MMA issuer:   tcgen05.mma.cta_group::1.kind::f16, M128 N256 K16,
//                                 fp32 accumulator in TMEM (256 columns)
//       warp 2      TMEM allocator
//       warps 4-11  operator generator: F'[r_i][j] = cos(pi r_i (2j+1) / 2M) (DCT; 1/sqrt2
//                   for r = 0) or (-1)^popc(r_i & j) (WHT), exact integer phase
//                   reduction once per 32 columns + fp32 rotation recurrence, rounded
//                   to fp16 straight into the 128B-swizzled K-major A tile; then the
//                   epilogue: tcgen05.ld -> scale sqrt(2/M) (DCT) or 1/sqrt(M) (WHT)
//                   -> fp32 split-K partials
//   reduce kernel : fixed-order sum of the split-K partials -> f64 (column-major d x n)
// sk_sketch_finalize then applies the binary16 rounding and scale of the reference.
#include "tc.cuh"

namespace sk {

int make_tmap_2d(CUtensorMap *map, CUtensorMapDataType dtype, const void *base, uint64_t inner, uint64_t outer,
                 uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer, CUtensorMapSwizzle swz) {
    using EncodeFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static EncodeFn fn = nullptr;
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !p) {
            set_error("cuTensorMapEncodeTiled unavailable");
            return SK_ERR_CUDA;
        }
        fn = reinterpret_cast<EncodeFn>(p);
    }
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {row_stride_bytes};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(map, dtype, 2, const_cast<void *>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled failed (%d)", (int)r);
        return SK_ERR_CUDA;
    }
    return SK_OK;
}

int make_tmap_3d(CUtensorMap *map, CUtensorMapDataType dtype, const void *base, uint64_t d0, uint64_t d1,
                 uint64_t d2, uint64_t stride1_bytes, uint64_t stride2_bytes, uint32_t box0, uint32_t box1,
                 CUtensorMapSwizzle swz, CUtensorMapL2promotion promo) {
    using EncodeFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static EncodeFn fn = nullptr;
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !p) {
            set_error("cuTensorMapEncodeTiled unavailable");
            return SK_ERR_CUDA;
        }
        fn = reinterpret_cast<EncodeFn>(p);
    }
    cuuint64_t dims[3] = {d0, d1, d2};
    cuuint64_t strides[2] = {stride1_bytes, stride2_bytes};
    cuuint32_t box[3] = {box0, box1, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = fn(map, dtype, 3, const_cast<void *>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    swz, promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled (3d) failed (%d)", (int)r);
        return SK_ERR_CUDA;
    }
    return SK_OK;
}

namespace sktc {

// A CTA owns 256 sampled rows (two M=128 UMMA accumulators, 2 x 256 TMEM columns)
// against one 256-column B tile, so every B byte staged from L2 feeds 256 rows.
constexpr int BM = 256, UMMA_M = 128, BN = 256, BK = 64, STAGES = 3;
constexpr int THREADS = 640, GEN_WARP0 = 4, NGEN_WARPS = 16;
constexpr uint32_t A_BYTES = BM * BK * 2;   // 32 KB (two 16 KB UMMA operands)
constexpr uint32_t B_BYTES = BN * BK * 2;   // 32 KB
constexpr size_t SMEM = 1024 + STAGES * (A_BYTES + B_BYTES) + 256;
constexpr int TMEM_COLS = 512;

// ------------------------------------------------------------ prep kernel ---
// A16[j][c] = sign_j * fp16(A[j][c]) in A's own row-major order (ld = n rounded up to 8):
// a pure streaming cast, 16-byte loads and stores.  The tensor cores read it MN-major.
constexpr int PV = 8;   // columns per thread item
__global__ void __launch_bounds__(256)
prep_f16r(const double *__restrict__ a, int64_t lda, int64_t m_local, int n, const double *__restrict__ signs,
          int64_t row_offset, __half *__restrict__ out, int64_t ldn, int vec, int *overflow_flag) {
    const int cpr = (n + PV - 1) / PV;
    const int rpi = cpr >= 256 ? 1 : 256 / cpr;       // rows per block iteration
    const int sub = cpr >= 256 ? 0 : threadIdx.x / cpr;
    const int cfirst = cpr >= 256 ? threadIdx.x : threadIdx.x % cpr;
    const int cstep = cpr >= 256 ? 256 : cpr;
    int over = 0;
    for (int64_t j0 = (int64_t)blockIdx.x * rpi; j0 < m_local; j0 += (int64_t)gridDim.x * rpi) {
        const int64_t j = j0 + sub;
        if (sub >= rpi || j >= m_local) continue;
        const bool neg = signs[row_offset + j] < 0;
        const double *src = a + j * lda;
        __half *dst = out + j * ldn;
        for (int ch = cfirst; ch < cpr; ch += cstep) {
            const int c0 = ch * PV;
            double v[PV];
            if (vec && c0 + PV <= n) {
#pragma unroll
                for (int q = 0; q < PV / 2; ++q) {
                    const double2 t = __ldcs(reinterpret_cast<const double2 *>(src + c0) + q);
                    v[2 * q] = t.x;
                    v[2 * q + 1] = t.y;
                }
            } else {
#pragma unroll
                for (int q = 0; q < PV; ++q) v[q] = c0 + q < n ? src[c0 + q] : 0.0;
            }
            uint32_t pk[PV / 2];
#pragma unroll
            for (int e = 0; e < PV / 2; ++e) {
                __half h0 = __double2half(v[2 * e]), h1 = __double2half(v[2 * e + 1]);
                over |= (isinf(__half2float(h0)) && isfinite(v[2 * e])) |
                        (isinf(__half2float(h1)) && isfinite(v[2 * e + 1]));
                if (neg) {
                    h0 = __hneg(h0);
                    h1 = __hneg(h1);
                }
                __half2 h = __halves2half2(h0, h1);
                pk[e] = *reinterpret_cast<uint32_t *>(&h);
            }
            *reinterpret_cast<uint4 *>(dst + c0) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        }
    }
    if (__any_sync(0xffffffffu, over) && (threadIdx.x & 31) == 0) atomicOr(overflow_flag, 1);
}

struct Params {
    const int64_t *rows;
    int64_t mpad, row_offset, m_local, kchunk;
    int n, d, ntm, ntn, ntiles, groups, nslots;
    int wht;
    float epi_scale;
    float *part;
};

// CTA b owns sampled-row tile tm = b % ntm for the whole launch and walks the groups
// (tn, split) g = slot, slot + nslots, ...: the ntm CTAs of one slot stream the same
// B chunk at the same time, so each B byte comes from HBM once and from L2 ntm - 1 times.
__device__ __forceinline__ void group_coords(const Params &p, int g, int &tn, int &split, int64_t &k0, int &nkb) {
    tn = g % p.ntn;
    split = g / p.ntn;
    k0 = (int64_t)split * p.kchunk;
    const int64_t k1 = min(p.m_local, k0 + p.kchunk);
    nkb = (int)((k1 - k0 + BK - 1) / BK);
}

template <bool WHT>
__global__ void __launch_bounds__(THREADS, 1)
sketch_tc_kernel(const __grid_constant__ CUtensorMap tmap_b, const Params p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *sa = smem;
    uint8_t *sb = smem + STAGES * A_BYTES;
    uint64_t *full = reinterpret_cast<uint64_t *>(sb + STAGES * B_BYTES);
    uint64_t *empty = full + STAGES;
    uint64_t *tfull = empty + STAGES;
    uint64_t *tempty = tfull + 1;
    uint32_t *tslot = reinterpret_cast<uint32_t *>(tempty + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tm = blockIdx.x % p.ntm, slot = blockIdx.x / p.ntm;
    if (warp == 0 && lane == 0) {
        for (int s = 0; s < STAGES; ++s) {
            tc::mbar_init(&full[s], 1 + NGEN_WARPS);
            tc::mbar_init(&empty[s], 1);
        }
        tc::mbar_init(tfull, 1);
        tc::mbar_init(tempty, NGEN_WARPS);
        tc::mbar_fence_init();
        tc::tma_prefetch_desc(&tmap_b);
    }
    if (warp == 2) tc::tmem_alloc<TMEM_COLS>(tslot);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = *tslot;

    if (warp == 0) {
        if (lane == 0) {   // ---------------- TMA producer
            int stage = 0;
            unsigned phase = 0;
            for (int g = slot; g < p.groups; g += p.nslots) {
                int tn, split, nkb;
                int64_t k0;
                group_coords(p, g, tn, split, k0, nkb);
                for (int kb = 0; kb < nkb; ++kb) {
                    tc::mbar_wait(&empty[stage], phase ^ 1);
                    tc::mbar_arrive_expect_tx(&full[stage], B_BYTES);
                    const int krow = (int)(k0 + (int64_t)kb * BK);
#pragma unroll
                    for (int q = 0; q < BN / 64; ++q)   // four 64-column x 64-row SW128 boxes
                        tc::tma_load_2d(sb + stage * B_BYTES + q * (B_BYTES / (BN / 64)), &tmap_b, &full[stage],
                                        tn * BN + q * 64, krow);
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {   // ---------------- MMA issuer
            constexpr uint32_t idesc = tc::idesc_f32acc(UMMA_M, BN, 0, 0, 0, 1);   // B MN-major
            int stage = 0;
            unsigned phase = 0, tphase = 0;
            for (int g = slot; g < p.groups; g += p.nslots) {
                int tn, split, nkb;
                int64_t k0;
                group_coords(p, g, tn, split, k0, nkb);
                tc::mbar_wait(tempty, tphase ^ 1);
                tc::tc_fence_after();
                for (int kb = 0; kb < nkb; ++kb) {
                    tc::mbar_wait(&full[stage], phase);
                    tc::tc_fence_after();
                    const uint64_t ad0 = tc::desc_kmajor_sw128(smem_u32(sa + stage * A_BYTES));
                    const uint64_t ad1 = tc::desc_kmajor_sw128(smem_u32(sa + stage * A_BYTES + A_BYTES / 2));
                    // B: 64-column blocks 8 KB apart (LBO), 8-row K groups 1 KB apart (SBO)
                    const uint64_t bd = tc::desc_mnmajor_sw128(smem_u32(sb + stage * B_BYTES), B_BYTES / (BN / 64), 1024);
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k) {   // A: +32 bytes along K; B: +16 rows = 2 KB
                        tc::mma_f16_ss(tmem, ad0 + 2 * k, bd + 128 * k, idesc, (kb | k) ? 1u : 0u);
                        tc::mma_f16_ss(tmem + BN, ad1 + 2 * k, bd + 128 * k, idesc, (kb | k) ? 1u : 0u);
                    }
                    tc::mma_commit(&empty[stage]);
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
                tc::mma_commit(tfull);
                tphase ^= 1;
            }
        }
    } else if (warp >= GEN_WARP0) {
        // ---------------- operator generator + epilogue
        const int gt = threadIdx.x - GEN_WARP0 * 32;   // 0..255
        const int row = gt >> 1, half = gt & 1;
        const uint64_t M = (uint64_t)p.mpad, fourM = 4 * M;
        const float inv2M = 1.0f / (2.0f * (float)p.mpad);
        int stage = 0;
        unsigned phase = 0, tphase = 0;
        const int i = tm * BM + row;
        const bool valid = i < p.d;
        const uint64_t r = valid ? (uint64_t)p.rows[i] : 0;
        const uint64_t f1 = r % fourM;
        // per-row offset table e^{i pi r (2t) / 2M}, t = 0..31 (exact integer phases)
        // 16-entry table (registers): columns 16..31 use the base rotated by e^{i 16 delta}
        float wc[16], ws[16], wc16 = 1.f, ws16 = 0.f;
        // DCT rows with r = 0 (all entries 1/sqrt2) or past d (zeros) use the same
        // branch-free formula with a constant table: z = 1, wc = that constant, ws = 0
        const bool flat = !WHT && (r == 0 || !valid);
        if (!WHT) {
            if (flat) {
                const float cflat = valid ? 0.70710678118654752f : 0.f;
#pragma unroll
                for (int t = 0; t < 16; ++t) {
                    wc[t] = cflat;
                    ws[t] = 0.f;
                }
            } else {
#pragma unroll
                for (int t = 0; t < 16; ++t) {
                    const uint64_t q = (f1 * (uint64_t)(2 * t)) % fourM;
                    sincospif((float)q * inv2M, &ws[t], &wc[t]);
                }
                const uint64_t q16 = (f1 * (uint64_t)32) % fourM;
                sincospif((float)q16 * inv2M, &ws16, &wc16);
            }
        }
        for (int g = slot; g < p.groups; g += p.nslots) {
            int tn, split, nkb;
            int64_t k0;
            group_coords(p, g, tn, split, k0, nkb);
            // phase of this thread's first column, advanced exactly by r*2*BK per K-block
            uint64_t ph = (f1 * ((uint64_t)(2 * (p.row_offset + k0 + half * 32) + 1) % fourM)) % fourM;
            const uint64_t dph = (f1 * (uint64_t)(2 * BK)) % fourM;
            for (int kb = 0; kb < nkb; ++kb) {
                tc::mbar_wait(&empty[stage], phase ^ 1);
                const int64_t jg0 = p.row_offset + k0 + (int64_t)kb * BK + half * 32;
                uint8_t *tile = sa + stage * A_BYTES;
                // 32 operator values of this (row, half) -> four 16-byte swizzled chunks,
                // each stored as soon as its 8 values are rounded (few live registers)
                float zs = 0.f, zc = 1.f;
                if (!WHT && !flat) {
                    sincospif((float)ph * inv2M, &zs, &zc);
                    ph += dph;
                    if (ph >= fourM) ph -= fourM;
                }
                const float zc2 = zc * wc16 - zs * ws16, zs2 = zs * wc16 + zc * ws16;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    uint32_t pk[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int t = q * 8 + 2 * e;
                        float a0, a1;
                        if constexpr (WHT) {
                            const uint64_t j0 = (uint64_t)(jg0 + t), j1 = j0 + 1;
                            a0 = valid ? ((__popcll(r & j0) & 1) ? -1.f : 1.f) : 0.f;
                            a1 = valid ? ((__popcll(r & j1) & 1) ? -1.f : 1.f) : 0.f;
                        } else if (t < 16) {
                            a0 = zc * wc[t] - zs * ws[t];
                            a1 = zc * wc[t + 1] - zs * ws[t + 1];
                        } else {
                            a0 = zc2 * wc[t - 16] - zs2 * ws[t - 16];
                            a1 = zc2 * wc[t - 15] - zs2 * ws[t - 15];
                        }
                        __half2 h = __floats2half2_rn(a0, a1);
                        pk[e] = *reinterpret_cast<uint32_t *>(&h);
                    }
                    *reinterpret_cast<uint4 *>(tile + tc::sw128_offset(row, half * 4 + q)) =
                        make_uint4(pk[0], pk[1], pk[2], pk[3]);
                }
                tc::fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&full[stage]);
                if (++stage == STAGES) { stage = 0; phase ^= 1; }
            }
            // ---- epilogue: TMEM -> registers -> fp32 partial (column-major within the tile)
            tc::mbar_wait(tfull, tphase);
            tc::tc_fence_after();
            tphase ^= 1;
            // warp w reads TMEM lanes 32*(w%4)..; the 16 warps split 2 accumulators x 2 column halves
            const int lg = warp & 3, quarter = (warp - GEN_WARP0) >> 2;
            const int acc = quarter >> 1, colhalf = quarter & 1;
            const int tile = tm * p.ntn + tn;
            float *out = p.part + ((size_t)split * p.ntiles + tile) * (size_t)(BM * BN);
            const int orow = acc * UMMA_M + lg * 32 + lane;
#pragma unroll 1
            for (int cb = 0; cb < 4; ++cb) {
                const int col = colhalf * 128 + cb * 32;
                uint32_t v[32];
                tc::tmem_ld_32x32b_x32(tmem + ((uint32_t)(lg * 32) << 16) + (uint32_t)(acc * BN + col), v);
                tc::tmem_ld_wait();
#pragma unroll
                for (int q = 0; q < 32; ++q) out[(size_t)(col + q) * BM + orow] = __uint_as_float(v[q]) * p.epi_scale;
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
        tc::tmem_dealloc<TMEM_COLS>(tmem);
    }
}

__global__ void reduce_part(const float *__restrict__ part, int splits, int ntiles, int ntn, int d, int n,
                            double *__restrict__ out, int64_t ldo, int accumulate) {
    const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= (int64_t)d * n) return;
    const int c = (int)(idx / d), i = (int)(idx % d);
    const int tile = (i / BM) * ntn + c / BN;
    const float *pp = part + (size_t)tile * (BM * BN) + (size_t)(c % BN) * BM + (i % BM);
    double s = 0.0;
    for (int k = 0; k < splits; ++k) s += (double)pp[(size_t)k * ntiles * (BM * BN)];
    double *o = out + (int64_t)c * ldo + i;
    *o = accumulate ? *o + s : s;
}

struct Plan {
    int ntm, ntn, ntiles, splits, groups, nslots, grid;
    int64_t kchunk, ldn;
    size_t at_bytes, part_bytes;
};

Plan make_plan(int64_t m_local, int64_t n, int64_t d) {
    Plan p;
    p.ntm = (int)((d + BM - 1) / BM);
    p.ntn = (int)((n + BN - 1) / BN);
    p.ntiles = p.ntm * p.ntn;
    const int sms = sm_count();
    p.nslots = sms >= p.ntm ? sms / p.ntm : 1;
    p.grid = p.ntm * p.nslots;
    const int64_t nkb_total = (m_local + BK - 1) / BK;
    // ~32 groups per slot; the split count is nudged so that every slot gets the same
    // number of groups (ntn * splits divisible by nslots)
    int64_t target = (int64_t)32 * p.nslots / p.ntn;
    if (target < 1) target = 1;
    const int64_t smax = std::max<int64_t>(1, (nkb_total + 15) / 16);   // >= 16 K-blocks per group
    if (target > smax) target = smax;
    int64_t best = target;
    for (int64_t s = target; s < target + p.nslots && s <= smax; ++s)
        if (((int64_t)p.ntn * s) % p.nslots == 0) { best = s; break; }
    const int64_t kb_per = (nkb_total + best - 1) / best;
    p.kchunk = kb_per * BK;
    p.splits = (int)((m_local + p.kchunk - 1) / p.kchunk);
    if (p.splits < 1) p.splits = 1;
    p.groups = p.ntn * p.splits;
    p.ldn = (n + 7) / 8 * 8;
    p.at_bytes = align_up((size_t)m_local * p.ldn * sizeof(__half), 1024);
    p.part_bytes = (size_t)p.splits * p.ntiles * BM * BN * sizeof(float);
    return p;
}

}  // namespace sktc

size_t sketch_tc_workspace(int64_t m_local, int64_t n, int64_t d) {
    sktc::Plan p = sktc::make_plan(m_local, n, d);
    return p.at_bytes + p.part_bytes + 1024;
}

int sketch_tc_run(int transform, const double *a, int64_t lda, int64_t m_local, int64_t row_offset, int64_t m_pad,
                  int64_t n, const double *signs, const int64_t *rows, int64_t d, double *out, int64_t ldo,
                  int accumulate, int *overflow_flag_dev, void *ws, size_t ws_bytes, cudaStream_t st) {
    using namespace sktc;
    Plan p = make_plan(m_local, n, d);
    if (ws_bytes < p.at_bytes + p.part_bytes) {
        set_error("sketch_tc: workspace %zu < %zu", ws_bytes, p.at_bytes + p.part_bytes);
        return SK_ERR_ARG;
    }
    __half *at = static_cast<__half *>(ws);
    float *part = reinterpret_cast<float *>(static_cast<uint8_t *>(ws) + p.at_bytes);
    if (m_local == 0) {
        if (!accumulate) {
            for (int64_t c = 0; c < n; ++c) SK_CUDA(cudaMemsetAsync(out + c * ldo, 0, (size_t)d * sizeof(double), st));
        }
        return SK_OK;
    }
    const int vec = ((reinterpret_cast<uintptr_t>(a) & 15) == 0) && (lda % 2 == 0);
    prep_f16r<<<sm_count() * 8, 256, 0, st>>>(a, lda, m_local, (int)n, signs, row_offset, at, p.ldn, vec,
                                              overflow_flag_dev);
    SK_LAUNCH_CHECK("prep_f16r");
    CUtensorMap tmap;
    int rc = make_tmap_2d(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, at, (uint64_t)n, (uint64_t)m_local,
                          (uint64_t)p.ldn * sizeof(__half), 64, BK, CU_TENSOR_MAP_SWIZZLE_128B);
    if (rc) return rc;
    Params prm;
    prm.rows = rows;
    prm.mpad = m_pad;
    prm.row_offset = row_offset;
    prm.m_local = m_local;
    prm.kchunk = p.kchunk;
    prm.n = (int)n;
    prm.d = (int)d;
    prm.ntm = p.ntm;
    prm.ntn = p.ntn;
    prm.ntiles = p.ntiles;
    prm.groups = p.groups;
    prm.nslots = p.nslots;
    prm.wht = transform == SK_WHT;
    prm.epi_scale = transform == SK_WHT ? (float)(1.0 / sqrt((double)m_pad)) : (float)sqrt(2.0 / (double)m_pad);
    prm.part = part;
    auto kfn = prm.wht ? sketch_tc_kernel<true> : sketch_tc_kernel<false>;
    SK_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM));
    kfn<<<p.grid, THREADS, SMEM, st>>>(tmap, prm);
    SK_LAUNCH_CHECK("sketch_tc_kernel");
    const int64_t total = d * n;
    reduce_part<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(part, p.splits, p.ntiles, p.ntn, (int)d, (int)n, out,
                                                                 ldo, accumulate);
    SK_LAUNCH_CHECK("reduce_part");
    return SK_OK;
}

}  // namespace sk
