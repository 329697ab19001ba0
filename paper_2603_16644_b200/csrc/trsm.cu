// A_p = A R^{-1}: right-side, upper-triangular FP64 solve on the DMMA pipe.
//
// Reference: precondition_matrix src/solvers.py:205-215, which calls
// triangular_solve(r_s, a.T, transposed=True) src/dense.py:204-242 — forward
// substitution over the columns of A_p, x_i = (a_i - sum_{l<i} r_li x_l) / r_ii,
// independently for every row of A.
//
// B200 design: row panels are independent, so each CTA owns BMR rows and walks
// the NB-wide column blocks left to right ("left-looking"):
//   T            = A[rows, J] - A_p[rows, <J] . R[<J, J]   (DMMA GEMM, cp.async ring)
//   A_p[rows, J] = substitution of T against R[J, J]      (two threads per row, the
//                                                          row's columns split even/odd
//                                                          in registers, R_JJ in smem)
// The diagonal block is solved by substitution (dot-then-divide, like the
// reference), never through an explicit inverse, so the solve stays backward
// stable for kappa(R) up to 1e14.  The panel's earlier A_p columns are re-read
// from L2/HBM (compute-bound: ~BMR/4 flop per byte); R stays L2-resident.
// The T tile and R_JJ are staged with cp.async ahead of the GEMM so their latency
// hides behind it.  A_p may alias A (in place).
#include "common.cuh"

namespace sk {
namespace trsm {

#ifndef SK_TRSM_BK
#define SK_TRSM_BK 16
#define SK_TRSM_STAGES 3
#endif
#ifndef SK_TRSM_BMR
#define SK_TRSM_BMR 128   // rows per CTA; 2 threads per row in the substitution
#endif
constexpr int BMR = SK_TRSM_BMR, NB = 64, BK = SK_TRSM_BK, STAGES = SK_TRSM_STAGES, THREADS = 2 * BMR;
constexpr int MINB = BMR >= 128 ? 2 : 3;   // CTAs per SM (shared memory: 102 KB at 128 rows, 69 KB at 64)
constexpr int WM = 32, WN = 32;             // 4 x 2 warps
constexpr int APITCH = BK + 4;              // 20 = 4 (mod 16): conflict-free A fragments
constexpr int BPITCH = NB + 4;              // 68 = 4 (mod 16): conflict-free B fragments
#ifndef SK_TRSM_TPAD
#define SK_TRSM_TPAD 2
#endif
// T tile rows, 16-byte aligned: 66 doubles (528 B) puts the 16 rows a warp's
// substitution threads walk on distinct bank pairs (68 made them 4-way)
constexpr int TPITCH = NB + SK_TRSM_TPAD;
// R_JJ rows 68 doubles apart, odd columns 34 after the even ones: the DMMA B-fragment
// loads of the sub-block update (k = lane % 4 rows, n = lane / 4 columns) then touch each
// bank pair at most twice (2 wavefronts, the minimum for 256 B); with 64 / 32 they were
// 8-way conflicted (ncu: 15 excess wavefronts per load).
constexpr int RPITCH = NB + 4;
constexpr int RHALF = NB / 2 + 2;
// The T tile and R_JJ alias the GEMM staging ring (they are loaded after the GEMM),
// which keeps a CTA at ~102 KB so two CTAs share an SM: one CTA's substitution and
// staging latency hides behind the other's DMMA work.
constexpr size_t RING = sizeof(double) * (size_t(STAGES) * BMR * APITCH + size_t(STAGES) * BK * BPITCH);
constexpr size_t TILE = sizeof(double) * (size_t(BMR) * TPITCH + size_t(NB) * RPITCH);
constexpr size_t SMEM = RING > TILE ? RING : TILE;

// R_JJ in shared memory with each row split by column parity: element (i, j) at
// i*RPITCH + (j&1)*RHALF + j/2, so a substitution thread's half-row is contiguous.
__device__ __forceinline__ int ridx(int i, int j) { return i * RPITCH + (j & 1) * RHALF + (j >> 1); }

__device__ __forceinline__ void load_stage(double *as, double *bs, const double *ap, int64_t ldap,
                                           const double *__restrict__ r, int64_t ldr, int64_t row0, int64_t m, int k0,
                                           int kend, int j0, int n, bool vec) {
    const int tid = threadIdx.x;
    if (vec && row0 + BMR <= m && k0 + BK <= kend && j0 + NB <= n) {
        // interior tile: no bounds arithmetic (the common case)
#pragma unroll
        for (int i = 0; i < (BMR * (BK / 2)) / THREADS; ++i) {
            const int c = tid + i * THREADS;
            const int rr = c / (BK / 2), kc = (c % (BK / 2)) * 2;
            cp_async16(as + rr * APITCH + kc, ap + (row0 + rr) * ldap + k0 + kc, 16);
        }
#pragma unroll
        for (int i = 0; i < (BK * (NB / 2)) / THREADS; ++i) {
            const int c = tid + i * THREADS;
            const int kr = c / (NB / 2), jc = (c % (NB / 2)) * 2;
            cp_async16(bs + kr * BPITCH + jc, r + (int64_t)(k0 + kr) * ldr + j0 + jc, 16);
        }
        return;
    }
    if (vec) {
        for (int c = tid; c < BMR * (BK / 2); c += THREADS) {
            const int rr = c / (BK / 2), kc = (c % (BK / 2)) * 2;
            const int64_t row = row0 + rr;
            const int k = k0 + kc;
            int bytes = (row < m) ? (kend - k) * 8 : 0;
            bytes = bytes < 0 ? 0 : (bytes > 16 ? 16 : bytes);
            cp_async16(as + rr * APITCH + kc, bytes ? ap + row * ldap + k : ap, bytes);
        }
        for (int c = tid; c < BK * (NB / 2); c += THREADS) {
            const int kr = c / (NB / 2), jc = (c % (NB / 2)) * 2;
            const int k = k0 + kr, j = j0 + jc;
            int bytes = (k < kend) ? (n - j) * 8 : 0;
            bytes = bytes < 0 ? 0 : (bytes > 16 ? 16 : bytes);
            cp_async16(bs + kr * BPITCH + jc, bytes ? r + (int64_t)k * ldr + j : r, bytes);
        }
    } else {
        for (int c = tid; c < BMR * BK; c += THREADS) {
            const int rr = c / BK, kc = c % BK;
            const int64_t row = row0 + rr;
            const int k = k0 + kc;
            const int bytes = (row < m && k < kend) ? 8 : 0;
            cp_async8(as + rr * APITCH + kc, bytes ? ap + row * ldap + k : ap, bytes);
        }
        for (int c = tid; c < BK * NB; c += THREADS) {
            const int kr = c / NB, jc = c % NB;
            const int k = k0 + kr, j = j0 + jc;
            const int bytes = (k < kend && j < n) ? 8 : 0;
            cp_async8(bs + kr * BPITCH + jc, bytes ? r + (int64_t)k * ldr + j : r, bytes);
        }
    }
}

// T tile A[rows, j0:j0+jw] and R[j0:j0+jw, j0:j0+jw] (zero-filled outside)
__device__ __forceinline__ void load_block(double *ts, double *rs, const double *a, int64_t lda,
                                           const double *__restrict__ r, int64_t ldr, int64_t row0, int64_t m, int j0,
                                           int jw, bool vec) {
    const int tid = threadIdx.x;
    if (vec) {
        for (int c = tid; c < BMR * (NB / 2); c += THREADS) {
            const int rr = c / (NB / 2), jc = (c % (NB / 2)) * 2;
            const int64_t row = row0 + rr;
            int bytes = (row < m) ? (jw - jc) * 8 : 0;
            bytes = bytes < 0 ? 0 : (bytes > 16 ? 16 : bytes);
            cp_async16(ts + rr * TPITCH + jc, bytes ? a + row * lda + j0 + jc : a, bytes);
        }
        for (int c = tid; c < NB * NB; c += THREADS) {
            const int i = c / NB, jc = c % NB;
            const int bytes = (i < jw && jc < jw) ? 8 : 0;
            cp_async8(rs + ridx(i, jc), bytes ? r + (int64_t)(j0 + i) * ldr + j0 + jc : r, bytes);
        }
    } else {
        for (int c = tid; c < BMR * NB; c += THREADS) {
            const int rr = c / NB, jc = c % NB;
            const int64_t row = row0 + rr;
            const int bytes = (row < m && jc < jw) ? 8 : 0;
            cp_async8(ts + rr * TPITCH + jc, bytes ? a + row * lda + j0 + jc : a, bytes);
        }
        for (int c = tid; c < NB * NB; c += THREADS) {
            const int i = c / NB, jc = c % NB;
            const int bytes = (i < jw && jc < jw) ? 8 : 0;
            cp_async8(rs + ridx(i, jc), bytes ? r + (int64_t)(j0 + i) * ldr + j0 + jc : r, bytes);
        }
    }
}

__global__ void __launch_bounds__(THREADS, MINB)
trsm_kernel(const double *a, int64_t lda, int64_t m, int n, const double *__restrict__ r, int64_t ldr, double *ap,
            int64_t ldap, bool vec, const int *gate) {
    if (gate && *gate == 0) return;   // gated fallback (deferred verdicts): run only when flagged
    extern __shared__ __align__(16) double smem[];
    double *as_base = smem;
    double *bs_base = as_base + STAGES * BMR * APITCH;
    double *ts = smem;                   // aliases the ring (used after the GEMM)
    double *rs = ts + BMR * TPITCH;

    const int64_t row0 = (int64_t)blockIdx.x * BMR;
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
    const int wm = warp % (BMR / WM), wn = warp / (BMR / WM);
    const int nblocks = (n + NB - 1) / NB;
    // substitution role: two threads per row, columns split by parity
    const int srow = tid >> 1, hf = tid & 1;

    for (int J = 0; J < nblocks; ++J) {
        const int j0 = J * NB;
        const int jw = min(NB, n - j0);

        double acc[WM / 8][WN / 8][2];
#pragma unroll
        for (int x = 0; x < WM / 8; ++x)
#pragma unroll
            for (int y = 0; y < WN / 8; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
        const int nk = (j0 + BK - 1) / BK;
        // Each CTA starts its K sweep at a different block (rotation by blockIdx): the
        // concurrently resident panels are 2 MB apart, so walking the same columns in
        // lockstep would hammer the same L2/HBM channels.
        int kload = nk ? (int)(blockIdx.x % (unsigned)nk) : 0;   // next K block to stage (rotated)
#pragma unroll
        for (int s = 0; s < STAGES - 1; ++s) {
            if (s < nk) {
                load_stage(as_base + s * BMR * APITCH, bs_base + s * BK * BPITCH, ap, ldap, r, ldr, row0, m,
                           kload * BK, j0, j0, n, vec);
                if (++kload == nk) kload = 0;
            }
            cp_async_commit();
        }
        for (int kt = 0; kt < nk; ++kt) {
            cp_async_wait<STAGES - 2>();
            __syncthreads();
            const int nxt = kt + STAGES - 1;
            if (nxt < nk) {
                const int s = nxt % STAGES;
                load_stage(as_base + s * BMR * APITCH, bs_base + s * BK * BPITCH, ap, ldap, r, ldr, row0, m,
                           kload * BK, j0, j0, n, vec);
                if (++kload == nk) kload = 0;
            }
            cp_async_commit();
            const double *as = as_base + (kt % STAGES) * BMR * APITCH;
            const double *bs = bs_base + (kt % STAGES) * BK * BPITCH;
#pragma unroll
            for (int kk = 0; kk < BK; kk += 4) {
                double af[WM / 8], bf[WN / 8];
#pragma unroll
                for (int x = 0; x < WM / 8; ++x) af[x] = as[(wm * WM + x * 8 + g) * APITCH + kk + t];
#pragma unroll
                for (int y = 0; y < WN / 8; ++y) bf[y] = bs[(kk + t) * BPITCH + wn * WN + y * 8 + g];
#pragma unroll
                for (int x = 0; x < WM / 8; ++x)
#pragma unroll
                    for (int y = 0; y < WN / 8; ++y) dmma884(acc[x][y][0], acc[x][y][1], af[x], bf[y]);
            }
        }
        cp_async_wait<0>();
        __syncthreads();                 // ring free: stage T and R_JJ into it
        load_block(ts, rs, a, lda, r, ldr, row0, m, j0, jw, vec);
        cp_async_commit();
        cp_async_wait<0>();
        __syncthreads();
        // -- T -= acc  (padded diagonal entries of R_JJ become 1)
        if (nk > 0) {
#pragma unroll
            for (int x = 0; x < WM / 8; ++x)
#pragma unroll
                for (int y = 0; y < WN / 8; ++y) {
                    const int rr = wm * WM + x * 8 + g, cc = wn * WN + y * 8 + 2 * t;
                    ts[rr * TPITCH + cc] -= acc[x][y][0];
                    ts[rr * TPITCH + cc + 1] -= acc[x][y][1];
                }
        }
        // reciprocals of the diagonal (padded entries -> 1): the substitution's dependency
        // chain is then DMUL -> SHFL -> DFMA per column instead of a full division (the
        // optimised BLAS dtrsm kernels the reference reaches also scale by 1/r_jj)
        __shared__ double rinv[NB];
        if (tid < NB) rinv[tid] = tid >= jw ? 1.0 : 1.0 / rs[ridx(tid, tid)];
        __syncthreads();
        // -- the diagonal block in SB-wide sub-blocks: substitution on the sub-block's
        //    triangle (two threads per row, columns split by parity), then the rest of
        //    T loses X_s R[s, >s] on the DMMA pipe.  A quarter of the SIMT FP64 work of a
        //    full 64-wide substitution; the order of the dot products per entry changes
        //    (blocked instead of column by column), not the algorithm.
#ifndef SK_TRSM_NOSUB   // (timing experiments only: -DSK_TRSM_NOSUB skips the solve)
#ifndef SK_TRSM_SB
#define SK_TRSM_SB 32   // measured at 4M x 2048: SB 8 592 ms, 16 584 ms, 32 580 ms, none (no solve) 533 ms
#endif
        constexpr int SB = SK_TRSM_SB;
#pragma unroll 1
        for (int s = 0; s < NB / SB; ++s) {
            const int cs = s * SB;
            {
                double v[SB / 2];
#pragma unroll
                for (int k = 0; k < SB / 2; ++k) v[k] = ts[srow * TPITCH + cs + 2 * k + hf];
                const int base = lane & ~1;
#pragma unroll
                for (int c = 0; c < SB; ++c) {
                    const int owner = c & 1, kc = c >> 1;
                    double x = 0.0;
                    if (hf == owner) {
                        v[kc] = v[kc] * rinv[cs + c];
                        x = v[kc];
                    }
                    x = __shfl_sync(0xffffffffu, x, base | owner);
                    // this thread's half of row cs+c of R_JJ, sub-block columns: contiguous
                    const double *rrow = rs + (cs + c) * RPITCH + hf * RHALF + cs / 2;
#pragma unroll
                    for (int kp = ((c + 1) >> 1) >> 1; kp < SB / 4; ++kp) {
                        const double2 rv = *reinterpret_cast<const double2 *>(rrow + 2 * kp);
                        if (4 * kp + hf > c) v[2 * kp] -= x * rv.x;
                        if (4 * kp + 2 + hf > c) v[2 * kp + 1] -= x * rv.y;
                    }
                }
#pragma unroll
                for (int k = 0; k < SB / 2; ++k) ts[srow * TPITCH + cs + 2 * k + hf] = v[k];
            }
            __syncthreads();
            const int rest = NB - cs - SB;                  // columns right of the sub-block
            if (rest > 0) {
                // warp w: rows 16w..16w+15 (two 8-row m-tiles) x all `rest` columns
                const int nt = rest / 8;
                double am[2][SB / 4];
#pragma unroll
                for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                    for (int kk = 0; kk < SB / 4; ++kk)
                        am[mt][kk] = -ts[(warp * 16 + mt * 8 + g) * TPITCH + cs + kk * 4 + t];
#pragma unroll 1
                for (int y = 0; y < nt; ++y) {
                    const int c0 = cs + SB + y * 8;
                    double bf[SB / 4];
#pragma unroll
                    for (int kk = 0; kk < SB / 4; ++kk) bf[kk] = rs[ridx(cs + kk * 4 + t, c0 + g)];
#pragma unroll
                    for (int mt = 0; mt < 2; ++mt) {
                        double *crow = ts + (warp * 16 + mt * 8 + g) * TPITCH + c0 + 2 * t;
                        double c0v = crow[0], c1v = crow[1];
#pragma unroll
                        for (int kk = 0; kk < SB / 4; ++kk) dmma884(c0v, c1v, am[mt][kk], bf[kk]);
                        crow[0] = c0v;
                        crow[1] = c1v;
                    }
                }
            }
            __syncthreads();
        }
#endif
        __syncthreads();
        // -- store A_p[rows, J]
        if (vec && jw == NB) {
            for (int c = tid; c < BMR * (NB / 2); c += THREADS) {
                const int rr = c / (NB / 2), jc = (c % (NB / 2)) * 2;
                const int64_t row = row0 + rr;
                if (row < m)
                    *reinterpret_cast<double2 *>(ap + row * ldap + j0 + jc) =
                        *reinterpret_cast<const double2 *>(ts + rr * TPITCH + jc);
            }
        } else {
            for (int c = tid; c < BMR * NB; c += THREADS) {
                const int rr = c / NB, jc = c % NB;
                const int64_t row = row0 + rr;
                if (row < m && jc < jw) ap[row * ldap + j0 + jc] = ts[rr * TPITCH + jc];
            }
        }
        __syncthreads();
    }
}

// one block: index of the first exactly-zero diagonal entry (INT32_MAX if none),
// written straight into mapped pinned host memory
__global__ void __launch_bounds__(1024) first_zero_diag(const double *__restrict__ r, int64_t ldr, int n, int *out) {
    __shared__ int wmin[32];
    int best = INT32_MAX;
    for (int i = threadIdx.x; i < n; i += blockDim.x)
        if (r[(int64_t)i * ldr + i] == 0.0) { best = i; break; }
    for (int o = 16; o > 0; o >>= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
    if ((threadIdx.x & 31) == 0) wmin[threadIdx.x >> 5] = best;
    __syncthreads();
    if (threadIdx.x < 32) {
        best = wmin[threadIdx.x];
        for (int o = 16; o > 0; o >>= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
        if (threadIdx.x == 0) *reinterpret_cast<volatile int *>(out) = best;
    }
}

// one mapped pinned int per host thread (calls on one thread are serialised by the
// synchronize that reads it)
int *zero_diag_slot() {
    thread_local int *slot = nullptr;
    if (!slot) {
        void *p = nullptr;
        if (cudaHostAlloc(&p, sizeof(int), cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess) return nullptr;
        slot = static_cast<int *>(p);
    }
    return slot;
}

// the kernel alone (no argument or diagonal checks); used by the blocked INT8 TRSM too
int launch(const double *a, int64_t lda, int64_t m, int n, const double *r, int64_t ldr, double *ap, int64_t ldap,
           cudaStream_t st, const int *gate) {
    if (m == 0) return SK_OK;
    const bool vec = ((reinterpret_cast<uintptr_t>(ap) | reinterpret_cast<uintptr_t>(r) |
                       reinterpret_cast<uintptr_t>(a)) % 16 == 0) &&
                     (ldap % 2 == 0) && (ldr % 2 == 0) && (lda % 2 == 0);
    SK_CUDA(cudaFuncSetAttribute(trsm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM));
    const unsigned grid = (unsigned)((m + BMR - 1) / BMR);
    trsm_kernel<<<grid, THREADS, SMEM, st>>>(a, lda, m, n, r, ldr, ap, ldap, vec, gate);
    SK_LAUNCH_CHECK("trsm_kernel");
    return SK_OK;
}

// first exactly-zero diagonal entry of R (INT32_MAX if none); synchronizes the stream
int first_zero_diagonal(const double *r, int64_t ldr, int n, cudaStream_t st, int *out) {
    int *first = zero_diag_slot();
    if (!first) {
        set_error("trsm: pinned status slot unavailable");
        return SK_ERR_CUDA;
    }
    first_zero_diag<<<1, 1024, 0, st>>>(r, ldr, n, first);
    SK_LAUNCH_CHECK("first_zero_diag");
    SK_CUDA(cudaStreamSynchronize(st));
    *out = *reinterpret_cast<volatile int *>(first);
    return SK_OK;
}

}  // namespace trsm
}  // namespace sk

using namespace sk;

extern "C" int sk_trsm_right_upper_f64(const double *a, int64_t lda, int64_t m, int64_t n, const double *r,
                                       int64_t ldr, double *ap, int64_t ldap, sk_status *status,
                                       sk_stream_t stream) {
    if (!a || !r || !ap || m < 0 || n <= 0 || lda < n || ldr < n || ldap < n || n > (1 << 20) ||
        (a == ap && lda != ldap)) {
        set_error("sk_trsm_right_upper_f64: bad arguments");
        return SK_ERR_ARG;
    }
    cudaStream_t st = (cudaStream_t)stream;
    // exactly-zero diagonal -> SingularTriangular (src/dense.py:231-233).  No stream-
    // ordered allocation here: a cudaMallocAsync / cudaFreeAsync pair per call made the
    // following synchronize wait on pool trimming (measured 0.2-900 ms per call).
    if (deferred_status()) {   // deferred verdicts: recorded on the device, no host read
        int rc = note_zero_diagonal(r, ldr, n, SK_SINGULAR_TRIANGULAR, st);
        if (rc) return rc;
        rc = trsm::launch(a, lda, m, (int)n, r, ldr, ap, ldap, st, nullptr);
        if (rc) return rc;
        return fill_status(status, SK_OK, -1, 0, 0);
    }
    int first_zero = 0;
    int rc = trsm::first_zero_diagonal(r, ldr, (int)n, st, &first_zero);
    if (rc) return rc;
    if (first_zero != INT32_MAX) {
        set_error("zero diagonal entry at index %d", first_zero);
        return fill_status(status, SK_SINGULAR_TRIANGULAR, first_zero, 0.0, 0.0);
    }
    rc = trsm::launch(a, lda, m, (int)n, r, ldr, ap, ldap, st, nullptr);
    if (rc) return rc;
    return fill_status(status, SK_OK, -1, 0, 0);
}
