// Level-precision Householder QR of the d x n sketch, R factor only.
//
// Reference: qr_in_precision src/precision.py:153-202 on top of householder_reduce
// src/dense.py:108-161.  binary16 is emulated per operation in the reference
// (_HalfOps src/precision.py:118-150: every product / add / sqrt / div rounded to
// binary16, reductions as the pairwise tree of src/precision.py:106-115), after an
// exact power-of-two prescale that puts max|A_s| in [0.5, 1).  Whether that
// emulation collapses (tau = 2/v.v leaving the binary16 range -> RankDeficient)
// decides the precision escalation of src/solvers.py:255-279, so this kernel
// reproduces it operation for operation: same tree shape, same rounding points,
// no FMA contraction.  binary32 / binary64 run the same algorithm natively (the
// reference uses BLAS there, whose summation order is unspecified; we use the
// same fixed tree, deterministic run to run).
//
// The pairwise tree of src/precision.py:106-115 over L values is the left-aligned
// binary tree whose node (l, i) covers [i 2^l, min((i+1) 2^l, L)) and adds its two
// children when the right one is non-empty.  Its level-8 nodes are independent
// 256-element chunks, which makes a 2-D (chunk x column) decomposition exact.
// One cooperative persistent kernel, two grid barriers per column j:
//
//   phase 1  every (256-row chunk q, column c > j) warp unit computes the level-8
//            node of v_j . w[j:, c]: 8-leaf subtrees per lane, then a 5-level
//            shuffle tree (lane pairs at distance 1, 2, 4, 8, 16)
//   phase 2  every unit recomputes t_c = tau_j * root (levels 9.. over the chunk
//            nodes, identical in every unit) and applies w[j:, c] -= v_j * t_c to its
//            chunk (rounded product, rounded difference); CTA 0 updates column j+1 and,
//            in the same pass, the chunk nodes of x = w[j+1:, j+1] -> reflector j+1
//
// The reflector is kept in compact form, like LAPACK: v_j is column j below the
// diagonal with only v_0 = x_0 - alpha held apart (ctl), and alpha_j goes to a
// side array; R's diagonal and exact-zero lower triangle are produced by
// extract_r.  v.v differs from x.x only in element 0, so only chunk 0 is redone.
// The Q factor is not formed (build_preconditioner only uses R,
// src/solvers.py:196-197); see DESIGN.md for the reference's non-finite-Q check.
#include <cstdio>
#include <type_traits>
#include <vector>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace sk {
namespace qr {

constexpr int THREADS = 1024, WARPS = THREADS / 32;   // one CTA per SM, 32 warps to hide L2 latency
constexpr int CH = 256;          // chunk = level-8 subtree
constexpr int MAXCH = 1024;      // chunk nodes a single warp combines: d <= 262144

template <typename T>
struct Ctl {
    T tau[2];
    T v0[2];
    int fail_code;
    int fail_col;
};

// Level-8 node over chunk q of u_i * v_i, i in [q*CH, min((q+1)*CH, L)), by one warp.
// ov: bit 0 replaces u[0] by v0, bit 1 replaces v[0] by v0 (compact reflector).
template <typename T>
__device__ __forceinline__ T chunk_node(const T *u, const T *v, int L, int q, int ov = 0, T v0 = T()) {
    using O = LevelOps<T>;
    const int lane = threadIdx.x & 31;
    const int base = q * CH + lane * 8;
    const int cnt = max(0, min(8, L - base));
    T x[8];
    T node;
    if (cnt == 8 && (ov == 0 || base != 0)) {   // full leaves, no compact-reflector element: no guards
        bool paired = false;
        if constexpr (std::is_same<T, __half>::value) {
            // 4-byte aligned operands: the products and the first two tree levels as half2
            // ops (each half rounded like the scalar op, so the node is bitwise the same)
            if (((reinterpret_cast<uintptr_t>(u + base) | reinterpret_cast<uintptr_t>(v + base)) & 3) == 0) {
                const __half2 *u2 = reinterpret_cast<const __half2 *>(u + base);
                const __half2 *v2 = reinterpret_cast<const __half2 *>(v + base);
                const __half2 p0 = __hmul2_rn(u2[0], v2[0]), p1 = __hmul2_rn(u2[1], v2[1]);
                const __half2 p2 = __hmul2_rn(u2[2], v2[2]), p3 = __hmul2_rn(u2[3], v2[3]);
                const __half2 y01 = __hadd2_rn(__lows2half2(p0, p1), __highs2half2(p0, p1));   // (x0+x1, x2+x3)
                const __half2 y23 = __hadd2_rn(__lows2half2(p2, p3), __highs2half2(p2, p3));   // (x4+x5, x6+x7)
                const __half2 z = __hadd2_rn(__lows2half2(y01, y23), __highs2half2(y01, y23)); // (z0, z1)
                node = O::add(__low2half(z), __high2half(z));
                paired = true;
            }
        }
        if (!paired) {
#pragma unroll
            for (int e = 0; e < 8; ++e) x[e] = O::mul(u[base + e], v[base + e]);
            node = O::add(O::add(O::add(x[0], x[1]), O::add(x[2], x[3])), O::add(O::add(x[4], x[5]), O::add(x[6], x[7])));
        }
    } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            if (e < cnt) {
                const bool first = (base + e) == 0;
                const T a = (first && (ov & 1)) ? v0 : u[base + e];
                const T b = (first && (ov & 2)) ? v0 : v[base + e];
                x[e] = O::mul(a, b);
            } else {
                x[e] = O::zero();
            }
        }
        const T y0 = (1 < cnt) ? O::add(x[0], x[1]) : x[0];
        const T y1 = (3 < cnt) ? O::add(x[2], x[3]) : x[2];
        const T y2 = (5 < cnt) ? O::add(x[4], x[5]) : x[4];
        const T y3 = (7 < cnt) ? O::add(x[6], x[7]) : x[6];
        const int c1 = (cnt + 1) >> 1;
        const T z0 = (1 < c1) ? O::add(y0, y1) : y0;
        const T z1 = (3 < c1) ? O::add(y2, y3) : y2;
        const int c2 = (c1 + 1) >> 1;
        node = (1 < c2) ? O::add(z0, z1) : z0;
    }
#pragma unroll
    for (int s = 1; s < 32; s <<= 1) {
        const T other = __shfl_xor_sync(0xffffffffu, node, s);
        const bool left = (lane & s) == 0;
        const bool has_r = q * CH + (lane | s) * 8 < L;   // right child's first leaf exists
        const T l = left ? node : other, r = left ? other : node;
        node = has_r ? O::add(l, r) : l;
    }
    return node;
}

// Root of the tree over `count` level-8 nodes get(i), by one warp (count <= 1024).
// Lane l reduces the aligned block [l B, (l+1) B) of B leaves (B a power of two).
template <typename T, class G>
__device__ __forceinline__ T warp_tree_root(int count, G get) {
    using O = LevelOps<T>;
    const int lane = threadIdx.x & 31;
    int B = 1;
    while (B * 32 < count) B <<= 1;
    const int base = lane * B;
    int cnt = max(0, min(B, count - base));
    T node = O::zero();
    if (B == 1) {
        node = cnt ? get(base) : O::zero();
    } else {
        T buf[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) buf[e] = (e < cnt) ? get(base + e) : O::zero();
#pragma unroll
        for (int sz = 32; sz > 1; sz >>= 1) {
#pragma unroll
            for (int i = 0; i < sz / 2; ++i) buf[i] = (2 * i + 1 < cnt) ? O::add(buf[2 * i], buf[2 * i + 1]) : buf[2 * i];
            cnt = (cnt + 1) >> 1;
        }
        node = buf[0];
    }
#pragma unroll
    for (int s = 1; s < 32; s <<= 1) {
        const T other = __shfl_xor_sync(0xffffffffu, node, s);
        const bool left = (lane & s) == 0;
        const bool has_r = (lane | s) * B < count;
        const T l = left ? node : other, r = left ? other : node;
        node = has_r ? O::add(l, r) : l;
    }
    return node;
}

// Reflector for column jj given the chunk nodes of x.x in sh_nodes[0..nq), x = w[jj:, jj].
template <typename T>
__device__ int reflect_from_nodes(const T *x, int L, T *tau_out, T *v0_out, T *alphas, int jj, T *sh_nodes,
                                  T *sh_root) {
    using O = LevelOps<T>;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nq = (L + CH - 1) / CH;
    __shared__ T sh_v0, sh_tau, sh_alpha;
    __shared__ int sh_rc;
    if (warp == 0) {
        const T nrm = O::sqrt(warp_tree_root<T>(nq, [&](int i) { return sh_nodes[i]; }));
        int rc = SK_OK;
        T alpha = O::zero(), v0 = O::zero(), tau = O::zero();
        if (O::to_f64(nrm) == 0.0) {
            rc = SK_RANK_DEFICIENT;
        } else {
            const T x0 = x[0];
            alpha = (O::to_f64(x0) >= 0.0) ? O::sub(O::zero(), nrm) : nrm;   // -norm if x0 >= 0
            v0 = O::sub(x0, alpha);
            const T node0 = chunk_node<T>(x, x, L, 0, 3, v0);                 // v.v: chunk 0 redone
            if (lane == 0) sh_nodes[0] = node0;
            __syncwarp();
            const T vtv = warp_tree_root<T>(nq, [&](int i) { return sh_nodes[i]; });
            if (O::to_f64(vtv) == 0.0) {
                rc = SK_RANK_DEFICIENT;
            } else {
                tau = O::div(O::from_f64(2.0), vtv);
                if (!O::finite(tau)) rc = SK_RANK_DEFICIENT;
            }
        }
        if (lane == 0) { sh_rc = rc; sh_v0 = v0; sh_tau = tau; sh_alpha = alpha; }
    }
    __syncthreads();
    const int rc = sh_rc;
    if (rc == SK_OK && threadIdx.x == 0) {
        *tau_out = sh_tau;
        *v0_out = sh_v0;
        alphas[jj] = sh_alpha;
    }
    (void)sh_root;
    __syncthreads();
    return rc;
}

template <typename T>
__device__ int make_reflector(const T *w, int64_t ld, int d, int jj, T *tau_out, T *v0_out, T *alphas, T *sh_nodes,
                              T *sh_root) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int L = d - jj;
    const T *x = w + (int64_t)jj * ld + jj;
    const int nq = (L + CH - 1) / CH;
    for (int q = warp; q < nq; q += WARPS) {
        const T node = chunk_node<T>(x, x, L, q);
        if (lane == 0) sh_nodes[q] = node;
    }
    __syncthreads();
    return reflect_from_nodes<T>(x, L, tau_out, v0_out, alphas, jj, sh_nodes, sh_root);
}

template <typename T>
__global__ void __launch_bounds__(THREADS)
householder_kernel(T *w, int64_t ld, int d, int n, T *alphas /* n */, T *part /* nqmax x n */, Ctl<T> *ctl) {
    using O = LevelOps<T>;
    __shared__ T sh_nodes[MAXCH];
    __shared__ T sh_root;
    cg::grid_group grid = cg::this_grid();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int gwarp = blockIdx.x * WARPS + warp;
    const int nwarps = gridDim.x * WARPS;

    if (blockIdx.x == 0) {
        const int rc = make_reflector<T>(w, ld, d, 0, &ctl->tau[0], &ctl->v0[0], alphas, sh_nodes, &sh_root);
        if (rc != SK_OK && threadIdx.x == 0) { ctl->fail_code = rc; ctl->fail_col = 0; }
    }
    grid.sync();
    for (int j = 0; j < n - 1; ++j) {
        if (ctl->fail_code != SK_OK) return;   // uniform: read after a barrier
        const int buf = j & 1;
        const T *v = w + (int64_t)j * ld + j;  // compact reflector: v[0] is ctl->v0
        const T tau = ctl->tau[buf], v0 = ctl->v0[buf];
        const int L = d - j;
        const int nq = (L + CH - 1) / CH;
        const int ncols = n - j - 1;           // columns j+1 .. n-1
        // ---- phase 1: chunk nodes of v . w[j:, c]
        for (int u = gwarp; u < nq * ncols; u += 2 * nwarps) {   // two independent units in flight
            const int u2 = u + nwarps;
            const int q = u % nq, c = j + 1 + u / nq;
            const int q2 = u2 % nq, c2 = j + 1 + u2 / nq;
            const bool has2 = u2 < nq * ncols;
            const T node = chunk_node<T>(v, w + (int64_t)c * ld + j, L, q, 1, v0);
            const T node2 = has2 ? chunk_node<T>(v, w + (int64_t)c2 * ld + j, L, q2, 1, v0) : O::zero();
            if (lane == 0) {
                part[(size_t)q * n + c] = node;
                if (has2) part[(size_t)q2 * n + c2] = node2;
            }
        }
        grid.sync();
        // ---- phase 2
        if (blockIdx.x == 0) {
            // column j+1: t, update (rows j..), chunk nodes of x = w[j+1:, j+1], reflector j+1
            if (warp == 0) {
                const T root = warp_tree_root<T>(nq, [&](int i) { return part[(size_t)i * n + j + 1]; });
                if (lane == 0) sh_root = O::mul(tau, root);
            }
            __syncthreads();
            const T t = sh_root;
            T *colj = w + (int64_t)(j + 1) * ld + j;
            if (threadIdx.x == 0) colj[0] = O::sub(colj[0], O::mul(v0, t));   // R entry (row j)
            T *x = colj + 1;
            const T *vx = v + 1;
            const int Lx = L - 1, nqx = (Lx + CH - 1) / CH;
            for (int q = warp; q < nqx; q += WARPS) {
                const int base = q * CH + lane * 8;
                const int cnt = max(0, min(8, Lx - base));
#pragma unroll
                for (int e = 0; e < 8; ++e)
                    if (e < cnt) x[base + e] = O::sub(x[base + e], O::mul(vx[base + e], t));
                __syncwarp();
                const T node = chunk_node<T>(x, x, Lx, q);
                if (lane == 0) sh_nodes[q] = node;
            }
            __syncthreads();
            const int rc = reflect_from_nodes<T>(x, Lx, &ctl->tau[buf ^ 1], &ctl->v0[buf ^ 1], alphas, j + 1, sh_nodes,
                                                 &sh_root);
            if (rc != SK_OK && threadIdx.x == 0) { ctl->fail_code = rc; ctl->fail_col = j + 1; }
        } else {
            // CTA-major: CTA b >= 1 owns columns j+2+k*(G-1)+(b-1); its warps compute t_c for
            // all owned columns in parallel, then update (column, chunk) units, two in flight
            const int G1 = gridDim.x - 1, b1 = blockIdx.x - 1;
            const int rest = ncols - 1;                               // columns j+2 .. n-1
            const int mine = rest > b1 ? (rest - b1 + G1 - 1) / G1 : 0;
            for (int k = warp; k < mine; k += WARPS) {
                const int c = j + 2 + b1 + k * G1;
                const T root = warp_tree_root<T>(nq, [&](int i) { return part[(size_t)i * n + c]; });
                if (lane == 0) sh_nodes[k] = O::mul(tau, root);
            }
            __syncthreads();
            const int units = mine * nq;
            for (int u = warp; u < units; u += 2 * WARPS) {
                const int u2 = u + WARPS;
                const bool has2 = u2 < units;
                const int k1 = u / nq, q1 = u % nq, k2 = u2 / nq, q2 = u2 % nq;
                T *col1 = w + (int64_t)(j + 2 + b1 + k1 * G1) * ld + j + q1 * CH;
                T *col2 = w + (int64_t)(j + 2 + b1 + (has2 ? k2 : k1) * G1) * ld + j + (has2 ? q2 : q1) * CH;
                const T t1 = sh_nodes[k1], t2 = has2 ? sh_nodes[k2] : O::zero();
                const int cnt1 = min(CH, L - q1 * CH), cnt2 = has2 ? min(CH, L - q2 * CH) : 0;
                const T *v1 = v + q1 * CH, *v2 = v + (has2 ? q2 : q1) * CH;
#pragma unroll 4
                for (int i = lane; i < CH; i += 32) {
                    T a1 = O::zero(), a2 = O::zero(), x1 = O::zero(), x2 = O::zero();
                    if (i < cnt1) { a1 = col1[i]; x1 = (q1 == 0 && i == 0) ? v0 : v1[i]; }
                    if (i < cnt2) { a2 = col2[i]; x2 = (q2 == 0 && i == 0) ? v0 : v2[i]; }
                    if (i < cnt1) col1[i] = O::sub(a1, O::mul(x1, t1));
                    if (i < cnt2) col2[i] = O::sub(a2, O::mul(x2, t2));
                }
            }
            __syncthreads();
        }
        grid.sync();
    }
}

// ---------------------------------------------------------------------------
// Dataflow variant: no grid barriers.  Column c (> 0) is owned by CTA c mod G and only
// its owner ever updates it, in reflector order.  Reflector j+1 is formed by the owner
// of column j+1 right after applying reflector j to that column (before its other
// columns) and published through flags[j+1]; every CTA waits on that flag alone before
// applying reflector j+1.  The arithmetic (chunk trees, update order, scalar ops) is the
// barrier kernel's, so R is bitwise the same.
// SMEM = true: CTA b keeps its columns c = b + q G in shared memory for the whole
// factorisation (binary16 at d x n = 6144 x 2048 on 148 SMs: 14 x 12 KB); the leader
// stores the finished reflector column to global memory before publishing it, and every
// CTA writes its columns back at the end.  Same arithmetic, so R is bitwise the same.
template <typename T, bool SMEM>
__global__ void __launch_bounds__(THREADS)
householder_flow_kernel(T *w, int64_t ld, int d, int n, T *alphas, T *part /* nqmax x n */, T *taus, T *v0s,
                        int *flags, Ctl<T> *ctl, int qs) {
    using O = LevelOps<T>;
    __shared__ T sh_nodes[MAXCH];
    __shared__ T sh_t[MAXCH];
    __shared__ T sh_root;
    __shared__ int sh_flag;
    extern __shared__ __align__(16) unsigned char qr_dyn[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int G = gridDim.x, b = blockIdx.x;
    const int nloc = b < n ? (n - b + G - 1) / G : 0;
    const int nqd = (d + CH - 1) / CH;
    // SMEM with qs > 0 (binary32 / binary64 at 6144 x 2048 do not fit whole): the CTA's
    // first qs local columns stay in global memory, the later ones (which take the most
    // reflector updates) in shared memory; all accesses go through generic pointers
    T *sm_cols = reinterpret_cast<T *>(qr_dyn);                         // (nloc - qs) x d
    T *sm_part = sm_cols + (SMEM ? (size_t)max(nloc - qs, 0) * d : 0); // nloc x nqd chunk nodes
    // owned column c (c mod G == b)
    auto in_smem = [&](int c) { return SMEM && c / G >= qs; };
    auto col = [&](int c) -> T * {
        return in_smem(c) ? sm_cols + (size_t)(c / G - qs) * d : w + (int64_t)c * ld;
    };
    auto part_at = [&](int k, int q, int c) -> T & { return SMEM ? sm_part[k * nqd + q] : part[(size_t)q * n + c]; };
    if (SMEM) {
        for (int q = qs; q < nloc; ++q) {
            const T *src = w + (int64_t)(b + q * G) * ld;
            T *dst = sm_cols + (size_t)(q - qs) * d;
            for (int i = threadIdx.x; i < d; i += THREADS) dst[i] = src[i];
        }
        __syncthreads();
    }

    auto publish = [&](int jj, int rc) {
        __syncthreads();
        if (threadIdx.x == 0) {
            if (rc != SK_OK) { ctl->fail_code = rc; ctl->fail_col = jj; }
            __threadfence();
            atomicExch(flags + jj, rc == SK_OK ? 1 : 2);
        }
    };
    if (b == 0) publish(0, make_reflector<T>(w, ld, d, 0, taus, v0s, alphas, sh_nodes, &sh_root));
    for (int j = 0; j < n - 1; ++j) {
        if (threadIdx.x == 0) sh_flag = wait_flag(flags + j);
        __syncthreads();
        if (sh_flag != 1) {                        // failure upstream (or a stuck chain)
            if (sh_flag < 0 && threadIdx.x == 0) { ctl->fail_code = SK_ERR_CUDA; ctl->fail_col = j; }
            return;
        }
        const T tau = *reinterpret_cast<volatile T *>(taus + j), v0 = *reinterpret_cast<volatile T *>(v0s + j);
        const T *v = w + (int64_t)j * ld + j;
        const int L = d - j, nq = (L + CH - 1) / CH;
        int c0 = j + 1 + ((b - (j + 1)) % G + G) % G;   // first owned column > j
        if (c0 == j + 1) {
            // ---- leader: column j+1 first, then reflector j+1
            for (int q = warp; q < nq; q += WARPS) {
                const T node = chunk_node<T>(v, col(j + 1) + j, L, q, 1, v0);
                if (lane == 0) sh_nodes[q] = node;
            }
            __syncthreads();
            if (warp == 0) {
                const T root = warp_tree_root<T>(nq, [&](int i) { return sh_nodes[i]; });
                if (lane == 0) sh_root = O::mul(tau, root);
            }
            __syncthreads();
            const T t = sh_root;
            T *colj = col(j + 1) + j;
            if (threadIdx.x == 0) colj[0] = O::sub(colj[0], O::mul(v0, t));   // R entry (row j)
            T *x = colj + 1;
            const T *vx = v + 1;
            const int Lx = L - 1, nqx = (Lx + CH - 1) / CH;
            for (int q = warp; q < nqx; q += WARPS) {
                const int base = q * CH + lane * 8;
                const int cnt = max(0, min(8, Lx - base));
#pragma unroll
                for (int e = 0; e < 8; ++e)
                    if (e < cnt) x[base + e] = O::sub(x[base + e], O::mul(vx[base + e], t));
                __syncwarp();
                const T node = chunk_node<T>(x, x, Lx, q);
                if (lane == 0) sh_nodes[q] = node;
            }
            __syncthreads();
            const int rc = j + 1 < n ? reflect_from_nodes<T>(x, Lx, taus + j + 1, v0s + j + 1, alphas, j + 1,
                                                             sh_nodes, &sh_root)
                                     : SK_OK;
            if (in_smem(j + 1)) {   // the reflector column (rows j+1..) goes to global memory for the other CTAs
                T *dst = w + (int64_t)(j + 1) * ld;
                for (int i = j + 1 + threadIdx.x; i < d; i += THREADS) dst[i] = colj[i - j];
                __threadfence();
            }
            publish(j + 1, rc);
            c0 += G;
        }
        // ---- the rest of the owned columns: t_c = tau * root(v . w[j:, c]), then the update
        const int mine = c0 < n ? (n - 1 - c0) / G + 1 : 0;
        if (mine == 0) continue;
        const int units = mine * nq;
        for (int u = warp, k = warp / nq, q = warp % nq; u < units; u += WARPS) {   // (k, q) = (u / nq, u % nq)
            const int c = c0 + k * G;
            const T node = chunk_node<T>(v, col(c) + j, L, q, 1, v0);
            if (lane == 0) part_at(k, q, c) = node;
            for (q += WARPS; q >= nq; q -= nq) ++k;
        }
        __syncthreads();
        for (int k = warp; k < mine; k += WARPS) {
            const int c = c0 + k * G;
            const T root = warp_tree_root<T>(nq, [&](int i) { return part_at(k, i, c); });
            if (lane == 0) sh_t[k] = O::mul(tau, root);
        }
        __syncthreads();
        for (int u = warp, kn = warp / nq, qn = warp % nq; u < units; u += 2 * WARPS) {
            const int u2 = u + WARPS;
            const bool has2 = u2 < units;
            const int k1 = kn, q1 = qn;                 // (u / nq, u % nq)
            int k2 = k1, q2 = q1;                       // (u2 / nq, u2 % nq)
            for (q2 += WARPS; q2 >= nq; q2 -= nq) ++k2;
            kn = k2;                                    // next u = u2 + WARPS
            for (qn = q2 + WARPS; qn >= nq; qn -= nq) ++kn;
            T *col1 = col(c0 + k1 * G) + j + q1 * CH;
            T *col2 = col(c0 + (has2 ? k2 : k1) * G) + j + (has2 ? q2 : q1) * CH;
            const T t1 = sh_t[k1], t2 = has2 ? sh_t[k2] : O::zero();
            const int cnt1 = min(CH, L - q1 * CH), cnt2 = has2 ? min(CH, L - q2 * CH) : 0;
            const T *v1 = v + q1 * CH, *v2 = v + (has2 ? q2 : q1) * CH;
            if (cnt1 == CH && cnt2 == CH && q1 != 0 && q2 != 0) {   // two full chunks without v_0: no guards
                if (std::is_same<T, __half>::value && (ld & 1) == 0 && (d & 1) == 0) {
                    // element pairs on 4-byte boundaries (column and reflector share the parity
                    // of j): HMUL2 / HSUB2 round each half exactly like the scalar ops
                    const int off = j & 1;
                    const __half2 tt1 = __half2half2(t1), tt2 = __half2half2(t2);
#pragma unroll
                    for (int r = 0; r < CH / 64; ++r) {
                        const int i = off + 2 * (lane + 32 * r);
                        if (i + 1 < CH) {
                            __half2 *p1 = reinterpret_cast<__half2 *>(col1 + i), *p2 = reinterpret_cast<__half2 *>(col2 + i);
                            const __half2 a1 = *p1, a2 = *p2;
                            const __half2 x1 = *reinterpret_cast<const __half2 *>(v1 + i);
                            const __half2 x2 = *reinterpret_cast<const __half2 *>(v2 + i);
                            *p1 = __hsub2_rn(a1, __hmul2_rn(x1, tt1));
                            *p2 = __hsub2_rn(a2, __hmul2_rn(x2, tt2));
                        }
                    }
                    if (off && lane < 2) {     // odd j: elements 0 and CH - 1 stay single
                        const int i = lane ? CH - 1 : 0;
                        col1[i] = O::sub(col1[i], O::mul(v1[i], t1));
                        col2[i] = O::sub(col2[i], O::mul(v2[i], t2));
                    }
                } else {
#pragma unroll
                    for (int i = lane; i < CH; i += 32) {
                        const T a1 = col1[i], a2 = col2[i], x1 = v1[i], x2 = v2[i];
                        col1[i] = O::sub(a1, O::mul(x1, t1));
                        col2[i] = O::sub(a2, O::mul(x2, t2));
                    }
                }
                continue;
            }
#pragma unroll 4
            for (int i = lane; i < CH; i += 32) {
                T a1 = O::zero(), a2 = O::zero(), x1 = O::zero(), x2 = O::zero();
                if (i < cnt1) { a1 = col1[i]; x1 = (q1 == 0 && i == 0) ? v0 : v1[i]; }
                if (i < cnt2) { a2 = col2[i]; x2 = (q2 == 0 && i == 0) ? v0 : v2[i]; }
                if (i < cnt1) col1[i] = O::sub(a1, O::mul(x1, t1));
                if (i < cnt2) col2[i] = O::sub(a2, O::mul(x2, t2));
            }
        }
        __syncthreads();
    }
    if (SMEM) {
        __syncthreads();
        for (int q = qs; q < nloc; ++q) {
            T *dst = w + (int64_t)(b + q * G) * ld;
            const T *src = sm_cols + (size_t)(q - qs) * d;
            for (int i = threadIdx.x; i < d; i += THREADS) dst[i] = src[i];
        }
    }
}

// prescale for binary16: max |A_s| (as f64)
__global__ void maxabs_half(const __half *a, int64_t count, unsigned long long *out_bits) {
    double mx = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
        mx = fmax(mx, fabs((double)__half2float(a[i])));
    mx = warp_max(mx);
    if ((threadIdx.x & 31) == 0) atomicMax(out_bits, (unsigned long long)__double_as_longlong(mx));
}
// the power-of-two scale from the device max (deferred verdicts: no host round trip);
// a zero matrix records RankDeficient and keeps scale 1
__global__ void half_scale_from_bits(const unsigned long long *bits, double *scale, DevStatus *ds) {
    const double maxabs = __longlong_as_double((long long)*bits);
    if (maxabs == 0.0) {
        *scale = 1.0;
        if (ds->code == 0) { ds->code = SK_RANK_DEFICIENT; ds->index = -1; ds->value = 0.0; ds->aux = 0.0; }
        return;
    }
    int e = 0;
    frexp(maxabs, &e);
    *scale = ldexp(1.0, -e);
}
__global__ void prescale_half(__half *a, int64_t count, double scale, const double *scale_dev) {
    if (scale_dev) scale = *scale_dev;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
        a[i] = __double2half((double)__half2float(a[i]) * scale);   // round_to_precision(work*scale, binary16)
}

// R (row-major f64) = promote(upper part, alphas on the diagonal, exact zeros below) / scale;
// non-finite entries are counted (src/precision.py:200 checks the binary16 R)
template <typename T>
__global__ void extract_r(const T *w, int64_t ld, const T *alphas, int n, double scale, double *r, int64_t ldr,
                          int *nonfinite, const double *scale_dev) {
    if (scale_dev) scale = *scale_dev;
    const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= (int64_t)n * n) return;
    const int i = (int)(idx / n), c = (int)(idx % n);
    T x = LevelOps<T>::zero();
    if (i < c) x = w[(int64_t)c * ld + i];
    else if (i == c) x = alphas[c];
    if (!LevelOps<T>::finite(x)) atomicAdd(nonfinite, 1);
    r[(int64_t)i * ldr + c] = LevelOps<T>::to_f64(x) / scale;
}

inline int64_t nq_max(int64_t d) { return (d + CH - 1) / CH; }

constexpr int NBQ = 64;          // panel width of the blocked (WY) binary32 / binary64 QR
constexpr int64_t BLOCKED_MAX_D = 32768;   // sketch heights; taller (TSQR blocks) keep the dataflow kernel
constexpr int QRB_SPLIT_MAX = 32;          // row slabs of the V^T [V | A_trail] products

template <typename T>
size_t blocked_ws_bytes(int64_t d, int64_t n) {
    if (std::is_same<T, __half>::value || d > BLOCKED_MAX_D || n <= NBQ) return 0;
    const size_t one = align_up((size_t)d * NBQ * sizeof(T), 256) + 2 * align_up((size_t)NBQ * NBQ * sizeof(T), 256) +
                       2 * align_up((size_t)NBQ * n * sizeof(T), 256) +   // V, V^T V, T, G, W
                       align_up((size_t)QRB_SPLIT_MAX * NBQ * std::max<int64_t>(n, NBQ) * sizeof(T), 256);   // partials
    return 2 * one;   // the lookahead pipeline keeps two sets (panel parity / stream)
}

template <typename T>
size_t ws_bytes(int64_t d, int64_t n) {
    return align_up(sizeof(Ctl<T>), 256) + align_up((size_t)n * sizeof(T), 256) +
           align_up((size_t)nq_max(d) * n * sizeof(T), 256) + 256 +
           2 * align_up((size_t)n * sizeof(T), 256) + align_up((size_t)n * sizeof(int), 256) +   // flow kernel
           blocked_ws_bytes<T>(d, n);
}

// ---------------------------------------------------- blocked (WY) QR pieces --
// binary32 / binary64: panels of NBQ columns are factored by the dataflow kernel (one
// column per CTA, so a reflector step is one column's work, not a CTA's 14), and the
// trailing columns take the panel's reflectors at once in compact WY form,
// A_trail <- (I - V T^T V^T) A_trail = A_trail - V (T^T (V^T A_trail)), with T from
// LAPACK's forward columnwise recurrence (xLARFT).  All arithmetic in the level type
// (true FP32 for binary32); the reference's own order here is BLAS-defined
// (src/precision.py:181-187), so R agrees to level roundoff, with the reference's
// sign convention (the panel reflectors are the same Householder steps).

// Panel factorisation on one thread-block cluster (QPC_CL CTAs, the panel's rows split
// in contiguous slabs held in shared memory), ONE cluster barrier per column: each CTA
// publishes, for column j, the partial sum of squares of x = P[j:, j] below the diagonal
// and the partial dots x . P[j:, c] for every later column c (row j included), plus -- on
// the CTA owning row j -- x0 and the row-j entries P[j, c]; after the barrier every CTA
// sums the partials in rank order (distributed shared memory) and forms alpha, v0, tau and
// v . P[:, c] = x . P[:, c] - alpha P[j, c] identically, then updates its slab.  The
// partial records alternate between two buffers, so a CTA may write column j+1's while a
// slower one still reads column j's.  Same Householder step and sign convention as
// householder_reduce (src/dense.py:137-160): norm 0, v.v 0 and a non-finite tau raise
// RankDeficient.  At the end the CTAs form V^T V of the panel (cluster-reduced) and rank
// 0 builds T = (diag(1/tau) + striu(V^T V))^-1 (the compact-WY T of xLARFT).
constexpr int QPC_THREADS = 512, QPC_WARPS = QPC_THREADS / 32;
constexpr int QPC_CL = 8;
template <typename T, int NBP, int CL>
__global__ void __launch_bounds__(QPC_THREADS) qrb_panel_cluster(T *wp, int64_t ld, int dv, int nbp, int slab,
                                                                  T *alphas, T *taus, T *v0s, Ctl<T> *ctl, int col0,
                                                                  T *tm /* NBQ x NBQ, col-major */, T *sbuf) {
    using O = LevelOps<T>;
    cg::cluster_group cluster = cg::this_cluster();
    extern __shared__ __align__(16) unsigned char qpc_raw[];
    T *P = reinterpret_cast<T *>(qpc_raw);                 // [NBP][slab]: this CTA's rows of the panel
    // partial record per buffer: [0] sum x^2 below the diagonal, [1] x0 (owner), [2 + c] dot x.P_c,
    // [2 + NBP + c] P[j, c] (owner)
    __shared__ T rec[2][2 + 2 * NBP];
    __shared__ T red[QPC_WARPS];
    __shared__ T tcol[NBP];
    __shared__ T vtv[NBP][NBP + 1];
    __shared__ T tau_s[NBP];
    const int rank = (int)cluster.block_rank();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int r_lo = rank * slab, r_hi = min(dv, r_lo + slab), nr = max(0, r_hi - r_lo);
    for (int c = 0; c < nbp; ++c)
        for (int i = tid; i < nr; i += QPC_THREADS) P[c * slab + i] = wp[(int64_t)c * ld + r_lo + i];
    __syncthreads();
    int done = nbp;
    for (int j = 0; j < nbp; ++j) {
        T *rb = rec[j & 1];
        const bool own = j >= r_lo && j < r_hi;
        const int i0 = max(0, j + 1 - r_lo);               // first slab row below the diagonal
        // ---- partials of column j: sum of squares (rows > j), dots with later columns (rows >= j)
        T sq = O::zero();
        for (int i = i0 + tid; i < nr; i += QPC_THREADS) { const T x = P[j * slab + i]; sq = sq + x * x; }
        for (int o = 16; o > 0; o >>= 1) sq = sq + __shfl_xor_sync(0xffffffffu, sq, o);
        if (lane == 0) red[warp] = sq;
        const T *pjc = P + j * slab;
        for (int c = j + 1 + warp; c < nbp; c += QPC_WARPS) {
            const T *pcc = P + c * slab;
            T d0 = O::zero(), d1 = O::zero();
            int i = i0 + lane;
            for (; i + 32 < nr; i += 64) {
                d0 = d0 + pjc[i] * pcc[i];
                d1 = d1 + pjc[i + 32] * pcc[i + 32];
            }
            if (i < nr) d0 = d0 + pjc[i] * pcc[i];
            T dsum = d0 + d1;
            for (int o = 16; o > 0; o >>= 1) dsum = dsum + __shfl_xor_sync(0xffffffffu, dsum, o);
            if (lane == 0) {
                const T pj = own ? P[c * slab + (j - r_lo)] : O::zero();
                const T xj = own ? P[j * slab + (j - r_lo)] : O::zero();
                rb[2 + c] = dsum + xj * pj;
                rb[2 + NBP + c] = pj;
            }
        }
        __syncthreads();
        if (tid == 0) {
            T t = O::zero();
            for (int k = 0; k < QPC_WARPS; ++k) t = t + red[k];
            rb[0] = t;
            rb[1] = own ? P[j * slab + (j - r_lo)] : O::zero();
        }
        cluster.sync();
        // ---- alpha, v0, tau and t_c (identical in every CTA: fixed rank order)
        // all remote loads in flight first (a distributed-shared-memory read is a round trip
        // through the cluster network), then the fixed-order sums
        T rs_[CL], xs_[CL];
#pragma unroll
        for (int k = 0; k < CL; ++k) {
            const T *ps = cluster.map_shared_rank(rb, k);
            rs_[k] = ps[0];
            xs_[k] = ps[1];
        }
        T rest = rs_[0], x0 = xs_[0];
#pragma unroll
        for (int k = 1; k < CL; ++k) {
            rest = rest + rs_[k];
            x0 = x0 + xs_[k];
        }
        const T nrm = O::sqrt(rest + x0 * x0);
        const T alpha = (x0 >= O::zero()) ? -nrm : nrm;
        const T v0 = x0 - alpha;
        const T vv = rest + v0 * v0;
        const T tau = T(2) / vv;
        if ((nrm == O::zero()) || (vv == O::zero()) || !O::finite(tau)) {
            if (rank == 0 && tid == 0 && ctl->fail_code == SK_OK) {
                ctl->fail_code = SK_RANK_DEFICIENT;
                ctl->fail_col = col0 + j;
            }
            done = j;
            break;   // uniform over the cluster (same values everywhere)
        }
        for (int c = j + 1 + tid; c < nbp; c += QPC_THREADS) {
            T dxs[CL], pjs[CL];
#pragma unroll
            for (int k = 0; k < CL; ++k) {
                const T *ps = cluster.map_shared_rank(rb, k);
                dxs[k] = ps[2 + c];
                pjs[k] = ps[2 + NBP + c];
            }
            T dx = dxs[0], pj = pjs[0];
#pragma unroll
            for (int k = 1; k < CL; ++k) {
                dx = dx + dxs[k];
                pj = pj + pjs[k];
            }
            tcol[c] = tau * (dx - alpha * pj);               // tau v . P[:, c]
        }
        if (tid == 0) tau_s[j] = tau;
        __syncthreads();
        // ---- update the later columns of this slab: P[:, c] -= t_c v (v_j = v0 on row j)
        for (int c = j + 1 + warp; c < nbp; c += QPC_WARPS) {
            const T tc = tcol[c];
            T *pcc = P + c * slab;
            int i = i0 + lane;
#pragma unroll 1
            for (; i + 96 < nr; i += 128) {
                const T a0 = pcc[i], a1 = pcc[i + 32], a2 = pcc[i + 64], a3 = pcc[i + 96];
                const T x0_ = pjc[i], x1_ = pjc[i + 32], x2_ = pjc[i + 64], x3_ = pjc[i + 96];
                pcc[i] = a0 - tc * x0_;
                pcc[i + 32] = a1 - tc * x1_;
                pcc[i + 64] = a2 - tc * x2_;
                pcc[i + 96] = a3 - tc * x3_;
            }
            for (; i < nr; i += 32) pcc[i] = pcc[i] - tc * pjc[i];
            if (lane == 0 && own) pcc[j - r_lo] = pcc[j - r_lo] - tc * v0;
        }
        if (tid == 0 && own) P[j * slab + (j - r_lo)] = v0;  // compact storage: v on and below the diagonal
        if (rank == 0 && tid == 0) { alphas[j] = alpha; taus[j] = tau; v0s[j] = v0; }
        __syncthreads();
    }
    // ---- V^T V of the panel (rows >= the reflector's diagonal; zeros above it), one warp per entry
    if (done == nbp && tm) {
        for (int e = warp; e < nbp * nbp; e += QPC_WARPS) {
            const int a_ = e % nbp, b_ = e / nbp;
            if (a_ > b_) continue;                           // upper triangle incl. diagonal
            T sacc = O::zero();
            const int ilo = max(0, b_ - r_lo);               // V[:, a] and V[:, b] both live from row b
            for (int i = ilo + lane; i < nr; i += 32) sacc = sacc + P[a_ * slab + i] * P[b_ * slab + i];
            for (int o = 16; o > 0; o >>= 1) sacc = sacc + __shfl_xor_sync(0xffffffffu, sacc, o);
            if (lane == 0) vtv[a_][b_] = sacc;
        }
    }
    __syncthreads();
    for (int c = 0; c < nbp; ++c)
        for (int i = tid; i < nr; i += QPC_THREADS) wp[(int64_t)c * ld + r_lo + i] = P[c * slab + i];
    cluster.sync();   // every CTA's partials are ready and its slab is written back (P is free)
    if (done == nbp && tm && rank == 0) {
        // S = diag(1/tau) + striu(V^T V) summed over the CTAs, staged in the freed slab area
        T *Ssm = P;                                          // [NBP][NBP + 1]
        T *Tsm = P + NBP * (NBP + 1);                        // [NBP][NBP + 1]: column b of T in Tsm[.][b]
        for (int e = tid; e < nbp * nbp; e += QPC_THREADS) {
            const int a_ = e % nbp, b_ = e / nbp;
            if (a_ >= b_) continue;
            T vs_[CL];
#pragma unroll
            for (int k = 0; k < CL; ++k) vs_[k] = *cluster.map_shared_rank(&vtv[a_][b_], k);
            T sacc = vs_[0];
#pragma unroll
            for (int k = 1; k < CL; ++k) sacc = sacc + vs_[k];
            Ssm[a_ * (NBP + 1) + b_] = sacc;
        }
        __syncthreads();
        if (tid < nbp) {   // column b of T = S^-1: t_b = tau_b, t_r = -tau_r sum_{r<k<=b} S_rk t_k
            const int b_ = tid;
            Tsm[b_ * (NBP + 1) + b_] = tau_s[b_];
            for (int r = b_ - 1; r >= 0; --r) {
                T sacc = O::zero();
                for (int k = r + 1; k <= b_; ++k) sacc = sacc + Ssm[r * (NBP + 1) + k] * Tsm[k * (NBP + 1) + b_];
                Tsm[r * (NBP + 1) + b_] = -tau_s[r] * sacc;
            }
            for (int r = 0; r <= b_; ++r) tm[(int64_t)b_ * NBQ + r] = Tsm[r * (NBP + 1) + b_];
        }
    }
    cluster.sync();   // no CTA leaves while rank 0 may still read its shared memory
}

// Short panels (dv <= PANEL_SMALL_ROWS): the panel lives in REGISTERS, column c in warp
// c % 32 (lane l holds rows l, l + 32, ...), one CTA of 1024 threads.  Per column the
// owner warp forms the reflector (sum of squares below the diagonal, the reference's
// alpha = -sign(x0) |x|, v0 = x0 - alpha, tau = 2 / v^T v, the RankDeficient checks)
// and publishes v through a double-buffered shared row, so each column costs ONE
// __syncthreads; every warp then applies H to its own later columns (v . P_c by a warp
// reduction, P_c -= tau (v . P_c) v).  V^T V (one thread per entry over an odd-pitch
// shared copy of V) and T = (diag(1/tau) + striu(V^T V))^-1 (back substitution, one
// thread per column) follow as in the cluster kernel.  Same outputs as
// qrb_panel_cluster; binary32/64 order is BLAS-defined in the reference
// (src/precision.py:181-187), so the different reduction shape is legal.
constexpr int QPS_THREADS = 1024;
// rows per lane: 16 (binary32, dv <= 512); 12 (binary64, dv <= 384: 64 registers per thread)
template <typename T> constexpr int qps_rpl() { return sizeof(T) == 8 ? 12 : 16; }
template <typename T> constexpr int panel_small_rows() { return 32 * qps_rpl<T>(); }
template <typename T, int NBP, int QPS_RPL>
__global__ void __launch_bounds__(QPS_THREADS, 1) qrb_panel_small(T *wp, int64_t ld, int dv, int nbp, T *alphas,
                                                                 T *taus, T *v0s, Ctl<T> *ctl, int col0, T *tm) {
    using O = LevelOps<T>;
    constexpr int PANEL_SMALL_ROWS = panel_small_rows<T>();   // (QPS_RPL = ceil(dv / 32), even)
    constexpr int CPW = (NBP + 31) / 32;
    extern __shared__ __align__(16) unsigned char qps_raw[];
    T *vb = reinterpret_cast<T *>(qps_raw);             // [2][PANEL_SMALL_ROWS]: the current reflector
    __shared__ T s_tau[NBP];
    __shared__ T Ssm[NBP][NBP + 1], Tsm[NBP][NBP + 1];
    __shared__ int s_fail;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    T x[CPW][QPS_RPL];
#pragma unroll
    for (int q = 0; q < CPW; ++q) {
        const int c = warp + 32 * q;
#pragma unroll
        for (int t = 0; t < QPS_RPL; ++t) {
            const int i = lane + 32 * t;
            x[q][t] = (c < nbp && i < dv) ? wp[(int64_t)c * ld + i] : O::zero();
        }
    }
    if (tid == 0) s_fail = -1;
    __syncthreads();
    int done = nbp;
    for (int j = 0; j < nbp; ++j) {
        T *v = vb + (j & 1) * PANEL_SMALL_ROWS;
        if (warp == (j & 31)) {
            const int qj = j >> 5;
            T sq = O::zero(), xj = O::zero();
#pragma unroll
            for (int q = 0; q < CPW; ++q) {              // (static register indices only)
                if (q != qj) continue;
#pragma unroll
                for (int t = 0; t < QPS_RPL; ++t) {
                    const int i = lane + 32 * t;
                    const T xv = x[q][t];
                    if (i > j && i < dv) sq = sq + xv * xv;
                    if (i == j) xj = xv;
                }
            }
            for (int o = 16; o > 0; o >>= 1) sq = sq + __shfl_xor_sync(0xffffffffu, sq, o);
            const T x0 = __shfl_sync(0xffffffffu, xj, j & 31);
            const T nrm = O::sqrt(sq + x0 * x0);
            const T alpha = (x0 >= O::zero()) ? -nrm : nrm;
            const T v0 = x0 - alpha;
            const T vv = sq + v0 * v0;
            const T tau = T(2) / vv;
            if ((nrm == O::zero()) || (vv == O::zero()) || !O::finite(tau)) {
                if (lane == 0) {
                    s_fail = j;
                    if (ctl->fail_code == SK_OK) { ctl->fail_code = SK_RANK_DEFICIENT; ctl->fail_col = col0 + j; }
                }
            } else {
#pragma unroll
                for (int q = 0; q < CPW; ++q) {
                    if (q != qj) continue;
#pragma unroll
                    for (int t = 0; t < QPS_RPL; ++t) {
                        const int i = lane + 32 * t;
                        if (i == j) x[q][t] = v0;            // compact storage: v0 on the diagonal
                        v[i] = (i >= j && i < dv) ? x[q][t] : O::zero();
                    }
                }
                if (lane == 0) { s_tau[j] = tau; alphas[j] = alpha; taus[j] = tau; v0s[j] = v0; }
            }
        }
        __syncthreads();
        if (s_fail >= 0) { done = s_fail; break; }      // uniform
        const T tau = s_tau[j];
#pragma unroll
        for (int q = 0; q < CPW; ++q) {
            const int c = warp + 32 * q;
            if (c > j && c < nbp) {
                T dsum = O::zero();
#pragma unroll
                for (int t = 0; t < QPS_RPL; ++t) dsum = dsum + v[lane + 32 * t] * x[q][t];
                for (int o = 16; o > 0; o >>= 1) dsum = dsum + __shfl_xor_sync(0xffffffffu, dsum, o);
                const T tc = tau * dsum;
                // (v is zero above j and below dv, so the whole register column takes the
                // update unpredicated: x - tc * 0 == x)
#pragma unroll
                for (int t = 0; t < QPS_RPL; ++t) x[q][t] = x[q][t] - tc * v[lane + 32 * t];
            }
        }
    }
    // write back (R above the diagonal, v0 on it, v below it)
#pragma unroll
    for (int q = 0; q < CPW; ++q) {
        const int c = warp + 32 * q;
        if (c < nbp) {
#pragma unroll
            for (int t = 0; t < QPS_RPL; ++t) {
                const int i = lane + 32 * t;
                if (i < dv) wp[(int64_t)c * ld + i] = x[q][t];
            }
        }
    }
    if (done != nbp || !tm) return;                      // uniform
    T *Vs = vb + 2 * PANEL_SMALL_ROWS;                   // [NBP][ldv]: V, zeros above the diagonal
    const int ldv = dv | 1;                              // odd pitch: conflict-free column reads
#pragma unroll
    for (int q = 0; q < CPW; ++q) {
        const int c = warp + 32 * q;
        if (c < nbp) {
#pragma unroll
            for (int t = 0; t < QPS_RPL; ++t) {
                const int i = lane + 32 * t;
                if (i < dv) Vs[c * ldv + i] = i < c ? O::zero() : x[q][t];
            }
        }
    }
    __syncthreads();
    for (int e = tid; e < nbp * nbp; e += QPS_THREADS) {   // S = striu(V^T V), one thread per entry
        const int a_ = e % nbp, b_ = e / nbp;
        if (a_ >= b_) continue;
        const T *va = Vs + a_ * ldv, *vbb = Vs + b_ * ldv;
        T s0 = O::zero(), s1 = O::zero();
        int i = b_;
        for (; i + 1 < dv; i += 2) {
            s0 = s0 + va[i] * vbb[i];
            s1 = s1 + va[i + 1] * vbb[i + 1];
        }
        if (i < dv) s0 = s0 + va[i] * vbb[i];
        Ssm[a_][b_] = s0 + s1;
    }
    __syncthreads();
    if (tid < nbp) {   // column b of T = S^-1: t_b = tau_b, t_r = -tau_r sum_{r<k<=b} S_rk t_k
        const int b_ = tid;
        Tsm[b_][b_] = s_tau[b_];
        for (int r = b_ - 1; r >= 0; --r) {
            T s0 = O::zero(), s1 = O::zero(), s2 = O::zero(), s3 = O::zero();   // four chains
            int k = r + 1;
            for (; k + 3 <= b_; k += 4) {
                s0 = s0 + Ssm[r][k] * Tsm[k][b_];
                s1 = s1 + Ssm[r][k + 1] * Tsm[k + 1][b_];
                s2 = s2 + Ssm[r][k + 2] * Tsm[k + 2][b_];
                s3 = s3 + Ssm[r][k + 3] * Tsm[k + 3][b_];
            }
            for (; k <= b_; ++k) s0 = s0 + Ssm[r][k] * Tsm[k][b_];
            Tsm[r][b_] = -s_tau[r] * ((s0 + s1) + (s2 + s3));
        }
        for (int r = 0; r <= b_; ++r) tm[(int64_t)b_ * NBQ + r] = Tsm[r][b_];
    }
}

// Panels of at most PANEL_ONE_CTA_ROWS rows are factored by ONE CTA (a cluster of 1:
// every reduction stays in its shared memory, no distributed-shared-memory round trips;
// config 1's 300 x 64 panel: ~3.7 -> ~1 us per column); taller ones by the 8-CTA cluster.
constexpr int PANEL_ONE_CTA_ROWS = 768;
inline int panel_cl(int dv) { return dv <= PANEL_ONE_CTA_ROWS ? 1 : QPC_CL; }
template <typename T, int NBW>
size_t panel_smem(int dv) {
    const int slab = (dv + panel_cl(dv) - 1) / panel_cl(dv);
    // the slab, and afterwards rank 0's S and T staging (2 x NBW x (NBW + 1))
    return std::max((size_t)slab * NBW, (size_t)2 * NBW * (NBW + 1)) * sizeof(T);
}
template <typename T, int NBW>
int launch_panel(T *wp, int64_t ld, int dv, int nbp, T *alphas, T *taus, T *v0s, Ctl<T> *ctl, int c0, T *tm,
                 T *vtv, cudaStream_t st) {
    if (dv <= panel_small_rows<T>()) {
        const size_t ssmem = (size_t)(2 * panel_small_rows<T>() + NBW * (dv | 1)) * sizeof(T);
        const int rpl = std::max(2, ((dv + 31) / 32 + 1) & ~1);   // register rows per lane, even
        auto sfn = qrb_panel_small<T, NBW, 16>;
        switch (rpl) {
            case 2: sfn = qrb_panel_small<T, NBW, 2>; break;
            case 4: sfn = qrb_panel_small<T, NBW, 4>; break;
            case 6: sfn = qrb_panel_small<T, NBW, 6>; break;
            case 8: sfn = qrb_panel_small<T, NBW, 8>; break;
            case 10: sfn = qrb_panel_small<T, NBW, 10>; break;
            case 12: sfn = qrb_panel_small<T, NBW, 12>; break;
            case 14: sfn = qrb_panel_small<T, NBW, sizeof(T) == 8 ? 12 : 14>; break;
            default: break;
        }
        SK_CUDA(cudaFuncSetAttribute((const void *)sfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssmem));
        sfn<<<1, QPS_THREADS, ssmem, st>>>(wp, ld, dv, nbp, alphas, taus, v0s, ctl, c0, tm);
        SK_LAUNCH_CHECK("qrb_panel_small");
        return SK_OK;
    }
    const int cl = panel_cl(dv);
    const int slab = (dv + cl - 1) / cl;
    const size_t psmem = panel_smem<T, NBW>(dv);
    auto pfn = cl == 1 ? qrb_panel_cluster<T, NBW, 1> : qrb_panel_cluster<T, NBW, QPC_CL>;
    SK_CUDA(cudaFuncSetAttribute((const void *)pfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psmem));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cl);
    cfg.blockDim = dim3(QPC_THREADS);
    cfg.dynamicSmemBytes = psmem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cl;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    SK_CUDA(cudaLaunchKernelEx(&cfg, pfn, wp, ld, dv, nbp, slab, alphas, taus, v0s, ctl, c0, tm, vtv));
    SK_LAUNCH_CHECK("qrb_panel_cluster");
    return SK_OK;
}

// V (dv x nbp, column-major, ld dv): zeros above the diagonal, v0 on it, the compact
// reflector storage of the panel below it
template <typename T>
__global__ void qrb_make_v(const T *wp, int64_t ld, int dv, int nbp, const T *v0s, T *v) {
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < (int64_t)dv * nbp;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int k = (int)(idx / dv), r = (int)(idx % dv);
        v[idx] = r < k ? LevelOps<T>::zero() : (r == k ? v0s[k] : wp[(int64_t)k * ld + r]);
    }
}

// C (nbp x nc, ld nbp) = X^T Y over dv rows; X: dv x nbp (ld ldx), Y: dv x nc (ld ldy).
// CTA: all nbp (<= 64) rows of C x 32 columns; thread (c = tid % 32, kq = tid / 32): 8 k.
// Split over rows: gridDim.y slabs of rows, slab z writes its partial C to c + z * pstride;
// qrb_reduce sums the partials in slab order (deterministic).
template <typename T>
__global__ void __launch_bounds__(256) qrb_gemm_tn(const T *x, int64_t ldx, const T *y, int64_t ldy, int dv, int nbp,
                                                   int nc, T *c, int64_t ldc, int64_t pstride) {
    __shared__ T xs[32][NBQ + 1];
    __shared__ T ys[32][33];
    const int tid = threadIdx.x, cc = tid & 31, kq = tid >> 5;
    const int c0 = blockIdx.x * 32;
    const int rows_per = ((dv + gridDim.y - 1) / gridDim.y + 31) / 32 * 32;
    const int rb = blockIdx.y * rows_per, re = min(dv, rb + rows_per);
    c += (int64_t)blockIdx.y * pstride;
    T acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = LevelOps<T>::zero();
    for (int r0 = rb; r0 < re; r0 += 32) {
        for (int e = tid; e < 32 * NBQ; e += 256) {
            const int rr = e & 31, k = e >> 5;
            xs[rr][k] = (r0 + rr < re && k < nbp) ? x[(int64_t)k * ldx + r0 + rr] : LevelOps<T>::zero();
        }
        for (int e = tid; e < 32 * 32; e += 256) {
            const int rr = e & 31, j = e >> 5;
            ys[rr][j] = (r0 + rr < re && c0 + j < nc) ? y[(int64_t)(c0 + j) * ldy + r0 + rr] : LevelOps<T>::zero();
        }
        __syncthreads();
#pragma unroll 8
        for (int rr = 0; rr < 32; ++rr) {
            const T yv = ys[rr][cc];
#pragma unroll
            for (int i = 0; i < 8; ++i) acc[i] = acc[i] + xs[rr][kq * 8 + i] * yv;
        }
        __syncthreads();
    }
    if (c0 + cc < nc)
#pragma unroll
        for (int i = 0; i < 8; ++i)
            if (kq * 8 + i < nbp) c[(int64_t)(c0 + cc) * ldc + kq * 8 + i] = acc[i];
}

template <typename T>
__global__ void qrb_reduce(const T *part, int64_t pstride, int nsplit, int64_t count, T *out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
        T s = part[i];
        for (int z = 1; z < nsplit; ++z) s = s + part[(int64_t)z * pstride + i];
        out[i] = s;
    }
}

// xLARFT (forward, columnwise): T upper nbp x nbp (column-major, ld NBQ) from V^T V and tau
template <typename T>
__global__ void qrb_larft(const T *vtv, const T *tau, int nbp, T *tm) {
    __shared__ T t[NBQ];
    const int i = threadIdx.x;
    for (int e = i; e < NBQ * NBQ; e += blockDim.x) tm[e] = LevelOps<T>::zero();
    __syncthreads();
    for (int j = 0; j < nbp; ++j) {
        if (i < j) t[i] = -tau[j] * vtv[(int64_t)j * nbp + i];    // -tau_j v_i . v_j
        __syncthreads();
        if (i < j) {
            T s = LevelOps<T>::zero();
            for (int k = i; k < j; ++k) s = s + tm[(int64_t)k * NBQ + i] * t[k];
            tm[(int64_t)j * NBQ + i] = s;
        }
        if (i == j) tm[(int64_t)j * NBQ + j] = tau[j];
        __syncthreads();
    }
}

// W (nbp x nc, ld nbp) = T^T G
template <typename T>
__global__ void qrb_tmul(const T *tm, const T *g, int nbp, int nc, T *wt) {
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < (int64_t)nbp * nc;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(idx % nbp), c = (int)(idx / nbp);
        T s = LevelOps<T>::zero();
        for (int k = 0; k <= i; ++k) s = s + tm[(int64_t)i * NBQ + k] * g[(int64_t)c * nbp + k];
        wt[idx] = s;
    }
}

// A_trail (dv x nc, ld) -= V (dv x nbp) W (nbp x nc); CTA: 32 rows x 32 columns,
// thread (row tid % 32, column group tid / 32 of 4)
template <typename T>
__global__ void __launch_bounds__(256) qrb_update(T *a, int64_t ld, const T *v, int dv, int nbp, const T *wt, int nc) {
    __shared__ T vs[NBQ][33];
    __shared__ T ws_[NBQ][33];
    const int tid = threadIdx.x, rr = tid & 31, cq = tid >> 5;
    const int r0 = blockIdx.x * 32, c0 = blockIdx.y * 32;
    for (int e = tid; e < 32 * NBQ; e += 256) {
        const int r = e & 31, k = e >> 5;
        vs[k][r] = (r0 + r < dv && k < nbp) ? v[(int64_t)k * dv + r0 + r] : LevelOps<T>::zero();
    }
    for (int e = tid; e < NBQ * 32; e += 256) {
        const int k = e & (NBQ - 1), j = e / NBQ;
        ws_[k][j] = (k < nbp && c0 + j < nc) ? wt[(int64_t)(c0 + j) * nbp + k] : LevelOps<T>::zero();
    }
    __syncthreads();
    T acc[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[i] = LevelOps<T>::zero();
    for (int k = 0; k < nbp; ++k) {
        const T vv = vs[k][rr];
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[i] = acc[i] + vv * ws_[k][cq * 4 + i];
    }
    if (r0 + rr < dv)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int c = c0 + cq * 4 + i;
            if (c < nc) a[(int64_t)c * ld + r0 + rr] = a[(int64_t)c * ld + r0 + rr] - acc[i];
        }
}


// Compact reflectors left behind by the dataflow kernels (taus[j], v0s[j] = v_j[0]),
// for forming Q afterwards.
template <typename T>
struct Reflectors {
    T *taus = nullptr, *v0s = nullptr;
};

template <typename T, bool HALF>
int run(T *w, int64_t d, int64_t n, double scale, double *r, int64_t ldr, sk_status *status, void *ws, size_t wsb,
        cudaStream_t st, Reflectors<T> *refl = nullptr, const double *scale_dev = nullptr) {
    DevStatus *defer = deferred_status();
    if (defer && refl) { set_error("sk_qr: deferred verdicts cover sk_qr_r only"); return SK_ERR_ARG; }
    if (wsb < ws_bytes<T>(d, n)) { set_error("sk_qr_r: workspace too small"); return SK_ERR_ARG; }
    if (nq_max(d) > MAXCH) { set_error("sk_qr_r: d too large"); return SK_ERR_ARG; }
    unsigned char *p = static_cast<unsigned char *>(ws);
    Ctl<T> *ctl = reinterpret_cast<Ctl<T> *>(p);
    p += align_up(sizeof(Ctl<T>), 256);
    T *alphas = reinterpret_cast<T *>(p);
    p += align_up((size_t)n * sizeof(T), 256);
    T *part = reinterpret_cast<T *>(p);
    p += align_up((size_t)nq_max(d) * n * sizeof(T), 256);
    int *nonfinite = reinterpret_cast<int *>(p);
    p += 256;
    T *taus = reinterpret_cast<T *>(p);
    p += align_up((size_t)n * sizeof(T), 256);
    T *v0s = reinterpret_cast<T *>(p);
    p += align_up((size_t)n * sizeof(T), 256);
    int *flags = reinterpret_cast<int *>(p);
    SK_CUDA(cudaMemsetAsync(ctl, 0, sizeof(Ctl<T>), st));
    SK_CUDA(cudaMemsetAsync(nonfinite, 0, sizeof(int), st));
    // A/B: the grid-barrier kernel (keeps only the current reflector, so never when Q is wanted)
    static const bool barrier_env = getenv("SK_QR_BARRIER") != nullptr;
    const bool barrier_kernel = barrier_env && refl == nullptr;
    if (refl) { refl->taus = taus; refl->v0s = v0s; }
    auto kfn = householder_kernel<T>;
    auto ffn = householder_flow_kernel<T, false>;
    const bool flow = !barrier_kernel;
    const int maxb = max_coop_blocks(flow ? (const void *)ffn : (const void *)kfn, THREADS, 0);
    if (maxb <= 0) { set_error("sk_qr_r: kernel cannot be co-resident"); return SK_ERR_ARG; }
    static const char *qr_smem_env = getenv("SK_QR_SMEM");
    const bool try_smem = flow && !(qr_smem_env && strcmp(qr_smem_env, "0") == 0);
    // one dataflow / barrier factorisation of the d_v x n_v view at wv (column stride d)
    auto launch_view = [&](T *wv, int dv_, int nv_, T *alv, T *tauv, T *v0v) -> int {
        const int64_t units = nq_max(dv_) * nv_;
        int blocks = (int)std::min<int64_t>(std::min<int64_t>(maxb, sm_count()), (units + WARPS - 1) / WARPS + 1);
        if (blocks < 2) blocks = std::min(2, maxb);
        int di = dv_, ni = nv_;
        int64_t ldw = d;
        // shared-memory-resident columns whenever they fit (SK_QR_SMEM=0 forces the global one)
        if (try_smem) {
            auto sfn = householder_flow_kernel<T, true>;
            const int gs = (int)std::min<int64_t>(sm_count(), nv_);
            const int64_t nloc = (nv_ + gs - 1) / gs;
            int optin = 0, dev = 0;
            cudaFuncAttributes fa{};
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
            const bool fa_ok = cudaFuncGetAttributes(&fa, (const void *)sfn) == cudaSuccess;
            // as many of each CTA's columns as fit (the later ones); SK_QR_SMEM=full: all or none
            const int64_t room = (int64_t)optin - (int64_t)fa.sharedSizeBytes - 1024 -
                                 (int64_t)(nloc * nq_max(dv_) * sizeof(T));
            const int64_t fit = room > 0 ? room / (int64_t)(dv_ * sizeof(T)) : 0;
            const bool whole_only = qr_smem_env && strcmp(qr_smem_env, "full") == 0;
            // partly resident only when at least half of a CTA's columns fit: binary32 at
            // 6144 x 2048 (9 of 14) 46.6 -> 42.3 ms; binary64 (4 of 14) measured slower
            int qs = (int)std::max<int64_t>(0, nloc - fit);
            if ((whole_only && qs > 0) || 2 * qs > nloc) qs = (int)nloc;
            const size_t smem = (size_t)((nloc - qs) * dv_ + nloc * nq_max(dv_)) * sizeof(T);
            if (gs >= 2 && fa_ok && qs < nloc && smem + fa.sharedSizeBytes + 1024 <= (size_t)optin &&
                cudaFuncSetAttribute((const void *)sfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) ==
                    cudaSuccess &&
                max_coop_blocks((const void *)sfn, THREADS, smem) >= gs) {
                SK_CUDA(cudaMemsetAsync(flags, 0, (size_t)nv_ * sizeof(int), st));
                void *args[] = {&wv, &ldw, &di, &ni, &alv, &part, &tauv, &v0v, &flags, &ctl, &qs};
                SK_CUDA(cudaLaunchCooperativeKernel((const void *)sfn, dim3(gs), dim3(THREADS), args, smem, st));
                SK_LAUNCH_CHECK("householder_flow_kernel (smem)");
                return SK_OK;
            }
            cudaGetLastError();   // a refused attribute / occupancy query falls back below
        }
        if (flow && (nv_ + blocks - 1) / blocks <= MAXCH) {
            SK_CUDA(cudaMemsetAsync(flags, 0, (size_t)nv_ * sizeof(int), st));
            int qs0 = 0;
            void *args[] = {&wv, &ldw, &di, &ni, &alv, &part, &tauv, &v0v, &flags, &ctl, &qs0};
            SK_CUDA(cudaLaunchCooperativeKernel((const void *)ffn, dim3(blocks), dim3(THREADS), args, 0, st));
            SK_LAUNCH_CHECK("householder_flow_kernel");
            return SK_OK;
        }
        if (refl) { set_error("sk_qr: Q needs the dataflow kernel (n too large)"); return SK_ERR_ARG; }
        void *args[] = {&wv, &ldw, &di, &ni, &alv, &part, &ctl};
        SK_CUDA(cudaLaunchCooperativeKernel((const void *)kfn, dim3(blocks), dim3(THREADS), args, 0, st));
        SK_LAUNCH_CHECK("householder_kernel");
        return SK_OK;
    };
    // binary32 / binary64 with more than one panel: blocked WY (SK_QR_BLOCKED=0: the
    // column-at-a-time dataflow kernel over the whole matrix)
    const char *blk_env = getenv("SK_QR_BLOCKED");
    // (with the dataflow kernel as the panel factorisation it measured binary64 75.2 ->
    // 66.3 ms, binary32 42.3 -> 46.8 ms at 6144 x 2048; the cluster panel kernel is the
    // default panel path, SK_QR_PANEL=flow the dataflow one)
    const bool want_blocked = !(blk_env && blk_env[0] == '0');
    const bool blocked = !HALF && flow && n > NBQ && d <= BLOCKED_MAX_D && want_blocked;
    if (!blocked) {
        const int rc0 = launch_view(w, (int)d, (int)n, alphas, taus, v0s);
        if (rc0 != SK_OK) return rc0;
    } else {
        unsigned char *q = reinterpret_cast<unsigned char *>(flags) + align_up((size_t)n * sizeof(int), 256);
        T *vb = reinterpret_cast<T *>(q);
        q += align_up((size_t)d * NBQ * sizeof(T), 256);
        T *vtv = reinterpret_cast<T *>(q);
        q += align_up((size_t)NBQ * NBQ * sizeof(T), 256);
        T *tm = reinterpret_cast<T *>(q);
        q += align_up((size_t)NBQ * NBQ * sizeof(T), 256);
        T *gm = reinterpret_cast<T *>(q);
        q += align_up((size_t)NBQ * n * sizeof(T), 256);
        T *wm = reinterpret_cast<T *>(q);
        q += align_up((size_t)NBQ * n * sizeof(T), 256);
        T *pm = reinterpret_cast<T *>(q);   // split partials
        const int sms_ = sm_count();
        // C (nbp x nc) = V^T Y over dv rows, split in row slabs so ~2 CTAs per SM work
        auto gemm_tn = [&](const T *yv, int64_t ldy, int dv_, int nbp_, int nc_, T *cout) {
            const int ncb = (nc_ + 31) / 32;
            const int ns = std::max(1, std::min(QRB_SPLIT_MAX, (2 * sms_ + ncb - 1) / ncb));
            const int64_t ps = (int64_t)nbp_ * nc_;
            qrb_gemm_tn<T><<<dim3((unsigned)ncb, (unsigned)ns), 256, 0, st>>>(vb, dv_, yv, ldy, dv_, nbp_, nc_, pm,
                                                                              nbp_, ps);
            qrb_reduce<T><<<(unsigned)std::min<int64_t>((ps + 255) / 256, 2048), 256, 0, st>>>(pm, ps, ns, ps, cout);
        };
        // panel width: 64 (binary32) / 32 (binary64) columns so that the panel fits the
        // shared memory of one 8-CTA cluster (slab x width x sizeof(T) <= 200 KB)
        constexpr int NBW = std::is_same<T, double>::value ? 32 : 64;
        const char *pc_env = getenv("SK_QR_PANEL");   // "flow": dataflow-kernel panels
        // the cluster panel kernel needs 8 co-scheduled CTAs with ~200 KB of shared memory
        // each (one GPC); where that cannot be scheduled the dataflow panels are used
        bool cluster_ok = !(pc_env && pc_env[0] == 'f');
        if (cluster_ok) {
            auto pfn0 = qrb_panel_cluster<T, std::is_same<T, double>::value ? 32 : 64, QPC_CL>;
            const size_t sm0 = 200 * 1024;   // the largest panel the per-panel check admits
            int nclusters = 0;
            cudaLaunchConfig_t qc = {};
            qc.gridDim = dim3(QPC_CL);
            qc.blockDim = dim3(QPC_THREADS);
            qc.dynamicSmemBytes = sm0;
            cudaLaunchAttribute qa[1];
            qa[0].id = cudaLaunchAttributeClusterDimension;
            qa[0].val.clusterDim.x = QPC_CL;
            qa[0].val.clusterDim.y = 1;
            qa[0].val.clusterDim.z = 1;
            qc.attrs = qa;
            qc.numAttrs = 1;
            if (cudaFuncSetAttribute((const void *)pfn0, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm0) !=
                    cudaSuccess ||
                cudaOccupancyMaxActiveClusters(&nclusters, (const void *)pfn0, &qc) != cudaSuccess || nclusters < 1) {
                cluster_ok = false;
                cudaGetLastError();
            }
        }
        static const bool qprof = getenv("SK_QR_PROF") != nullptr;   // panel / trailing split to stderr
        cudaEvent_t qe[3] = {nullptr, nullptr, nullptr};
        float t_panel = 0.f, t_trail = 0.f;
        if (qprof)
            for (auto &e : qe) cudaEventCreate(&e);
        // ---- lookahead pipeline (every panel on the cluster kernel): the main stream
        //      factors panel p+1 (after applying H_p to its columns) while a side stream
        //      applies H_p to the columns beyond it
        const char *la_env = getenv("SK_QR_LOOKAHEAD");
        const bool lookahead = cluster_ok && !qprof && !(la_env && la_env[0] == '0') &&
                               panel_smem<T, NBW>((int)d) <= 200 * 1024;
        if (lookahead) {
            // second buffer set right after the first (blocked_ws_bytes reserves both)
            unsigned char *q2 = reinterpret_cast<unsigned char *>(pm) +
                                align_up((size_t)QRB_SPLIT_MAX * NBQ * std::max<int64_t>(n, NBQ) * sizeof(T), 256);
            T *vb2 = reinterpret_cast<T *>(q2);
            q2 += align_up((size_t)d * NBQ * sizeof(T), 256);
            q2 += align_up((size_t)NBQ * NBQ * sizeof(T), 256);     // (second V^T V staging: unused)
            T *tm2 = reinterpret_cast<T *>(q2);
            q2 += align_up((size_t)NBQ * NBQ * sizeof(T), 256);
            T *gm2 = reinterpret_cast<T *>(q2);
            q2 += align_up((size_t)NBQ * n * sizeof(T), 256);
            T *wm2 = reinterpret_cast<T *>(q2);
            q2 += align_up((size_t)NBQ * n * sizeof(T), 256);
            T *pm2 = reinterpret_cast<T *>(q2);
            T *vbs[2] = {vb, vb2}, *tms[2] = {tm, tm2};
            int dev = 0;
            cudaGetDevice(&dev);
            static cudaStream_t side[64] = {};
            if (!side[dev]) SK_CUDA(cudaStreamCreateWithFlags(&side[dev], cudaStreamNonBlocking));
            cudaStream_t us = side[dev];
            const int np = (int)((n + NBW - 1) / NBW);
            std::vector<cudaEvent_t> ev_t(np), ev_u(np);
            for (int i = 0; i < np; ++i) {
                SK_CUDA(cudaEventCreateWithFlags(&ev_t[i], cudaEventDisableTiming));
                SK_CUDA(cudaEventCreateWithFlags(&ev_u[i], cudaEventDisableTiming));
            }
            SK_CUDA(cudaEventRecord(ev_u[0], st));     // placeholder order point for the side stream
            SK_CUDA(cudaStreamWaitEvent(us, ev_u[0], 0));
            // apply H (V: dvh x nbh at vbuf, T at tmat) to the dvh x nc block at a (ld d) on stream s
            auto apply = [&](cudaStream_t s, const T *vbuf, const T *tmat, int dvh, int nbh, T *a, int nc, T *g, T *w_,
                             T *pp) {
                const int ncb = (nc + 31) / 32;
                const int ns = std::max(1, std::min(QRB_SPLIT_MAX, (2 * sms_ + ncb - 1) / ncb));
                const int64_t ps = (int64_t)nbh * nc;
                qrb_gemm_tn<T><<<dim3((unsigned)ncb, (unsigned)ns), 256, 0, s>>>(vbuf, dvh, a, d, dvh, nbh, nc, pp, nbh,
                                                                                 ps);
                qrb_reduce<T><<<(unsigned)std::min<int64_t>((ps + 255) / 256, 2048), 256, 0, s>>>(pp, ps, ns, ps, g);
                qrb_tmul<T><<<(unsigned)std::min<int64_t>((ps + 255) / 256, 4096), 256, 0, s>>>(tmat, g, nbh, nc, w_);
                qrb_update<T><<<dim3((unsigned)((dvh + 31) / 32), (unsigned)ncb), 256, 0, s>>>(a, d, vbuf, dvh, nbh, w_,
                                                                                              nc);
            };
            for (int pi = 0; pi < np; ++pi) {
                const int64_t j0 = (int64_t)pi * NBW;
                const int nbp = (int)std::min<int64_t>(NBW, n - j0), dv = (int)(d - j0);
                T *wp = w + j0 * d + j0;
                if (pi >= 1) {
                    // H_{p-1} to this panel's columns, after the side stream applied H_{p-2} to them
                    if (pi >= 2) SK_CUDA(cudaStreamWaitEvent(st, ev_u[pi - 2], 0));
                    const int64_t jp = j0 - NBW;
                    apply(st, vbs[(pi - 1) & 1], tms[(pi - 1) & 1], (int)(d - jp), NBW, w + j0 * d + jp, nbp, gm, wm, pm);
                }
                const bool more = j0 + nbp < n;
                T *tmo = more ? tms[pi & 1] : nullptr;
                const int rcp = launch_panel<T, NBW>(wp, d, dv, nbp, alphas + j0, taus + j0, v0s + j0, ctl, (int)j0, tmo,
                                                     vtv, st);
                if (rcp) return rcp;
                if (!more) break;
                qrb_make_v<T><<<(unsigned)std::min<int64_t>(((int64_t)dv * nbp + 255) / 256, 4096), 256, 0, st>>>(
                    wp, d, dv, nbp, v0s + j0, vbs[pi & 1]);
                SK_CUDA(cudaEventRecord(ev_t[pi], st));
                // side stream: H_p to the columns beyond the next panel
                const int64_t cbeg = j0 + nbp + NBW;
                if (cbeg < n) {
                    SK_CUDA(cudaStreamWaitEvent(us, ev_t[pi], 0));
                    apply(us, vbs[pi & 1], tms[pi & 1], dv, nbp, w + cbeg * d + j0, (int)(n - cbeg), gm2, wm2, pm2);
                }
                SK_CUDA(cudaEventRecord(ev_u[pi], us));
            }
            SK_LAUNCH_CHECK("blocked QR lookahead");
            // join: the main stream waits for the side stream's last update
            cudaEvent_t done_ev;
            SK_CUDA(cudaEventCreateWithFlags(&done_ev, cudaEventDisableTiming));
            SK_CUDA(cudaEventRecord(done_ev, us));
            SK_CUDA(cudaStreamWaitEvent(st, done_ev, 0));
            SK_CUDA(cudaEventDestroy(done_ev));
            for (int i = 0; i < np; ++i) {
                cudaEventDestroy(ev_t[i]);
                cudaEventDestroy(ev_u[i]);
            }
        }
        bool have_t = false;
        for (int64_t j0 = 0; j0 < (lookahead ? 0 : n); j0 += NBW) {
            if (qprof) cudaEventRecord(qe[0], st);
            const int nbp = (int)std::min<int64_t>(NBW, n - j0), dv = (int)(d - j0);
            T *wp = w + j0 * d + j0;
            if (cluster_ok && panel_smem<T, NBW>(dv) <= 200 * 1024) {
                T *tmo = (j0 + nbp < n) ? tm : nullptr;   // T of the compact WY form, when a trailing update follows
                const int rcp = launch_panel<T, NBW>(wp, d, dv, nbp, alphas + j0, taus + j0, v0s + j0, ctl, (int)j0,
                                                     tmo, vtv, st);
                if (rcp) return rcp;
                have_t = true;
                // a collapse is recorded with its global column and checked once at the end
                // (the later panels then work on garbage that is never returned)
            } else {
                have_t = false;
                const int rc0 = launch_view(wp, dv, nbp, alphas + j0, taus + j0, v0s + j0);
                if (rc0 != SK_OK) return rc0;
                if (!defer) {   // deferred: the control record is read once, after the last panel
                    int fl[2];
                    SK_CUDA(cudaMemcpyAsync(fl, &ctl->fail_code, 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
                    SK_CUDA(cudaStreamSynchronize(st));
                    if (fl[0] != SK_OK) {
                        set_error("reflector %lld collapsed at working precision", (long long)(fl[1] + j0));
                        return fill_status(status, fl[0], (int)(fl[1] + j0), 0.0, 0.0);
                    }
                }
            }
            if (qprof) cudaEventRecord(qe[1], st);
            const int nc = (int)(n - j0 - nbp);
            if (nc <= 0) break;
            T *at = wp + (int64_t)nbp * d;   // trailing columns, rows j0..
            qrb_make_v<T><<<(unsigned)std::min<int64_t>(((int64_t)dv * nbp + 255) / 256, 4096), 256, 0, st>>>(
                wp, d, dv, nbp, v0s + j0, vb);
            if (!have_t) {   // the cluster kernel forms T itself
                gemm_tn(vb, dv, dv, nbp, nbp, vtv);
                qrb_larft<T><<<1, NBQ, 0, st>>>(vtv, taus + j0, nbp, tm);
            }
            gemm_tn(at, d, dv, nbp, nc, gm);
            qrb_tmul<T><<<(unsigned)std::min<int64_t>(((int64_t)nbp * nc + 255) / 256, 4096), 256, 0, st>>>(
                tm, gm, nbp, nc, wm);
            qrb_update<T><<<dim3((unsigned)((dv + 31) / 32), (unsigned)((nc + 31) / 32)), 256, 0, st>>>(at, d, vb, dv,
                                                                                                   nbp, wm, nc);
            SK_LAUNCH_CHECK("blocked QR trailing update");
            if (qprof) {
                cudaEventRecord(qe[2], st);
                cudaEventSynchronize(qe[2]);
                float a_ = 0.f, b_ = 0.f;
                cudaEventElapsedTime(&a_, qe[0], qe[1]);
                cudaEventElapsedTime(&b_, qe[1], qe[2]);
                t_panel += a_;
                t_trail += b_;
            }
        }
        if (qprof) {
            fprintf(stderr, "blocked qr d=%lld n=%lld T=%d: panels %.2f ms, trailing %.2f ms\n", (long long)d, (long long)n,
                    (int)sizeof(T), t_panel, t_trail);
            for (auto &e : qe) cudaEventDestroy(e);
        }
    }
    const int64_t total = n * n;
    if (defer) {   // record the collapse / the binary16 non-finite R on the device, no host read
        int rcn = note_verdict(&ctl->fail_code, 0, &ctl->fail_col, nullptr, nullptr, st);
        if (rcn) return rcn;
        extract_r<T><<<(unsigned)((total + 255) / 256), 256, 0, st>>>(w, d, alphas, (int)n, scale, r, ldr, nonfinite,
                                                                       scale_dev);
        SK_LAUNCH_CHECK("extract_r");
        if (HALF && (rcn = note_verdict(nonfinite, SK_OVERFLOW, nullptr, nullptr, nullptr, st))) return rcn;
        return fill_status(status, SK_OK, -1, 0.0, 0.0);
    }
    int fail[2];
    SK_CUDA(cudaMemcpyAsync(fail, &ctl->fail_code, 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
    SK_CUDA(cudaStreamSynchronize(st));
    if (fail[0] != SK_OK) {
        set_error("reflector %d collapsed at working precision", fail[1]);
        return fill_status(status, fail[0], fail[1], 0.0, 0.0);
    }
    extract_r<T><<<(unsigned)((total + 255) / 256), 256, 0, st>>>(w, d, alphas, (int)n, scale, r, ldr, nonfinite,
                                                                   nullptr);
    SK_LAUNCH_CHECK("extract_r");
    int nf = 0;
    SK_CUDA(cudaMemcpyAsync(&nf, nonfinite, sizeof(int), cudaMemcpyDeviceToHost, st));
    SK_CUDA(cudaStreamSynchronize(st));
    if (HALF && nf) {
        set_error("binary16 computation produced non-finite values");
        return fill_status(status, SK_OVERFLOW, -1, 0.0, 0.0);
    }
    return fill_status(status, SK_OK, -1, 0.0, 0.0);
}


// ------------------------------------------------ full factors (public API) --
// qr_in_precision / householder_reduce / accumulate_thin_q of the reference
// (src/precision.py:153-202, src/dense.py:108-172): the level QR from an f64 input
// (demotion and the binary16 power-of-two prescale on the f64 values, exactly as
// the reference orders them) plus, on request, the thin Q accumulated backward from
// the compact reflectors in the level arithmetic.

__global__ void maxabs_f64(const double *a, int64_t lda, int64_t rows, int64_t cols, unsigned long long *out_bits) {
    double mx = 0.0;
    const int64_t count = rows * cols;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
        mx = fmax(mx, fabs(a[(i / cols) * lda + i % cols]));
    mx = warp_max(mx);
    if ((threadIdx.x & 31) == 0) atomicMax(out_bits, (unsigned long long)__double_as_longlong(mx));
}

// w (column-major, ld = d) = level(a * scale): round_to_precision src/precision.py:90-103
// (one correctly rounded conversion from f64; `scale` is a power of two, so a * scale is
// exact); *overflow counts entries that became infinite from finite input
template <typename T>
__global__ void demote_colmajor(const double *a, int64_t lda, int64_t d, int64_t n, double scale, T *w,
                                int *overflow) {
    __shared__ double tile[32][33];
    const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // 32 x 8 threads
    for (int k = ty; k < 32; k += 8) {
        const int64_t r = r0 + k, c = c0 + tx;
        tile[k][tx] = (r < d && c < n) ? a[r * lda + c] : 0.0;
    }
    __syncthreads();
    int bad = 0;
    for (int k = ty; k < 32; k += 8) {
        const int64_t c = c0 + k, r = r0 + tx;
        if (r < d && c < n) {
            const double x = tile[tx][k];
            const T y = LevelOps<T>::from_f64(x * scale);
            bad |= (!LevelOps<T>::finite(y) && isfinite(x));
            w[c * d + r] = y;
        }
    }
    if (bad) atomicAdd(overflow, 1);
}

// compact reflector v_j = [v0_j, w[j+1:, j]]: put v0_j on the diagonal so every column
// holds its whole reflector
template <typename T>
__global__ void put_v0(T *w, int64_t ld, const T *v0s, int n) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j < n) w[(int64_t)j * ld + j] = v0s[j];
}

// accumulate_thin_q src/dense.py:164-172: Q = H_0 ... H_{n-1} eye(m, n), reflectors applied
// backward, each as t = tau_j * tree(v_j o Q[j:, c]) and Q[j:, c] -= v_j t (every product,
// sum and difference rounded in T; the tree is the pairwise one of src/precision.py:106-115).
// Columns are independent: one CTA per column.  Reflectors j > c leave column c exactly
// zero below row c (0 - v 0 = +0 for either sign of the product), so they are skipped.
template <typename T>
__global__ void __launch_bounds__(512)
accum_q_kernel(const T *v, int64_t ldv, const T *taus, int m, int n, T *q, int64_t ldq) {
    using O = LevelOps<T>;
    __shared__ T sh_nodes[MAXCH];
    __shared__ T sh_t;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int c = blockIdx.x; c < n; c += gridDim.x) {
        T *qc = q + (int64_t)c * ldq;
        for (int i = threadIdx.x; i < m; i += blockDim.x) qc[i] = (i == c) ? O::from_f64(1.0) : O::zero();
        __syncthreads();
        for (int j = c; j >= 0; --j) {
            const int L = m - j;
            const T *vj = v + (int64_t)j * ldv + j;
            T *x = qc + j;
            const int nq = (L + CH - 1) / CH;
            for (int qq = warp; qq < nq; qq += nw) {
                const T node = chunk_node<T>(vj, x, L, qq);
                if (lane == 0) sh_nodes[qq] = node;
            }
            __syncthreads();
            if (warp == 0) {
                const T root = warp_tree_root<T>(nq, [&](int i) { return sh_nodes[i]; });
                if (lane == 0) sh_t = O::mul(taus[j], root);
            }
            __syncthreads();
            const T t = sh_t;
            for (int i = threadIdx.x; i < L; i += blockDim.x) x[i] = O::sub(x[i], O::mul(vj[i], t));
            __syncthreads();
        }
    }
}

// column-major level-dtype d x n -> row-major f64 (exact promotion); counts non-finite
template <typename T>
__global__ void colmajor_to_f64(const T *src, int64_t lds, int64_t d, int64_t n, double *dst, int64_t ldd,
                                int lower_only, int *nonfinite) {
    __shared__ double tile[32][33];
    const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    int bad = 0;
    for (int k = ty; k < 32; k += 8) {
        const int64_t c = c0 + k, r = r0 + tx;
        double x = 0.0;
        if (r < d && c < n && (!lower_only || r >= c)) {
            x = LevelOps<T>::to_f64(src[c * lds + r]);
            bad |= !isfinite(x);
        }
        tile[tx][k] = x;
    }
    __syncthreads();
    for (int k = ty; k < 32; k += 8) {
        const int64_t r = r0 + k, c = c0 + tx;
        if (r < d && c < n) dst[r * ldd + c] = tile[k][tx];
    }
    if (bad && nonfinite) atomicAdd(nonfinite, 1);
}

template <typename T>
__global__ void vec_to_f64(const T *src, int n, double *dst) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j < n) dst[j] = LevelOps<T>::to_f64(src[j]);
}

template <typename T>
size_t factor_ws(int64_t d, int64_t n) {
    const size_t mat = align_up((size_t)d * n * sizeof(T), 256);
    return mat + ws_bytes<T>(d, n) + mat + 1024;
}

template <typename T, bool HALF>
int factor(const double *a, int64_t lda, int64_t d, int64_t n, double *r, int64_t ldr, double *q, int64_t ldq,
           double *v, int64_t ldv, double *taus_out, sk_status *status, void *ws, size_t wsb, cudaStream_t st) {
    if (wsb < factor_ws<T>(d, n)) { set_error("sk_qr: workspace too small"); return SK_ERR_ARG; }
    unsigned char *p = static_cast<unsigned char *>(ws);
    const size_t mat = align_up((size_t)d * n * sizeof(T), 256);
    T *w = reinterpret_cast<T *>(p);
    void *qws = p + mat;
    T *qb = reinterpret_cast<T *>(p + mat + ws_bytes<T>(d, n));
    int *flags = reinterpret_cast<int *>(p + 2 * mat + ws_bytes<T>(d, n));   // [0] overflow/non-finite [1..2] max bits
    SK_CUDA(cudaMemsetAsync(flags, 0, 64, st));
    double scale = 1.0;
    if (HALF) {   // src/precision.py:188-194: maxabs and the power-of-two scale on the f64 input
        unsigned long long *bits = reinterpret_cast<unsigned long long *>(flags + 2);
        const unsigned g = (unsigned)std::min<int64_t>((d * n + 255) / 256, 4 * sm_count());
        maxabs_f64<<<g, 256, 0, st>>>(a, lda, d, n, bits);
        SK_LAUNCH_CHECK("maxabs_f64");
        unsigned long long hb = 0;
        SK_CUDA(cudaMemcpyAsync(&hb, bits, sizeof(hb), cudaMemcpyDeviceToHost, st));
        SK_CUDA(cudaStreamSynchronize(st));
        double maxabs;
        memcpy(&maxabs, &hb, sizeof(double));
        if (maxabs == 0.0) {
            set_error("zero matrix");
            return fill_status(status, SK_RANK_DEFICIENT, -1, 0.0, 0.0);
        }
        int e = 0;
        frexp(maxabs, &e);
        scale = ldexp(1.0, -e);
    }
    const dim3 tg((unsigned)((n + 31) / 32), (unsigned)((d + 31) / 32));
    demote_colmajor<T><<<tg, 256, 0, st>>>(a, lda, d, n, scale, w, flags);
    SK_LAUNCH_CHECK("demote_colmajor");
    if (std::is_same<T, float>::value) {   // src/precision.py:181-184
        int ov = 0;
        SK_CUDA(cudaMemcpyAsync(&ov, flags, sizeof(int), cudaMemcpyDeviceToHost, st));
        SK_CUDA(cudaStreamSynchronize(st));
        if (ov) {
            set_error("input exceeds the binary32 range");
            return fill_status(status, SK_OVERFLOW, -1, 0.0, 0.0);
        }
    }
    Reflectors<T> refl;
    const bool need_refl = q || v || taus_out;
    const int rc = run<T, HALF>(w, d, n, scale, r, ldr, status, qws, ws_bytes<T>(d, n), st, need_refl ? &refl : nullptr);
    if (rc != SK_OK || !need_refl) return rc;
    put_v0<T><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(w, d, refl.v0s, (int)n);
    SK_LAUNCH_CHECK("put_v0");
    if (v) {
        colmajor_to_f64<T><<<tg, 256, 0, st>>>(w, d, d, n, v, ldv, 1, nullptr);
        SK_LAUNCH_CHECK("reflectors_to_f64");
    }
    if (taus_out) {
        vec_to_f64<T><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(refl.taus, (int)n, taus_out);
        SK_LAUNCH_CHECK("taus_to_f64");
    }
    if (!q) return SK_OK;
    const unsigned qg = (unsigned)std::min<int64_t>(n, 8 * (int64_t)sm_count());
    accum_q_kernel<T><<<qg, 512, 0, st>>>(w, d, refl.taus, (int)d, (int)n, qb, d);
    SK_LAUNCH_CHECK("accum_q_kernel");
    SK_CUDA(cudaMemsetAsync(flags, 0, sizeof(int), st));
    colmajor_to_f64<T><<<tg, 256, 0, st>>>(qb, d, d, n, q, ldq, 0, flags);
    SK_LAUNCH_CHECK("q_to_f64");
    if (HALF) {   // src/precision.py:200-201
        int nf = 0;
        SK_CUDA(cudaMemcpyAsync(&nf, flags, sizeof(int), cudaMemcpyDeviceToHost, st));
        SK_CUDA(cudaStreamSynchronize(st));
        if (nf) {
            set_error("binary16 computation produced non-finite values");
            return fill_status(status, SK_OVERFLOW, -1, 0.0, 0.0);
        }
    }
    return SK_OK;
}

}  // namespace qr
}  // namespace sk

using namespace sk;

extern "C" {

size_t sk_qr_workspace(int level, int64_t d, int64_t n) {
    if (level == 16) return qr::ws_bytes<__half>(d, n) + 256;
    if (level == 32) return qr::ws_bytes<float>(d, n);
    return qr::ws_bytes<double>(d, n);
}

int sk_qr_r(int level, void *a_s, int64_t d, int64_t n, double *r, int64_t ldr, sk_status *status, void *ws,
            size_t ws_bytes, sk_stream_t stream) {
    if (!a_s || !r || !ws || n <= 0 || d < n || ldr < n || qr::nq_max(d) > qr::MAXCH) {
        if (d < n && n > 0) {
            set_error("need rows >= cols, got %lld x %lld", (long long)d, (long long)n);
            return fill_status(status, SK_DIMENSION_MISMATCH, -1, 0, 0);
        }
        set_error("sk_qr_r: bad arguments");
        return SK_ERR_ARG;
    }
    cudaStream_t st = (cudaStream_t)stream;
    if (level == 64) return qr::run<double, false>(static_cast<double *>(a_s), d, n, 1.0, r, ldr, status, ws, ws_bytes, st);
    if (level == 32) return qr::run<float, false>(static_cast<float *>(a_s), d, n, 1.0, r, ldr, status, ws, ws_bytes, st);
    if (level != 16) { set_error("bad level"); return SK_ERR_ARG; }
    // binary16: exact power-of-two prescale (src/precision.py:188-194)
    __half *a = static_cast<__half *>(a_s);
    const int64_t count = d * n;
    unsigned long long *bits = reinterpret_cast<unsigned long long *>(static_cast<unsigned char *>(ws) +
                                                                      qr::ws_bytes<__half>(d, n));
    SK_CUDA(cudaMemsetAsync(bits, 0, sizeof(unsigned long long), st));
    const unsigned g = (unsigned)std::min<int64_t>((count + 255) / 256, 4 * sm_count());
    qr::maxabs_half<<<g, 256, 0, st>>>(a, count, bits);
    SK_LAUNCH_CHECK("maxabs_half");
    if (DevStatus *defer = deferred_status()) {   // the scale stays on the device
        double *scale_dev = reinterpret_cast<double *>(bits + 1);
        qr::half_scale_from_bits<<<1, 1, 0, st>>>(bits, scale_dev, defer);
        SK_LAUNCH_CHECK("half_scale_from_bits");
        qr::prescale_half<<<g, 256, 0, st>>>(a, count, 1.0, scale_dev);
        SK_LAUNCH_CHECK("prescale_half");
        return qr::run<__half, true>(a, d, n, 1.0, r, ldr, status, ws, ws_bytes, st, nullptr, scale_dev);
    }
    unsigned long long hb = 0;
    SK_CUDA(cudaMemcpyAsync(&hb, bits, sizeof(hb), cudaMemcpyDeviceToHost, st));
    SK_CUDA(cudaStreamSynchronize(st));
    double maxabs;
    memcpy(&maxabs, &hb, sizeof(double));
    if (maxabs == 0.0) {
        set_error("zero matrix");
        return fill_status(status, SK_RANK_DEFICIENT, -1, 0.0, 0.0);
    }
    int e = 0;
    frexp(maxabs, &e);
    const double scale = ldexp(1.0, -e);
    qr::prescale_half<<<g, 256, 0, st>>>(a, count, scale, nullptr);
    SK_LAUNCH_CHECK("prescale_half");
    return qr::run<__half, true>(a, d, n, scale, r, ldr, status, ws, ws_bytes, st);
}

size_t sk_qr_factors_workspace(int level, int64_t d, int64_t n) {
    if (level == 16) return qr::factor_ws<__half>(d, n) + 256;
    if (level == 32) return qr::factor_ws<float>(d, n);
    return qr::factor_ws<double>(d, n);
}

static int qr_factor_args(const double *a, int64_t lda, int64_t d, int64_t n, const double *r, int64_t ldr,
                          sk_status *status, void *ws) {
    if (n > 0 && d < n) {
        set_error("need rows >= cols, got %lld x %lld", (long long)d, (long long)n);
        return fill_status(status, SK_DIMENSION_MISMATCH, -1, 0, 0);
    }
    if (!a || !r || !ws || n <= 0 || lda < n || ldr < n || qr::nq_max(d) > qr::MAXCH || d > INT32_MAX) {
        set_error("sk_qr: bad arguments (d must be <= %d)", qr::MAXCH * qr::CH);
        return SK_ERR_ARG;
    }
    return SK_OK;
}

int sk_qr_in_precision_f64(int level, const double *a, int64_t lda, int64_t d, int64_t n, double *r, int64_t ldr,
                           double *q, int64_t ldq, sk_status *status, void *ws, size_t ws_bytes, sk_stream_t stream) {
    SK_NO_DEFER("sk_qr_in_precision_f64");
    const int rc = qr_factor_args(a, lda, d, n, r, ldr, status, ws);
    if (rc) return rc;
    if (q && ldq < n) { set_error("sk_qr_in_precision_f64: ldq < n"); return SK_ERR_ARG; }
    cudaStream_t st = (cudaStream_t)stream;
    if (level == 16)
        return qr::factor<__half, true>(a, lda, d, n, r, ldr, q, ldq, nullptr, 0, nullptr, status, ws, ws_bytes, st);
    if (level == 32)
        return qr::factor<float, false>(a, lda, d, n, r, ldr, q, ldq, nullptr, 0, nullptr, status, ws, ws_bytes, st);
    if (level == 64)
        return qr::factor<double, false>(a, lda, d, n, r, ldr, q, ldq, nullptr, 0, nullptr, status, ws, ws_bytes, st);
    set_error("bad level");
    return SK_ERR_ARG;
}

int sk_householder_f64(const double *a, int64_t lda, int64_t m, int64_t n, double *r, int64_t ldr, double *v,
                       int64_t ldv, double *taus, sk_status *status, void *ws, size_t ws_bytes, sk_stream_t stream) {
    SK_NO_DEFER("sk_householder_f64");
    const int rc = qr_factor_args(a, lda, m, n, r, ldr, status, ws);
    if (rc) return rc;
    if (v && ldv < n) { set_error("sk_householder_f64: ldv < n"); return SK_ERR_ARG; }
    return qr::factor<double, false>(a, lda, m, n, r, ldr, nullptr, 0, v, ldv, taus, status, ws, ws_bytes,
                                     (cudaStream_t)stream);
}

int sk_accumulate_q(int level, const void *v, int64_t ldv, const void *taus, int64_t m, int64_t n, void *q,
                    int64_t ldq, sk_stream_t stream) {
    if (!v || !taus || !q || n <= 0 || m < n || ldv < m || ldq < m || qr::nq_max(m) > qr::MAXCH) {
        set_error("sk_accumulate_q: bad arguments");
        return SK_ERR_ARG;
    }
    cudaStream_t st = (cudaStream_t)stream;
    const unsigned qg = (unsigned)std::min<int64_t>(n, 8 * (int64_t)sm_count());
    if (level == 16)
        qr::accum_q_kernel<__half><<<qg, 512, 0, st>>>(static_cast<const __half *>(v), ldv,
                                                       static_cast<const __half *>(taus), (int)m, (int)n,
                                                       static_cast<__half *>(q), ldq);
    else if (level == 32)
        qr::accum_q_kernel<float><<<qg, 512, 0, st>>>(static_cast<const float *>(v), ldv,
                                                      static_cast<const float *>(taus), (int)m, (int)n,
                                                      static_cast<float *>(q), ldq);
    else if (level == 64)
        qr::accum_q_kernel<double><<<qg, 512, 0, st>>>(static_cast<const double *>(v), ldv,
                                                       static_cast<const double *>(taus), (int)m, (int)n,
                                                       static_cast<double *>(q), ldq);
    else { set_error("bad level"); return SK_ERR_ARG; }
    SK_LAUNCH_CHECK("accum_q_kernel");
    return SK_OK;
}

}  // extern "C"

