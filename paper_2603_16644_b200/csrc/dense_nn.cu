// n x n FP64 kernels: Cholesky solve, LU solve with partial pivoting, triangular
// solves, and the kappa0 condition estimate.  These run replicated on every GPU
// (the n x n systems are tiny next to the m x n passes) and are latency-bound, so
// they are cooperative persistent kernels with grid barriers (factorisations) or
// single-CTA kernels (substitution, Hager).
//
// Reference semantics kept exactly:
//  - cholesky_factor src/dense.py:289-311: factor (S + S^T)/2, pivot must be > 0
//    and finite, else NotPositiveDefinite.  cholesky_solve :314-342 gates on
//    max|S - S^T| <= 10 eps max|S| (ValueError otherwise).
//  - lu_solve src/dense.py:245-286: partial pivoting, largest magnitude with the
//    LOWEST index on ties, threshold n*eps*max|G|, row swaps, multipliers
//    l = a_ik / a_kk then a_ij -= l * u_kj as a rounded product and a rounded
//    subtraction (np.outer then -=): the factorisation is op-for-op the reference's.
//  - triangular_solve src/dense.py:204-242: SingularTriangular on an exactly zero
//    diagonal; x_i = (b_i - sum) / r_ii.
//  - estimate_log10_condition src/precision.py:205-251 and Hager
//    src/dense.py:451-480 (x0 = 1/n, <= 5 iterations, lowest-index argmax,
//    stop when |z_j| <= z.x).
#include <cmath>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace sk {
namespace nxn {

constexpr int THREADS = 256;

// ------------------------------------------------------------ reductions ----
// out[0] = max|a_ij|, out[1] = max|a_ij - a_ji|, out[2] = #non-finite,
// out[3] = max_j sum_i |a_ij| (1-norm; columns)   (row-major input)
__global__ void sym_stats(const double *a, int n, double *out) {
    double mx = 0, dev = 0, nf = 0;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < (int64_t)n * n;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(idx / n), j = (int)(idx % n);
        const double v = a[idx];
        if (!isfinite(v)) nf += 1;
        mx = fmax(mx, fabs(v));
        dev = fmax(dev, fabs(v - a[(int64_t)j * n + i]));
    }
    mx = warp_max(mx);
    dev = warp_max(dev);
    nf = warp_sum(nf);
    if ((threadIdx.x & 31) == 0) {
        atomicMax(reinterpret_cast<unsigned long long *>(out), (unsigned long long)__double_as_longlong(mx));
        atomicMax(reinterpret_cast<unsigned long long *>(out + 1), (unsigned long long)__double_as_longlong(dev));
        atomicAdd(out + 2, nf);
    }
}
// deferred verdicts: the host gates of the LU / Cholesky solves on the device.
// lu != nullptr: non-finite -> SK_NON_FINITE, pivot threshold n eps max|a| into the LU
// control; else the Cholesky gates (non-finite, asymmetry > 10 eps max|s|)
__global__ void nxn_gate(const double *stats, int n, void *lu_ctl, DevStatus *ds) {
    const double mx = stats[0], dev = stats[1], nf = stats[2];
    int code = 0;
    if (nf > 0) code = SK_NON_FINITE;
    else if (!lu_ctl && dev > 10.0 * 2.220446049250313e-16 * mx) code = SK_NOT_SYMMETRIC;
    if (lu_ctl) reinterpret_cast<double *>(lu_ctl)[2] = (double)n * 2.220446049250313e-16 * mx;   // LuCtl::thresh
    if (code && ds->code == 0) { ds->code = code; ds->index = -1; ds->value = dev; ds->aux = mx; }
}
__global__ void trace_kernel(const double *a, int n, double *out) {
    double s = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) s += a[(int64_t)i * n + i];
    s = warp_sum(s);
    __shared__ double sh[32];
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t += sh[k];
        *out = t;
    }
}

__global__ void col_abs_sums(const double *a, int n, double *colsum) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    double s = 0;
    for (int i = 0; i < n; ++i) s += fabs(a[(int64_t)i * n + j]);
    colsum[j] = s;
}

// row-major g -> column-major w
__global__ void transpose_copy(const double *g, int n, double *w) {
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < (int64_t)n * n;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int j = (int)(idx / n), i = (int)(idx % n);
        w[idx] = g[(int64_t)i * n + j];
    }
}

// ------------------------------------------------------------- Cholesky -----
// W (col-major n x n) = (S + S^T)/2; L (col-major) receives the factor.
__global__ void symmetrize(const double *s, int n, double *w) {
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < (int64_t)n * n;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int j = (int)(idx / n), i = (int)(idx % n);   // w col-major: w[i + j n]
        w[idx] = (s[(int64_t)i * n + j] + s[(int64_t)j * n + i]) / 2.0;
    }
}

struct FactorCtl {
    int fail_code;
    int fail_col;
    double fail_value;
};

// Right-looking: at step j every thread computes d = sqrt(W_jj) (uniform verdict),
// writes L[:, j] = W[:, j] / d and updates the trailing lower triangle.  L is a
// separate array so W's column j is never overwritten while being read.
__global__ void __launch_bounds__(THREADS) chol_kernel(double *w, double *l, int n, FactorCtl *ctl) {
    cg::grid_group grid = cg::this_grid();
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
    for (int j = 0; j < n; ++j) {
        const double c0 = w[(int64_t)j * n + j];
        if (!(c0 > 0.0) || !isfinite(c0)) {
            if (tid == 0) { ctl->fail_code = SK_NOT_POSITIVE_DEFINITE; ctl->fail_col = j; ctl->fail_value = c0; }
            return;
        }
        const double d = sqrt(c0);
        const int rem = n - j - 1;
        // column j of L
        for (int64_t t = tid; t <= rem; t += nthreads) {
            const int i = j + (int)t;
            l[(int64_t)j * n + i] = (t == 0) ? d : w[(int64_t)j * n + i] / d;
        }
        // trailing lower triangle (i, k), j < k <= i: a thread keeps one row i
        // (consecutive threads -> consecutive i: coalesced) and strides over k
        if (rem > 0) {
            const int64_t groups = nthreads / rem > 0 ? nthreads / rem : 1;
            for (int64_t t = tid; t < groups * rem; t += nthreads) {
                const int i = j + 1 + (int)(t % rem);
                const int g0 = (int)(t / rem);
                const double li = w[(int64_t)j * n + i] / d;
                constexpr int U = 8;
                const int G = (int)groups;
                for (int kb = j + 1 + g0; kb <= i; kb += U * G) {
                    double wv[U], wk[U];
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const int k = kb + u * G;
                        if (k <= i) { wv[u] = w[(int64_t)k * n + i]; wk[u] = w[(int64_t)j * n + k]; }
                    }
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const int k = kb + u * G;
                        if (k <= i) w[(int64_t)k * n + i] = __dsub_rn(wv[u], __dmul_rn(li, wk[u] / d));
                    }
                }
            }
        }
        grid.sync();
    }
}

// Blocked right-looking Cholesky, in place on the lower triangle of W (col-major),
// panels of CB = 32 columns, three grid barriers per panel (64 panels at n = 2048
// instead of one barrier per column):
//   1. CTA 0 factors the 32 x 32 diagonal block in shared memory (pivot > 0 and
//      finite, else NotPositiveDefinite at that column)
//   2. every CTA solves its rows of the panel against the diagonal block
//   3. every CTA applies the rank-32 update to 32 x 32 tiles of the trailing lower
//      triangle
// Same quantities as the column algorithm, blocked summation order.
constexpr int CB = 32;

__global__ void __launch_bounds__(THREADS) chol_blocked_kernel(double *w, int n, FactorCtl *ctl) {
    cg::grid_group grid = cg::this_grid();
    __shared__ double dblk[CB][CB + 1];
    __shared__ double ti[CB][CB + 1], tk[CB][CB + 1];
    const int tid = threadIdx.x;
    for (int J = 0; J < n; J += CB) {
        const int jb = min(CB, n - J);
        // ---- 1. diagonal block
        if (blockIdx.x == 0) {
            for (int e = tid; e < CB * CB; e += blockDim.x) {
                const int i = e / CB, k = e % CB;
                dblk[i][k] = (i < jb && k < jb && k <= i) ? w[(int64_t)(J + k) * n + J + i] : 0.0;
            }
            __syncthreads();
            if (tid < 32) {
                const int lane = tid;
                int fail = -1;
                double fval = 0.0;
                for (int j = 0; j < jb; ++j) {
                    const double c0 = dblk[j][j];
                    if (!(c0 > 0.0) || !isfinite(c0)) { fail = j; fval = c0; break; }
                    const double d = sqrt(c0);
                    __syncwarp();
                    if (lane == 0) dblk[j][j] = d;
                    if (lane > j && lane < jb) dblk[lane][j] = dblk[lane][j] / d;
                    __syncwarp();
                    if (lane > j && lane < jb)
                        for (int k = j + 1; k <= lane; ++k)
                            dblk[lane][k] = __dsub_rn(dblk[lane][k], __dmul_rn(dblk[lane][j], dblk[k][j]));
                    __syncwarp();
                }
                if (lane == 0 && fail >= 0) {
                    ctl->fail_code = SK_NOT_POSITIVE_DEFINITE;
                    ctl->fail_col = J + fail;
                    ctl->fail_value = fval;
                }
            }
            __syncthreads();
            for (int e = tid; e < CB * CB; e += blockDim.x) {
                const int i = e / CB, k = e % CB;
                if (i < jb && k < jb && k <= i) w[(int64_t)(J + k) * n + J + i] = dblk[i][k];
            }
        }
        grid.sync();
        if (ctl->fail_code) return;
        // ---- 2. panel rows below the diagonal block: x = w_row * L_JJ^{-T}
        for (int e = tid; e < CB * CB; e += blockDim.x) {
            const int i = e / CB, k = e % CB;
            dblk[i][k] = (i < jb && k < jb && k <= i) ? w[(int64_t)(J + k) * n + J + i] : 0.0;
        }
        __syncthreads();
        for (int64_t r = J + jb + blockIdx.x * (int64_t)blockDim.x + tid; r < n; r += (int64_t)gridDim.x * blockDim.x) {
            double x[CB];
#pragma unroll
            for (int k = 0; k < CB; ++k) x[k] = (k < jb) ? w[(int64_t)(J + k) * n + r] : 0.0;
#pragma unroll
            for (int k = 0; k < CB; ++k) {
                if (k < jb) {
                    double s = x[k];
#pragma unroll
                    for (int l = 0; l < k; ++l) s = __dsub_rn(s, __dmul_rn(x[l], dblk[k][l]));
                    x[k] = s / dblk[k][k];
                }
            }
#pragma unroll
            for (int k = 0; k < CB; ++k)
                if (k < jb) w[(int64_t)(J + k) * n + r] = x[k];
        }
        grid.sync();
        // ---- 3. trailing update of the lower triangle, 32 x 32 tiles
        const int t0 = J + jb;
        const int nt = (n - t0 + CB - 1) / CB;
        const int ntri = nt * (nt + 1) / 2;
        for (int tix = blockIdx.x; tix < ntri; tix += gridDim.x) {
            int bi = (int)((sqrt(8.0 * tix + 1.0) - 1.0) * 0.5);
            while ((bi + 1) * (bi + 2) / 2 <= tix) ++bi;
            while (bi * (bi + 1) / 2 > tix) --bi;
            const int bk = tix - bi * (bi + 1) / 2;
            const int i0 = t0 + bi * CB, k0 = t0 + bk * CB;
            __syncthreads();
            for (int e = tid; e < CB * CB; e += blockDim.x) {
                const int rr = e % CB, l = e / CB;
                ti[rr][l] = (i0 + rr < n && l < jb) ? w[(int64_t)(J + l) * n + i0 + rr] : 0.0;
                tk[rr][l] = (k0 + rr < n && l < jb) ? w[(int64_t)(J + l) * n + k0 + rr] : 0.0;
            }
            __syncthreads();
            for (int e = tid; e < CB * CB; e += blockDim.x) {
                const int rr = e % CB, cc = e / CB;
                const int i = i0 + rr, k = k0 + cc;
                if (i < n && k < n && k <= i) {
                    double s = 0.0;
#pragma unroll 8
                    for (int l = 0; l < CB; ++l) s += ti[rr][l] * tk[cc][l];
                    double *p = w + (int64_t)k * n + i;
                    *p = *p - s;
                }
            }
        }
        grid.sync();
    }
}

__global__ void lower_to_l(const double *w, int n, double *l) {
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < (int64_t)n * n;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int k = (int)(idx / n), i = (int)(idx % n);   // col-major: l[i + k n]
        l[idx] = (i >= k) ? w[idx] : 0.0;
    }
}

// --------------------------------------------------------------------- LU ---
struct LuCtl {
    int fail_code;
    int fail_col;
    double fail_value;
    double thresh;
};

// candidate (value, index) per block, double-buffered by step parity
__device__ __forceinline__ void better(double &bv, int &bi, double v, int i) {
    if (v > bv || (v == bv && i < bi)) { bv = v; bi = i; }
}

__device__ void block_argmax(double v, int i, double *sv, int *si, double *outv, int *outi) {
    // lowest index wins ties; NaN never wins (reference np.argmax would pick NaN,
    // but a NaN pivot fails the threshold either way)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, v, o);
        const int oi = __shfl_xor_sync(0xffffffffu, i, o);
        better(v, i, ov, oi);
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) { sv[warp] = v; si[warp] = i; }
    __syncthreads();
    if (threadIdx.x == 0) {
        double bv = -1.0;
        int bi = INT32_MAX;
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) better(bv, bi, sv[k], si[k]);
        *outv = bv;
        *outi = bi;
    }
    __syncthreads();
}

// w: col-major n x n working copy (U in the upper part); lmul: col-major multipliers;
// perm: int permutation.  cand: 2 x gridDim.x (value, index) pairs.
__global__ void __launch_bounds__(THREADS)
lu_kernel(double *w, double *lmul, int *perm, int n, double *candv, int *candi, LuCtl *ctl) {
    __shared__ double sv[THREADS / 32];
    __shared__ int si[THREADS / 32];
    cg::grid_group grid = cg::this_grid();
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
    const double thresh = ctl->thresh;
    // candidates for column 0
    {
        double bv = -1.0;
        int bi = INT32_MAX;
        for (int64_t i = tid; i < n; i += nthreads) better(bv, bi, fabs(w[i]), (int)i);
        block_argmax(bv, bi, sv, si, &candv[blockIdx.x], &candi[blockIdx.x]);
    }
    for (int64_t i = tid; i < n; i += nthreads) perm[i] = (int)i;
    grid.sync();
    for (int k = 0; k < n; ++k) {
        const int buf = k & 1;
        // warp 0 of every block reduces the block candidates (the (value, lowest index)
        // order is total, so the result is deterministic) and broadcasts through smem
        __shared__ double s_piv;
        __shared__ int s_p;
        if (threadIdx.x < 32) {
            double bv = -1.0;
            int bi = INT32_MAX;
            for (int b = threadIdx.x; b < (int)gridDim.x; b += 32)
                better(bv, bi, candv[buf * gridDim.x + b], candi[buf * gridDim.x + b]);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
                const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                better(bv, bi, ov, oi);
            }
            if (threadIdx.x == 0) { s_piv = bv; s_p = bi; }
        }
        __syncthreads();
        const double piv = s_piv;
        const int p = s_p;
        __syncthreads();
        if (piv < thresh || piv == 0.0 || !(piv == piv)) {
            if (tid == 0) { ctl->fail_code = SK_NUMERICALLY_SINGULAR; ctl->fail_col = k; ctl->fail_value = piv; }
            return;
        }
        // swap rows k and p over all columns (one thread per column: no race)
        if (p != k) {
            for (int64_t j = tid; j < n; j += nthreads) {
                double *a = w + j * n;
                const double t = a[k];
                a[k] = a[p];
                a[p] = t;
                if (j < k) {   // multipliers of earlier steps move with their rows
                    double *lm = lmul + j * n;
                    const double u = lm[k];
                    lm[k] = lm[p];
                    lm[p] = u;
                }
            }
            if (tid == 0) { const int t = perm[k]; perm[k] = perm[p]; perm[p] = t; }
        }
        grid.sync();
        // multipliers and trailing update; candidates for column k+1 on the fly
        const double akk = w[(int64_t)k * n + k];
        const int rem = n - k - 1;
        double cbv = -1.0;
        int cbi = INT32_MAX;
        // a thread keeps one row i (one division per step) and strides over the
        // columns j = k..n-1; consecutive threads take consecutive rows (coalesced)
        if (rem > 0) {
            const int64_t groups = nthreads / rem > 0 ? nthreads / rem : 1;
            for (int64_t t = tid; t < groups * rem; t += nthreads) {
                const int i = k + 1 + (int)(t % rem);
                const int g0 = (int)(t / rem);
                const double li = __ddiv_rn(w[(int64_t)k * n + i], akk);
                if (g0 == 0) lmul[(int64_t)k * n + i] = li;
                // columns j = k+1+g0 + u*groups, 8 at a time: loads first (memory-level parallelism)
                constexpr int U = 8;
                const int G = (int)groups;
                for (int jb = k + 1 + g0; jb < n; jb += U * G) {
                    double wv[U], uk[U];
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const int j = jb + u * G;
                        if (j < n) { wv[u] = w[(int64_t)j * n + i]; uk[u] = w[(int64_t)j * n + k]; }
                    }
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const int j = jb + u * G;
                        if (j < n) {
                            const double nv = __dsub_rn(wv[u], __dmul_rn(li, uk[u]));
                            w[(int64_t)j * n + i] = nv;
                            if (j == k + 1) better(cbv, cbi, fabs(nv), i);
                        }
                    }
                }
            }
        }
        block_argmax(cbv, cbi, sv, si, &candv[(buf ^ 1) * gridDim.x + blockIdx.x], &candi[(buf ^ 1) * gridDim.x + blockIdx.x]);
        grid.sync();
    }
}

// LU with one grid barrier per step: rows are never swapped.  A row keeps its physical
// slot; pos[] (logical position of a physical row) and at[] (physical row at a logical
// position) record the swaps, double-buffered by step parity and rebuilt by all threads
// from (k, p, lp) so no thread races another.  Pivot ties resolve by logical position,
// as with physical swaps; every multiplier and update is the same rounded operation as
// lu_kernel's, so the factors agree bit for bit once gathered into logical order.
__device__ __forceinline__ void better3(double &bv, int &bl, int &br, double v, int l, int r) {
    if (v > bv || (v == bv && l < bl)) { bv = v; bl = l; br = r; }
}

__global__ void __launch_bounds__(THREADS)
lu_perm_kernel(double *w, double *lmul, int n, int *pos2, int *at2, double *candv, int *candl, int *candr,
               LuCtl *ctl) {
    __shared__ double sv[THREADS / 32];
    __shared__ int sl[THREADS / 32], sr[THREADS / 32];
    __shared__ double s_piv;
    __shared__ int s_lp, s_p;
    cg::grid_group grid = cg::this_grid();
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
    const int G = gridDim.x;
    const double thresh = ctl->thresh;
    auto block_cand = [&](double bv, int bl, int br, int slot) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
            const int ol = __shfl_xor_sync(0xffffffffu, bl, o), orr = __shfl_xor_sync(0xffffffffu, br, o);
            better3(bv, bl, br, ov, ol, orr);
        }
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        if (lane == 0) { sv[warp] = bv; sl[warp] = bl; sr[warp] = br; }
        __syncthreads();
        if (threadIdx.x == 0) {
            double v = -1.0;
            int l = INT32_MAX, r = INT32_MAX;
            for (int q = 0; q < THREADS / 32; ++q) better3(v, l, r, sv[q], sl[q], sr[q]);
            candv[slot * G + blockIdx.x] = v;
            candl[slot * G + blockIdx.x] = l;
            candr[slot * G + blockIdx.x] = r;
        }
        __syncthreads();
    };
    {
        double bv = -1.0;
        int bl = INT32_MAX, br = INT32_MAX;
        for (int64_t i = tid; i < n; i += nthreads) {
            better3(bv, bl, br, fabs(w[i]), (int)i, (int)i);
            pos2[i] = (int)i;
            at2[i] = (int)i;
        }
        block_cand(bv, bl, br, 0);
    }
    grid.sync();
    for (int k = 0; k < n; ++k) {
        const int buf = k & 1;
        const int *pos = pos2 + buf * n, *at = at2 + buf * n;
        int *npos = pos2 + (buf ^ 1) * n, *nat = at2 + (buf ^ 1) * n;
        if (threadIdx.x < 32) {
            double bv = -1.0;
            int bl = INT32_MAX, br = INT32_MAX;
            for (int b = threadIdx.x; b < G; b += 32)
                better3(bv, bl, br, candv[buf * G + b], candl[buf * G + b], candr[buf * G + b]);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
                const int ol = __shfl_xor_sync(0xffffffffu, bl, o), orr = __shfl_xor_sync(0xffffffffu, br, o);
                better3(bv, bl, br, ov, ol, orr);
            }
            if (threadIdx.x == 0) { s_piv = bv; s_lp = bl; s_p = br; }
        }
        __syncthreads();
        const double piv = s_piv;
        const int lp = s_lp, p = s_p;
        if (piv < thresh || piv == 0.0 || !(piv == piv)) {
            if (tid == 0) { ctl->fail_code = SK_NUMERICALLY_SINGULAR; ctl->fail_col = k; ctl->fail_value = piv; }
            return;
        }
        const int rk = at[k];                    // physical row at logical k before the swap
        // next-step maps: p -> k, rk -> lp
        for (int64_t i = tid; i < n; i += nthreads) {
            npos[i] = (i == p) ? k : (i == rk ? lp : pos[i]);
            nat[i] = (i == k) ? p : (i == lp ? rk : at[i]);
        }
        const double akk = w[(int64_t)k * n + p];
        double cbv = -1.0;
        int cbl = INT32_MAX, cbr = INT32_MAX;
        const int rem = n - k - 1;               // active rows other than p
        if (rem > 0) {
            // thread -> (active row, column group); active rows are those with pos >= k,
            // enumerated by logical position lpos in (k, n): physical row at[lpos], except
            // that logical k's row rk moved to lp (and p left the active set)
            const int64_t groups = nthreads / rem > 0 ? nthreads / rem : 1;
            for (int64_t t = tid; t < groups * rem; t += nthreads) {
                const int lpos = k + 1 + (int)(t % rem);
                const int i = (lpos == lp) ? rk : at[lpos];   // the row that ends up at lpos
                const int g0 = (int)(t / rem);
                const double li = __ddiv_rn(w[(int64_t)k * n + i], akk);
                if (g0 == 0) lmul[(int64_t)k * n + i] = li;
                constexpr int U = 8;
                const int GG = (int)groups;
                for (int jb = k + 1 + g0; jb < n; jb += U * GG) {
                    double wv[U], uk[U];
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const int j = jb + u * GG;
                        if (j < n) { wv[u] = w[(int64_t)j * n + i]; uk[u] = w[(int64_t)j * n + p]; }
                    }
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const int j = jb + u * GG;
                        if (j < n) {
                            const double nv = __dsub_rn(wv[u], __dmul_rn(li, uk[u]));
                            w[(int64_t)j * n + i] = nv;
                            if (j == k + 1) better3(cbv, cbl, cbr, fabs(nv), lpos, i);
                        }
                    }
                }
            }
        }
        block_cand(cbv, cbl, cbr, buf ^ 1);
        grid.sync();
    }
}

// gather the physically stored factors into logical row order (at = final at[] map)
__global__ void lu_gather(const double *w, const double *lmul, const int *at, int n, double *wl, double *ll,
                          int *perm) {
    const int64_t total = (int64_t)n * n;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int j = (int)(e / n), i = (int)(e % n);    // column-major: column j, logical row i
        const int r = at[i];
        wl[e] = w[(int64_t)j * n + r];
        ll[e] = (i > j) ? lmul[(int64_t)j * n + r] : 0.0;
        if (j == 0) perm[i] = r;
    }
}

// Dataflow LU (no grid barriers), the same arithmetic as lu_kernel: column c of the
// column-major working copy is owned by CTA c mod G and only its owner swaps/updates
// it.  Step k's pivot and multipliers come from the owner of column k right after it
// applied steps < k to that column (published through flags[k]: 1 = ok, 2 = singular);
// every CTA then applies step k to its own columns (the next pivot column first when it
// owns it) and swaps rows k, p of the multiplier columns it owns.
__global__ void __launch_bounds__(THREADS)
lu_flow_kernel(double *w, double *lmul, int *perm, int n, int *pivots, int *flags, LuCtl *ctl) {
    __shared__ double sv[THREADS / 32];
    __shared__ int si[THREADS / 32];
    __shared__ double s_piv;
    __shared__ int s_p, s_flag;
    const int G = gridDim.x, b = blockIdx.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = THREADS / 32;
    const double thresh = ctl->thresh;

    // pivot, swap and multipliers of step k on column k (owned by this CTA, up to date)
    auto pivot_step = [&](int k) {
        double *col = w + (int64_t)k * n;
        double bv = -1.0;
        int bi = INT32_MAX;
        for (int i = k + threadIdx.x; i < n; i += THREADS) better(bv, bi, fabs(col[i]), i);
        block_argmax(bv, bi, sv, si, &s_piv, &s_p);
        const double piv = s_piv;
        const int p = s_p;
        const bool bad = piv < thresh || piv == 0.0 || !(piv == piv);
        if (!bad) {
            if (threadIdx.x == 0 && p != k) {
                const double t = col[k];
                col[k] = col[p];
                col[p] = t;
            }
            __syncthreads();
            const double akk = col[k];
            for (int i = k + 1 + threadIdx.x; i < n; i += THREADS) lmul[(int64_t)k * n + i] = __ddiv_rn(col[i], akk);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            if (bad) { ctl->fail_code = SK_NUMERICALLY_SINGULAR; ctl->fail_col = k; ctl->fail_value = piv; }
            pivots[k] = p;
            __threadfence();
            atomicExch(flags + k, bad ? 2 : 1);
        }
    };
    // step k on column c: swap rows k, p, then rows i > k -= l_i * row k (one warp)
    auto apply_warp = [&](int k, int p, const double *l, int c) {
        double *col = w + (int64_t)c * n;
        if (lane == 0 && p != k) {
            const double t = col[k];
            col[k] = col[p];
            col[p] = t;
        }
        __syncwarp();
        const double ukc = col[k];
        for (int i = k + 1 + lane; i < n; i += 32) col[i] = __dsub_rn(col[i], __dmul_rn(l[i], ukc));
    };

    (void)perm;                                   // built from pivots afterwards (perm_from_pivots)
    if (b == 0) pivot_step(0);
    for (int k = 0; k < n - 1; ++k) {
        if (threadIdx.x == 0) s_flag = wait_flag(flags + k);
        __syncthreads();
        if (s_flag != 1) {
            if (s_flag < 0 && threadIdx.x == 0) { ctl->fail_code = SK_ERR_CUDA; ctl->fail_col = k; }
            return;
        }
        const int p = *reinterpret_cast<volatile int *>(pivots + k);
        const double *l = lmul + (int64_t)k * n;
        int c0 = k + 1 + ((b - (k + 1)) % G + G) % G;    // first owned column > k
        if (c0 == k + 1) {                                 // next pivot column first
            double *col = w + (int64_t)c0 * n;
            if (threadIdx.x == 0 && p != k) {
                const double t = col[k];
                col[k] = col[p];
                col[p] = t;
            }
            __syncthreads();
            const double ukc = col[k];
            for (int i = k + 1 + threadIdx.x; i < n; i += THREADS) col[i] = __dsub_rn(col[i], __dmul_rn(l[i], ukc));
            __syncthreads();
            pivot_step(k + 1);
            c0 += G;
        }
        int wi = 0;
        for (int c = c0; c < n; c += G, ++wi)
            if (wi % nw == warp) apply_warp(k, p, l, c);
        // multipliers of earlier steps move with their rows (owned L columns j < k)
        if (p != k)
            for (int j = b + threadIdx.x * G; j < k; j += THREADS * G) {
                double *lm = lmul + (int64_t)j * n;
                const double u = lm[k];
                lm[k] = lm[p];
                lm[p] = u;
            }
        __syncthreads();
    }
}

// Shared-memory-resident dataflow LU (n <= ~2070 on 148 SMs): CTA b keeps its columns
// c = b + q G (q < nloc) in shared memory for the whole factorisation, so a step touches
// no global memory but the published multiplier column.  Rows are swapped physically
// inside every CTA's own columns (finished L columns included, as src/dense.py:264-281
// swaps whole rows), so the logical order is the physical one and the pivot tie rule
// (first maximum, np.argmax) needs no position map.  The owner of column s publishes
// step s (pivot row, multipliers l = w[s+1:, s] / w[s, s]) through flags[s]; the owner
// of column k+1 applies step k to that column first, then publishes step k+1 before it
// updates its other columns (lookahead 1).  Every multiplier and update is the
// reference's separately rounded division, product and difference, as in lu_kernel.
constexpr int LUS_THREADS = 1024, LUS_ROWS = 2;   // rows per thread: n <= LUS_THREADS * LUS_ROWS

__device__ __forceinline__ int spin_flag(const int *flag) {
    int v;
    long long spins = 0;
    while ((v = *reinterpret_cast<const volatile int *>(flag)) == 0)
        if (++spins > (1ll << 27)) return -1;     // stuck chain: fail instead of hanging the GPU
    __threadfence();
    return v;
}

__global__ void __launch_bounds__(LUS_THREADS, 1)
lu_smem_kernel(double *w, int n, double *gl, int *piv, int *flags, double *lout, LuCtl *ctl) {
    extern __shared__ double W[];                 // nloc x n, column q = global column b + q G
    __shared__ double sv[LUS_THREADS / 32];
    __shared__ int si[LUS_THREADS / 32];
    __shared__ double s_piv;
    __shared__ int s_p, s_flag;
    const int G = gridDim.x, b = blockIdx.x, tid = threadIdx.x, T = blockDim.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int nloc = b < n ? (n - b + G - 1) / G : 0;
    const double thresh = ctl->thresh;
    for (int q = 0; q < nloc; ++q) {
        const double *src = w + (int64_t)(b + q * G) * n;
        for (int i = tid; i < n; i += T) W[q * n + i] = src[i];
    }
    __syncthreads();

    // pivot search, swap and multipliers of column s (owned; steps < s applied); false on failure
    auto lead = [&](int s) -> bool {
        double *col = W + (s / G) * n;
        double bv = -1.0;
        int bi = INT32_MAX;
        for (int i = s + tid; i < n; i += T) better(bv, bi, fabs(col[i]), i);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            better(bv, bi, ov, oi);
        }
        if (lane == 0) { sv[warp] = bv; si[warp] = bi; }
        __syncthreads();
        if (warp == 0) {
            bv = lane < T / 32 ? sv[lane] : -1.0;
            bi = lane < T / 32 ? si[lane] : INT32_MAX;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
                const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                better(bv, bi, ov, oi);
            }
            if (lane == 0) {
                s_piv = bv;
                s_p = bi;
                if (bi != s && bi < n) { const double t = col[s]; col[s] = col[bi]; col[bi] = t; }
            }
        }
        __syncthreads();
        const double pv = s_piv;
        if (pv < thresh || pv == 0.0 || !(pv == pv)) {
            if (tid == 0) {
                ctl->fail_code = SK_NUMERICALLY_SINGULAR;
                ctl->fail_col = s;
                ctl->fail_value = pv;
                __threadfence();
                atomicExch(flags + s, 2);
            }
            return false;
        }
        const double akk = col[s];
        double *g = gl + (int64_t)s * n;
        for (int i = s + 1 + tid; i < n; i += T) {
            const double li = __ddiv_rn(col[i], akk);
            col[i] = li;
            g[i] = li;
        }
        __threadfence();
        __syncthreads();
        if (tid == 0) {
            piv[s] = s_p;
            __threadfence();
            atomicExch(flags + s, 1);
        }
        return true;
    };

    if (b == 0 && n > 0 && !lead(0)) return;
    for (int k = 0; k < n; ++k) {
        if (tid == 0) s_flag = spin_flag(flags + k);
        __syncthreads();
        if (s_flag != 1) {
            if (s_flag < 0 && tid == 0) { ctl->fail_code = SK_ERR_CUDA; ctl->fail_col = k; }
            return;
        }
        const int p = __ldcg(piv + k);
        if (p != k)
            for (int q = tid; q < nloc; q += T)
                if (b + q * G != k) {
                    double *col = W + q * n;
                    const double t = col[k];
                    col[k] = col[p];
                    col[p] = t;
                }
        __syncthreads();
        if (k == n - 1) break;
        const double *g = gl + (int64_t)k * n;
        double l[LUS_ROWS];
#pragma unroll
        for (int r = 0; r < LUS_ROWS; ++r) {
            const int i = k + 1 + tid + r * T;
            l[r] = i < n ? __ldcg(g + i) : 0.0;
        }
        auto update = [&](int q) {
            double *col = W + q * n;
            const double u = col[k];
#pragma unroll
            for (int r = 0; r < LUS_ROWS; ++r) {
                const int i = k + 1 + tid + r * T;
                if (i < n) col[i] = __dsub_rn(col[i], __dmul_rn(l[r], u));
            }
        };
        int q0 = k >= b ? (k - b) / G + 1 : 0;       // first owned column > k
        if (q0 < nloc && b + q0 * G == k + 1) {
            update(q0);
            __syncthreads();
            if (!lead(k + 1)) return;
            ++q0;
        }
        for (int q = q0; q < nloc; ++q) update(q);
    }
    __syncthreads();
    for (int q = 0; q < nloc; ++q) {
        const int c = b + q * G;
        double *dw = w + (int64_t)c * n, *dl = lout + (int64_t)c * n;
        for (int i = tid; i < n; i += T) {
            const double v = W[q * n + i];
            dw[i] = v;
            dl[i] = i > c ? v : 0.0;
        }
    }
}

// Small n (n x n doubles fit one CTA's shared memory): the whole LU in ONE CTA, every
// step's element updates spread over all threads instead of one column per CTA.  The
// arithmetic is lu_smem_kernel's op for op (first-maximum pivot, __ddiv_rn multipliers,
// a - l * u rounded twice, whole-row swaps), so the factors are bitwise the same; what
// goes away is the inter-CTA flag chain (config 1, n = 100: ~3.8 us per step).
constexpr int LU_SMALL_MAX = 160;
__global__ void __launch_bounds__(512, 1)
lu_small_kernel(double *w, int n, int *piv, int *perm, double *lout, LuCtl *ctl) {
    extern __shared__ double W[];                 // column-major n x n
    __shared__ double s_pv, s_akk;
    __shared__ int s_p, s_piv[LU_SMALL_MAX], s_perm[LU_SMALL_MAX];
    const int tid = threadIdx.x, T = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = T >> 5;
    const double thresh = ctl->thresh;
    for (int64_t e = tid; e < (int64_t)n * n; e += T) W[e] = w[e];
    __syncthreads();
    // pivot of column k: first maximum of |A[k:, k]| (one warp), with its signed value
    auto pivot = [&](int k) {
        const double *ck = W + (int64_t)k * n;
        double bv = -1.0;
        int bi = INT32_MAX;
        for (int i = k + lane; i < n; i += 32) better(bv, bi, fabs(ck[i]), i);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            better(bv, bi, ov, oi);
        }
        if (lane == 0) { s_pv = bv; s_p = bi; s_akk = bi < n ? ck[bi] : 0.0; }
    };
    if (warp == 0) pivot(0);
    __syncthreads();
    // two barriers per step: (1) multipliers of column k (with its row swap folded in)
    // and the row swap of every other column; (2) the trailing update, where warp 0 takes
    // column k + 1 alone and then finds its pivot while the other warps update the rest
    for (int k = 0; k < n; ++k) {
        const double pv = s_pv, akk = s_akk;
        const int p = s_p;
        if (pv < thresh || pv == 0.0 || !(pv == pv)) {   // uniform
            if (tid == 0) { ctl->fail_code = SK_NUMERICALLY_SINGULAR; ctl->fail_col = k; ctl->fail_value = pv; }
            for (int i = tid; i < n; i += T) perm[i] = i;   // a valid permutation for deferred callers
            return;
        }
        double *ck = W + (int64_t)k * n;
        for (int i = k + tid; i < n; i += T) {
            if (i == k) {
                if (p != k) ck[p] = __ddiv_rn(ck[k], akk);   // old row k lands in row p
                ck[k] = akk;
            } else if (i != p) {
                ck[i] = __ddiv_rn(ck[i], akk);
            }
        }
        if (p != k)
            for (int j = tid; j < n; j += T) {
                if (j == k) continue;
                double *cj = W + (int64_t)j * n;
                const double t = cj[k];
                cj[k] = cj[p];
                cj[p] = t;
            }
        if (tid == 0) { piv[k] = p; s_piv[k] = p; }
        __syncthreads();
        if (warp == 0) {
            if (k + 1 < n) {
                double *cj = W + (int64_t)(k + 1) * n;
                const double u = cj[k];
                for (int i = k + 1 + lane; i < n; i += 32) cj[i] = __dsub_rn(cj[i], __dmul_rn(ck[i], u));
                __syncwarp();
                pivot(k + 1);
            }
        } else {
            for (int j = k + 2 + (warp - 1); j < n; j += nw - 1) {   // a warp per column
                double *cj = W + (int64_t)j * n;
                const double u = cj[k];
                for (int i = k + 1 + lane; i < n; i += 32) cj[i] = __dsub_rn(cj[i], __dmul_rn(ck[i], u));
            }
        }
        __syncthreads();
    }
    for (int i = tid; i < n; i += T) s_perm[i] = i;
    __syncthreads();
    if (tid == 0)   // perm = the row swaps (k, piv[k]) applied in order to the identity
        for (int k = 0; k < n; ++k) {
            const int q = s_piv[k];
            if (q != k) { const int t = s_perm[k]; s_perm[k] = s_perm[q]; s_perm[q] = t; }
        }
    __syncthreads();
    for (int i = tid; i < n; i += T) perm[i] = s_perm[i];
    for (int c = warp; c < n; c += nw)
        for (int i = lane; i < n; i += 32) {
            const double v = W[(int64_t)c * n + i];
            w[(int64_t)c * n + i] = v;
            lout[(int64_t)c * n + i] = i > c ? v : 0.0;
        }
}

// perm = the row swaps (k, pivots[k]) applied in order to the identity (one thread)
__global__ void perm_from_pivots(const int *pivots, int n, int *perm) {
    if (blockIdx.x != 0 || threadIdx.x != 0) return;
    for (int i = 0; i < n; ++i) perm[i] = i;
    for (int k = 0; k < n; ++k) {
        const int p = pivots[k];
        if (p != k && p >= 0 && p < n) {
            const int t = perm[k];
            perm[k] = perm[p];
            perm[p] = t;
        }
    }
}

// ------------------------------------------------------------ substitution --
// Single-CTA blocked triangular solve over an element accessor M(i,k) = m[i*rs + k*cs].
// lower: x_i depends on k < i (forward); else k > i (backward).  unit: diag == 1.
// x holds rhs on entry (in shared or global memory) and the solution on exit.
struct TriView {
    const double *m;
    int64_t rs, cs;
    __device__ __forceinline__ double operator()(int i, int k) const { return m[i * rs + k * cs]; }
};

__device__ void block_trsv(const TriView M, int n, bool lower, bool unit, double *x) {
    const int tid = threadIdx.x, nt = blockDim.x;
    const int warp = tid >> 5, lane = tid & 31, nw = nt >> 5;
    const int nb = (n + 31) / 32;
    __shared__ double dblk[32][33];   // the diagonal block, staged so the sequential
                                      // 32-step solve reads shared memory, not L2
    for (int bb = 0; bb < nb; ++bb) {
        const int b = lower ? bb : nb - 1 - bb;
        const int r0 = b * 32, r1 = min(n, r0 + 32);
        const int w = r1 - r0;
        for (int e = tid; e < 32 * 32; e += nt) {
            const int i = e >> 5, k = e & 31;
            dblk[i][k] = (i < w && k < w) ? M(r0 + i, r0 + k) : 0.0;
        }
        __syncthreads();
        if (warp == 0) {
            double v = (lane < w) ? x[r0 + lane] : 0.0;
            for (int s = 0; s < w; ++s) {
                const int r = lower ? s : w - 1 - s;
                double xr = 0.0;
                if (lane == r) { xr = unit ? v : v / dblk[r][r]; v = xr; }
                xr = __shfl_sync(0xffffffffu, xr, r);
                const bool dep = lower ? (lane > r) : (lane < r);
                if (dep && lane < w) v -= dblk[lane][r] * xr;
            }
            if (lane < w) x[r0 + lane] = v;
        }
        __syncthreads();
        // update the rows not yet solved: lower -> rows >= r1, upper -> rows < r0
        const int lo = lower ? r1 : 0, hi = lower ? n : r0;
        if (M.rs == 1) {   // column-major: thread per row, coalesced
            for (int i = lo + tid; i < hi; i += nt) {
                double s = 0.0;
                for (int k = r0; k < r1; ++k) s += M(i, k) * x[k];
                x[i] -= s;
            }
        } else {           // row-major: a warp takes 32 rows x the block's 32 columns
            // lanes read rows coalesced (lane = column); the 32 row sums come out of a
            // reduce-scatter butterfly (31 shuffles for 32 rows; lane r ends with row r)
            const double xl = (lane < w) ? x[r0 + lane] : 0.0;
            for (int i0 = lo + warp * 32; i0 < hi; i0 += nw * 32) {
                const int rows = min(32, hi - i0);
                double v[32];
#pragma unroll
                for (int rr = 0; rr < 32; ++rr) v[rr] = (rr < rows && lane < w) ? M(i0 + rr, r0 + lane) * xl : 0.0;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    const bool upper = (lane & o) != 0;
#pragma unroll
                    for (int j = 0; j < o; ++j) {
                        const double send = upper ? v[j] : v[j + o];
                        const double keep = upper ? v[j + o] : v[j];
                        v[j] = keep + __shfl_xor_sync(0xffffffffu, send, o);
                    }
                }
                if (lane < rows) x[i0 + lane] -= v[0];
            }
        }
        __syncthreads();
    }
}

constexpr int TRSV_THREADS = 512;   // 128 registers: the 32-row butterfly tile without spills
__global__ void __launch_bounds__(TRSV_THREADS) trsv_kernel(TriView M, int n, bool lower, bool unit, const double *rhs,
                                                    const int *perm, double *x) {
    extern __shared__ double xs[];
    for (int i = threadIdx.x; i < n; i += blockDim.x) xs[i] = perm ? rhs[perm[i]] : rhs[i];
    __syncthreads();
    block_trsv(M, n, lower, unit, xs);
    for (int i = threadIdx.x; i < n; i += blockDim.x) x[i] = xs[i];
}

__global__ void first_zero_diag(TriView M, int n, int *out) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        if (M(i, i) == 0.0) atomicMin(out, i);
}

// Hager on G^{-1} with G = L L^T (L col-major), all in one CTA.
// est_out = best (the estimate of ||G^{-1}||_1).
constexpr int HAGER_THREADS = 1024;   // measured faster than 512 despite a small spill
__global__ void __launch_bounds__(HAGER_THREADS) hager_kernel(const double *l, int n, double *est_out) {
    extern __shared__ double hs[];
    double *x = hs, *y = hs + n, *z = hs + 2 * n;
    __shared__ double red[32];
    __shared__ int redi[32];
    __shared__ int stop;
    const TriView Lv{l, 1, n};          // L(i,k) = l[i + k n]
    const TriView LTv{l, n, 1};         // L^T(i,k) = L(k,i) = l[k + i n]
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
    for (int i = tid; i < n; i += nt) x[i] = 1.0 / n;
    double best = 0.0;
    __syncthreads();
    for (int it = 0; it < 5; ++it) {
        // y = G^{-1} x : forward with L, backward with L^T
        for (int i = tid; i < n; i += nt) y[i] = x[i];
        __syncthreads();
        block_trsv(Lv, n, true, false, y);
        block_trsv(LTv, n, false, false, y);
        // ||y||_1
        double s = 0.0;
        for (int i = tid; i < n; i += nt) s += fabs(y[i]);
        s = warp_sum(s);
        if (lane == 0) red[warp] = s;
        __syncthreads();
        if (tid == 0) {
            double t = 0.0;
            for (int k = 0; k < nw; ++k) t += red[k];
            best = fmax(best, t);
            red[0] = best;
        }
        __syncthreads();
        best = red[0];
        __syncthreads();
        // z = G^{-T} sign(y)  (G symmetric: same solve)
        for (int i = tid; i < n; i += nt) z[i] = (y[i] >= 0.0) ? 1.0 : -1.0;
        __syncthreads();
        block_trsv(Lv, n, true, false, z);
        block_trsv(LTv, n, false, false, z);
        // j = argmax |z| (lowest index), z.x
        double bv = -1.0, zx = 0.0;
        int bi = INT32_MAX;
        for (int i = tid; i < n; i += nt) {
            better(bv, bi, fabs(z[i]), i);
            zx += z[i] * x[i];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            better(bv, bi, ov, oi);
        }
        zx = warp_sum(zx);
        __shared__ double zxs[32];
        if (lane == 0) { red[warp] = bv; redi[warp] = bi; zxs[warp] = zx; }
        __syncthreads();
        if (tid == 0) {
            double v = -1.0, t = 0.0;
            int idx = INT32_MAX;
            for (int k = 0; k < nw; ++k) { better(v, idx, red[k], redi[k]); t += zxs[k]; }
            stop = (v <= t) ? 1 : 0;
            redi[0] = idx;
        }
        __syncthreads();
        if (stop) break;
        const int j = redi[0];
        for (int i = tid; i < n; i += nt) x[i] = (i == j) ? 1.0 : 0.0;
        __syncthreads();
    }
    if (tid == 0) *est_out = best;
}

// --------------------------------------------------------------- helpers ----
struct Ws {
    double *w, *l, *stats, *vec, *candv;
    int *perm, *candi, *flag, *lflags, *pivots;
    void *ctl;
    double *wphys, *lphys;   // lu_perm_kernel: factors in physical row slots
    int *pos2, *at2, *candr;
};
static size_t ws_layout(int64_t n, void *base, Ws *o) {
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t at = off; off = align_up(off + bytes, 256); return at; };
    const size_t nn = (size_t)n * n * sizeof(double);
    size_t ow = take(nn), ol = take(nn), os = take(8 * sizeof(double)), ov = take((size_t)n * sizeof(double) * 2);
    size_t op = take((size_t)n * sizeof(int)), oc = take(2 * 4096 * sizeof(double)), oci = take(2 * 4096 * sizeof(int));
    size_t of = take(sizeof(int) * 4), octl = take(256);
    size_t olf = take((size_t)n * sizeof(int)), opv = take((size_t)n * sizeof(int));
    size_t owp = take(nn), olp = take(nn), op2 = take((size_t)2 * n * sizeof(int)),
           oa2 = take((size_t)2 * n * sizeof(int)), ocr = take(2 * 4096 * sizeof(int));
    if (o && base) {
        unsigned char *bb = static_cast<unsigned char *>(base);
        o->wphys = reinterpret_cast<double *>(bb + owp);
        o->lphys = reinterpret_cast<double *>(bb + olp);
        o->pos2 = reinterpret_cast<int *>(bb + op2);
        o->at2 = reinterpret_cast<int *>(bb + oa2);
        o->candr = reinterpret_cast<int *>(bb + ocr);
        o->lflags = reinterpret_cast<int *>(static_cast<unsigned char *>(base) + olf);
        o->pivots = reinterpret_cast<int *>(static_cast<unsigned char *>(base) + opv);
        unsigned char *b = static_cast<unsigned char *>(base);
        o->w = reinterpret_cast<double *>(b + ow);
        o->l = reinterpret_cast<double *>(b + ol);
        o->stats = reinterpret_cast<double *>(b + os);
        o->vec = reinterpret_cast<double *>(b + ov);
        o->perm = reinterpret_cast<int *>(b + op);
        o->candv = reinterpret_cast<double *>(b + oc);
        o->candi = reinterpret_cast<int *>(b + oci);
        o->flag = reinterpret_cast<int *>(b + of);
        o->ctl = b + octl;
    }
    return off;
}

static int coop_blocks(const void *fn, int threads, size_t smem, int64_t want) {
    int maxb = max_coop_blocks(fn, threads, smem);
    if (maxb <= 0) return 0;
    int64_t b = want < 1 ? 1 : want;
    return (int)(b > maxb ? maxb : b);
}

static int trsv_launch(TriView M, int n, bool lower, bool unit, const double *rhs, const int *perm, double *x,
                       cudaStream_t st) {
    const size_t smem = (size_t)n * sizeof(double);
    if (smem > 40 * 1024)
        SK_CUDA(cudaFuncSetAttribute(trsv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    trsv_kernel<<<1, TRSV_THREADS, smem, st>>>(M, n, lower, unit, rhs, perm, x);
    SK_LAUNCH_CHECK("trsv_kernel");
    return SK_OK;
}

// Cholesky factor of (S+S^T)/2 into ws.l; returns SK_OK or SK_NOT_POSITIVE_DEFINITE.
static int chol_factor(const double *s, int n, Ws &ws, sk_status *status, cudaStream_t st) {
    FactorCtl *ctl = static_cast<FactorCtl *>(ws.ctl);
    SK_CUDA(cudaMemsetAsync(ctl, 0, sizeof(FactorCtl), st));
    SK_CUDA(cudaMemsetAsync(ws.l, 0, (size_t)n * n * sizeof(double), st));
    symmetrize<<<(unsigned)std::min<int64_t>(((int64_t)n * n + 255) / 256, 4096), 256, 0, st>>>(s, n, ws.w);
    SK_LAUNCH_CHECK("symmetrize");
    DevStatus *defer = deferred_status();
    if (defer) {   // after an earlier recorded failure the factorisation runs on the identity
        int rc = guard_identity(ws.w, 8, n, n, n, true, st);
        if (rc) return rc;
    }
    // blocked: one CTA per SM (3 grid barriers per 32-column panel)
    const int blocks = coop_blocks((const void *)chol_blocked_kernel, THREADS, 0,
                                   std::min<int64_t>(sm_count(), ((int64_t)n * n / 2 + 1023) / 1024 + 1));
    if (!blocks) { set_error("chol_kernel not co-resident"); return SK_ERR_CUDA; }
    double *w = ws.w;
    int ni = n;
    void *args[] = {&w, &ni, &ctl};
    SK_CUDA(cudaLaunchCooperativeKernel((const void *)chol_blocked_kernel, dim3(blocks), dim3(THREADS), args, 0, st));
    SK_LAUNCH_CHECK("chol_blocked_kernel");
    lower_to_l<<<(unsigned)std::min<int64_t>(((int64_t)n * n + 255) / 256, 4096), 256, 0, st>>>(ws.w, n, ws.l);
    SK_LAUNCH_CHECK("lower_to_l");
    if (defer) return note_verdict(&ctl->fail_code, 0, &ctl->fail_col, &ctl->fail_value, nullptr, st);
    FactorCtl h;
    SK_CUDA(cudaMemcpyAsync(&h, ctl, sizeof(h), cudaMemcpyDeviceToHost, st));
    SK_CUDA(cudaStreamSynchronize(st));
    if (h.fail_code) {
        set_error("pivot %d is %g", h.fail_col, h.fail_value);
        return fill_status(status, h.fail_code, h.fail_col, h.fail_value, 0.0);
    }
    return SK_OK;
}

}  // namespace nxn
}  // namespace sk

using namespace sk;
using namespace sk::nxn;

extern "C" {

size_t sk_nxn_workspace(int64_t n) { return ws_layout(n, nullptr, nullptr) + 1024; }

int sk_chol_solve_f64(const double *s, int64_t n, const double *rhs, double *x, sk_status *status, void *wsp,
                      size_t ws_bytes, sk_stream_t stream) {
    if (!s || !rhs || !x || n <= 0 || n > 65536 || !wsp || ws_bytes < sk_nxn_workspace(n)) {
        set_error("sk_chol_solve_f64: bad arguments");
        return SK_ERR_ARG;
    }
    cudaStream_t st = (cudaStream_t)stream;
    Ws ws;
    ws_layout(n, wsp, &ws);
    // symmetry gate (src/dense.py:332-335)
    SK_CUDA(cudaMemsetAsync(ws.stats, 0, 4 * sizeof(double), st));
    sym_stats<<<(unsigned)std::min<int64_t>((n * n + 255) / 256, 1024), 256, 0, st>>>(s, (int)n, ws.stats);
    SK_LAUNCH_CHECK("sym_stats");
    if (DevStatus *defer = deferred_status()) {
        nxn_gate<<<1, 1, 0, st>>>(ws.stats, (int)n, nullptr, defer);
        SK_LAUNCH_CHECK("nxn_gate");
    } else {
        double h[4];
        SK_CUDA(cudaMemcpyAsync(h, ws.stats, 4 * sizeof(double), cudaMemcpyDeviceToHost, st));
        SK_CUDA(cudaStreamSynchronize(st));
        if (h[2] > 0) { set_error("s contains non-finite entries"); return fill_status(status, SK_NON_FINITE, -1, 0, 0); }
        if (h[1] > 10.0 * 2.220446049250313e-16 * h[0]) {
            set_error("s is not symmetric within 10*eps relative tolerance");
            return fill_status(status, SK_NOT_SYMMETRIC, -1, h[1], h[0]);
        }
    }
    int rc = chol_factor(s, (int)n, ws, status, st);
    if (rc != SK_OK) return rc;
    // y = L^{-1} rhs, x = L^{-T} y
    const TriView Lv{ws.l, 1, n}, LTv{ws.l, n, 1};
    rc = trsv_launch(Lv, (int)n, true, false, rhs, nullptr, ws.vec, st);
    if (rc) return rc;
    rc = trsv_launch(LTv, (int)n, false, false, ws.vec, nullptr, x, st);
    if (rc) return rc;
    return fill_status(status, SK_OK, -1, 0, 0);
}

int sk_gram_check(const double *g, int64_t n, double *out_host, void *wsp, size_t ws_bytes, sk_stream_t stream) {
    SK_NO_DEFER("sk_gram_check");
    if (!g || !out_host || n <= 0 || !wsp || ws_bytes < 64) {
        set_error("sk_gram_check: bad arguments");
        return SK_ERR_ARG;
    }
    cudaStream_t st = (cudaStream_t)stream;
    double *stats = static_cast<double *>(wsp);
    SK_CUDA(cudaMemsetAsync(stats, 0, 4 * sizeof(double), st));
    sym_stats<<<(unsigned)std::min<int64_t>((n * n + 255) / 256, 1024), 256, 0, st>>>(g, (int)n, stats);
    SK_LAUNCH_CHECK("sym_stats");
    trace_kernel<<<1, 256, 0, st>>>(g, (int)n, stats + 3);
    SK_LAUNCH_CHECK("trace_kernel");
    double h[4];
    SK_CUDA(cudaMemcpyAsync(h, stats, 4 * sizeof(double), cudaMemcpyDeviceToHost, st));
    SK_CUDA(cudaStreamSynchronize(st));
    out_host[0] = h[2];
    out_host[1] = h[3];
    return SK_OK;
}

int sk_chol_factor_f64(const double *s, int64_t n, double *r, sk_status *status, void *wsp, size_t ws_bytes,
                       sk_stream_t stream) {
    SK_NO_DEFER("sk_chol_factor_f64");
    if (!s || !r || n <= 0 || n > 65536 || !wsp || ws_bytes < sk_nxn_workspace(n)) {
        set_error("sk_chol_factor_f64: bad arguments");
        return SK_ERR_ARG;
    }
    cudaStream_t st = (cudaStream_t)stream;
    Ws ws;
    ws_layout(n, wsp, &ws);
    int rc = chol_factor(s, (int)n, ws, status, st);
    if (rc != SK_OK) return rc;
    // ws.l is L column-major, i.e. exactly R = L^T row-major
    SK_CUDA(cudaMemcpyAsync(r, ws.l, (size_t)n * n * sizeof(double), cudaMemcpyDeviceToDevice, st));
    return fill_status(status, SK_OK, -1, 0, 0);
}

int sk_lu_solve_f64(const double *g, int64_t n, const double *rhs, double *x, sk_status *status, void *wsp,
                    size_t ws_bytes, sk_stream_t stream) {
    if (!g || !rhs || !x || n <= 0 || n > 65536 || !wsp || ws_bytes < sk_nxn_workspace(n)) {
        set_error("sk_lu_solve_f64: bad arguments");
        return SK_ERR_ARG;
    }
    cudaStream_t st = (cudaStream_t)stream;
    Ws ws;
    ws_layout(n, wsp, &ws);
    SK_CUDA(cudaMemsetAsync(ws.stats, 0, 4 * sizeof(double), st));
    sym_stats<<<(unsigned)std::min<int64_t>((n * n + 255) / 256, 1024), 256, 0, st>>>(g, (int)n, ws.stats);
    SK_LAUNCH_CHECK("sym_stats");
    LuCtl *ctl = static_cast<LuCtl *>(ws.ctl);
    DevStatus *defer = deferred_status();
    if (defer) {   // gate and pivot threshold on the device
        SK_CUDA(cudaMemsetAsync(ctl, 0, sizeof(LuCtl), st));
        nxn_gate<<<1, 1, 0, st>>>(ws.stats, (int)n, ctl, defer);
        SK_LAUNCH_CHECK("nxn_gate");
    } else {
        double h[4];
        SK_CUDA(cudaMemcpyAsync(h, ws.stats, 4 * sizeof(double), cudaMemcpyDeviceToHost, st));
        SK_CUDA(cudaStreamSynchronize(st));
        if (h[2] > 0) { set_error("a contains non-finite entries"); return fill_status(status, SK_NON_FINITE, -1, 0, 0); }
        LuCtl c{};
        c.thresh = (double)n * 2.220446049250313e-16 * h[0];   // n * eps * max|a|
        SK_CUDA(cudaMemcpyAsync(ctl, &c, sizeof(c), cudaMemcpyHostToDevice, st));
    }
    // column-major working copy (the reference factors an order="F" copy)
    transpose_copy<<<(unsigned)std::min<int64_t>((n * n + 255) / 256, 4096), 256, 0, st>>>(g, (int)n, ws.w);
    SK_LAUNCH_CHECK("transpose_copy");
    if (defer) {   // after a recorded failure (this gate included) the LU runs on the identity
        int rg = guard_identity(ws.w, 8, n, n, n, true, st);
        if (rg) return rg;
    }
    SK_CUDA(cudaMemsetAsync(ws.l, 0, (size_t)n * n * sizeof(double), st));
    double *w = ws.w, *lm = ws.l, *cv = ws.candv;
    int *perm = ws.perm, *ci = ws.candi;
    int ni = (int)n;
    // The dataflow LU (SK_LU_FLOW=1) is bitwise the same but slower at n = 2048 (39 vs
    // 20 ms): its pivot-column critical path (update, argmax, swap, n divisions) is
    // longer than two grid barriers over the fully parallel step.
    // default: one grid barrier per step (lu_perm_kernel); SK_LU_KERNEL=barrier selects
    // the two-barrier swap kernel, SK_LU_FLOW=1 the dataflow one (all bitwise the same)
    // default for n <= 2048: the shared-memory-resident dataflow LU (lu_smem_kernel);
    // SK_LU_KERNEL=perm forces lu_perm_kernel (also the fallback when the columns do not
    // fit in shared memory)
    static const char *lu_choice = getenv("SK_LU_KERNEL");
    static const bool barrier_lu = getenv("SK_LU_FLOW") == nullptr;
    static const bool perm_lu = barrier_lu && !(lu_choice && strcmp(lu_choice, "barrier") == 0);
    static const bool smem_lu = perm_lu && !(lu_choice && strcmp(lu_choice, "perm") == 0);
    bool done = false;
    static const bool small_lu = !(lu_choice && strcmp(lu_choice, "smem") == 0);
    if (smem_lu && small_lu && n <= LU_SMALL_MAX) {
        const size_t smem = (size_t)n * n * sizeof(double);
        if (cudaFuncSetAttribute(lu_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) ==
            cudaSuccess) {
            lu_small_kernel<<<1, 512, smem, st>>>(w, ni, ws.pivots, perm, lm, ctl);
            SK_LAUNCH_CHECK("lu_small_kernel");
            done = true;
        }
        cudaGetLastError();
    }
    if (!done && smem_lu && n <= (int64_t)LUS_THREADS * LUS_ROWS) {
        const int gs = (int)std::min<int64_t>(sm_count(), n);
        const size_t smem = (size_t)((n + gs - 1) / gs) * (size_t)n * sizeof(double);
        int optin = 0, dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        if (smem + 1024 <= (size_t)optin &&
            cudaFuncSetAttribute(lu_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) == cudaSuccess &&
            coop_blocks((const void *)lu_smem_kernel, LUS_THREADS, smem, gs) == gs) {
            int *lf = ws.lflags, *pv = ws.pivots;
            double *gl = ws.lphys;
            SK_CUDA(cudaMemsetAsync(lf, 0, (size_t)n * sizeof(int), st));
            void *args[] = {&w, &ni, &gl, &pv, &lf, &lm, &ctl};
            SK_CUDA(cudaLaunchCooperativeKernel((const void *)lu_smem_kernel, dim3(gs), dim3(LUS_THREADS), args, smem, st));
            SK_LAUNCH_CHECK("lu_smem_kernel");
            perm_from_pivots<<<1, 32, 0, st>>>(pv, ni, perm);
            SK_LAUNCH_CHECK("perm_from_pivots");
            done = true;
        }
        cudaGetLastError();   // a refused attribute / occupancy query falls back below
    }
    if (done) {
    } else if (perm_lu) {
        static const char *lu_blocks_env = getenv("SK_LU_BLOCKS");   // grid-size sweeps (tools/lu_probe.py)
        const int64_t lu_want = lu_blocks_env ? atoll(lu_blocks_env) : 2 * (int64_t)sm_count();
        int blocks = coop_blocks((const void *)lu_perm_kernel, THREADS, 0,
                                 std::min<int64_t>(std::min<int64_t>(lu_want, 4096),
                                                   (n * n + THREADS * 8 - 1) / (THREADS * 8)));
        if (!blocks) { set_error("lu_perm_kernel not co-resident"); return SK_ERR_CUDA; }
        // the working copy moves to the physical-slot buffers; ws.w / ws.l get the gather
        SK_CUDA(cudaMemcpyAsync(ws.wphys, ws.w, (size_t)n * n * sizeof(double), cudaMemcpyDeviceToDevice, st));
        SK_CUDA(cudaMemsetAsync(ws.lphys, 0, (size_t)n * n * sizeof(double), st));
        double *wp = ws.wphys, *lp = ws.lphys;
        int *p2 = ws.pos2, *a2 = ws.at2, *cl = ws.candi, *cr = ws.candr;
        void *args[] = {&wp, &lp, &ni, &p2, &a2, &cv, &cl, &cr, &ctl};
        SK_CUDA(cudaLaunchCooperativeKernel((const void *)lu_perm_kernel, dim3(blocks), dim3(THREADS), args, 0, st));
        SK_LAUNCH_CHECK("lu_perm_kernel");
        lu_gather<<<(unsigned)std::min<int64_t>((n * n + 255) / 256, 4096), 256, 0, st>>>(
            ws.wphys, ws.lphys, ws.at2 + (n & 1) * n, ni, ws.w, ws.l, perm);
        SK_LAUNCH_CHECK("lu_gather");
    } else if (!barrier_lu) {
        const int blocks = coop_blocks((const void *)lu_flow_kernel, THREADS, 0, std::min<int64_t>(sm_count(), n));
        if (!blocks) { set_error("lu_flow_kernel not co-resident"); return SK_ERR_CUDA; }
        int *lf = ws.lflags, *pv = ws.pivots;
        SK_CUDA(cudaMemsetAsync(lf, 0, (size_t)n * sizeof(int), st));
        void *args[] = {&w, &lm, &perm, &ni, &pv, &lf, &ctl};
        SK_CUDA(cudaLaunchCooperativeKernel((const void *)lu_flow_kernel, dim3(blocks), dim3(THREADS), args, 0, st));
        SK_LAUNCH_CHECK("lu_flow_kernel");
        perm_from_pivots<<<1, 32, 0, st>>>(pv, ni, perm);
        SK_LAUNCH_CHECK("perm_from_pivots");
    } else {
        int blocks = coop_blocks((const void *)lu_kernel, THREADS, 0,
                                 std::min<int64_t>(2 * sm_count(), (n * n + THREADS * 8 - 1) / (THREADS * 8)));
        if (!blocks) { set_error("lu_kernel not co-resident"); return SK_ERR_CUDA; }
        void *args[] = {&w, &lm, &perm, &ni, &cv, &ci, &ctl};
        SK_CUDA(cudaLaunchCooperativeKernel((const void *)lu_kernel, dim3(blocks), dim3(THREADS), args, 0, st));
        SK_LAUNCH_CHECK("lu_kernel");
    }
    LuCtl hc{};
    if (defer) {
        int rn = note_verdict(&ctl->fail_code, 0, &ctl->fail_col, &ctl->fail_value, &ctl->thresh, st);
        if (rn) return rn;
    } else {
        SK_CUDA(cudaMemcpyAsync(&hc, ctl, sizeof(hc), cudaMemcpyDeviceToHost, st));
        SK_CUDA(cudaStreamSynchronize(st));
    }
    if (hc.fail_code) {
        set_error("pivot %d magnitude %.3e below threshold %.3e", hc.fail_col, hc.fail_value, hc.thresh);
        return fill_status(status, hc.fail_code, hc.fail_col, hc.fail_value, hc.thresh);
    }
    // x = U^{-1} L^{-1} rhs[perm]
    const TriView Lv{ws.l, 1, n}, Uv{ws.w, 1, n};
    int rc = trsv_launch(Lv, (int)n, true, true, rhs, perm, ws.vec, st);
    if (rc) return rc;
    rc = trsv_launch(Uv, (int)n, false, false, ws.vec, nullptr, x, st);
    if (rc) return rc;
    return fill_status(status, SK_OK, -1, 0, 0);
}

int sk_trsv_f64(const double *r, int64_t ldr, int64_t n, int transposed, const double *rhs, double *x,
                sk_status *status, void *wsp, size_t ws_bytes, sk_stream_t stream) {
    if (!r || !rhs || !x || n <= 0 || ldr < n || n > 65536 || !wsp || ws_bytes < 2 * sizeof(double) * (size_t)n + 256) {
        set_error("sk_trsv_f64: bad arguments");
        return SK_ERR_ARG;
    }
    cudaStream_t st = (cudaStream_t)stream;
    int *flag = static_cast<int *>(wsp);
    double *tmp = reinterpret_cast<double *>(static_cast<unsigned char *>(wsp) + 256);
    const TriView Rv{r, ldr, 1};       // R(i,k) = r[i*ldr + k]  (row-major upper)
    const TriView RTv{r, 1, ldr};      // R^T(i,k) = R(k,i)
    int big = INT32_MAX, first = INT32_MAX;
    if (deferred_status()) {   // zero diagonal recorded on the device
        int rc = note_zero_diagonal(r, ldr, n, SK_SINGULAR_TRIANGULAR, st);
        if (rc) return rc;
        SK_CUDA(cudaMemcpyAsync(tmp, rhs, (size_t)n * sizeof(double), cudaMemcpyDeviceToDevice, st));
        rc = transposed ? trsv_launch(RTv, (int)n, true, false, tmp, nullptr, x, st)
                        : trsv_launch(Rv, (int)n, false, false, tmp, nullptr, x, st);
        if (rc) return rc;
        return fill_status(status, SK_OK, -1, 0, 0);
    }
    SK_CUDA(cudaMemcpyAsync(flag, &big, sizeof(int), cudaMemcpyHostToDevice, st));
    first_zero_diag<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(Rv, (int)n, flag);
    SK_LAUNCH_CHECK("first_zero_diag");
    SK_CUDA(cudaMemcpyAsync(&first, flag, sizeof(int), cudaMemcpyDeviceToHost, st));
    SK_CUDA(cudaStreamSynchronize(st));
    if (first != INT32_MAX) {
        set_error("zero diagonal entry at index %d", first);
        return fill_status(status, SK_SINGULAR_TRIANGULAR, first, 0, 0);
    }
    SK_CUDA(cudaMemcpyAsync(tmp, rhs, (size_t)n * sizeof(double), cudaMemcpyDeviceToDevice, st));
    int rc = transposed ? trsv_launch(RTv, (int)n, true, false, tmp, nullptr, x, st)
                        : trsv_launch(Rv, (int)n, false, false, tmp, nullptr, x, st);
    if (rc) return rc;
    return fill_status(status, SK_OK, -1, 0, 0);
}

int sk_kappa0_from_gram(const double *g, int64_t n, double *kappa0_host, int *overflowed_host, void *wsp,
                        size_t ws_bytes, sk_stream_t stream) {
    SK_NO_DEFER("sk_kappa0_from_gram");
    if (!g || !kappa0_host || !overflowed_host || n <= 0 || n > 65536 || !wsp || ws_bytes < sk_nxn_workspace(n)) {
        set_error("sk_kappa0_from_gram: bad arguments");
        return SK_ERR_ARG;
    }
    cudaStream_t st = (cudaStream_t)stream;
    Ws ws;
    ws_layout(n, wsp, &ws);
    *kappa0_host = NAN;
    *overflowed_host = 1;
    // finite check and ||G||_1 (src/precision.py:231-235)
    SK_CUDA(cudaMemsetAsync(ws.stats, 0, 4 * sizeof(double), st));
    sym_stats<<<(unsigned)std::min<int64_t>((n * n + 255) / 256, 1024), 256, 0, st>>>(g, (int)n, ws.stats);
    SK_LAUNCH_CHECK("sym_stats");
    col_abs_sums<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(g, (int)n, ws.vec);
    SK_LAUNCH_CHECK("col_abs_sums");
    double h[4];
    SK_CUDA(cudaMemcpyAsync(h, ws.stats, 4 * sizeof(double), cudaMemcpyDeviceToHost, st));
    double *cs = static_cast<double *>(malloc((size_t)n * sizeof(double)));
    if (!cs) { set_error("host alloc"); return SK_ERR_ARG; }
    cudaError_t e = cudaMemcpyAsync(cs, ws.vec, (size_t)n * sizeof(double), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) { free(cs); return cuda_fail(e, "kappa0 norm1"); }
    double norm1 = -INFINITY;   // np.abs(g).sum(axis=0).max()
    for (int64_t j = 0; j < n; ++j) norm1 = (cs[j] > norm1 || cs[j] != cs[j]) ? cs[j] : norm1;
    free(cs);
    if (h[2] > 0) return SK_OK;                              // non-finite G
    if (norm1 == 0.0 || !std::isfinite(norm1)) return SK_OK;
    int rc = chol_factor(g, (int)n, ws, nullptr, st);
    if (rc == SK_NOT_POSITIVE_DEFINITE) return SK_OK;        // breakdown -> overflowed
    if (rc != SK_OK) return rc;
    const size_t smem = 3 * (size_t)n * sizeof(double);
    if (smem > 227 * 1024) { set_error("n too large for the single-CTA Hager kernel"); return SK_ERR_ARG; }
    if (smem > 40 * 1024)
        SK_CUDA(cudaFuncSetAttribute(hager_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    hager_kernel<<<1, HAGER_THREADS, smem, st>>>(ws.l, (int)n, ws.stats + 4);
    SK_LAUNCH_CHECK("hager_kernel");
    double est = 0.0;
    SK_CUDA(cudaMemcpyAsync(&est, ws.stats + 4, sizeof(double), cudaMemcpyDeviceToHost, st));
    SK_CUDA(cudaStreamSynchronize(st));
    const double value = (double)n * norm1 * est;
    if (!std::isfinite(value) || value <= 0.0) return SK_OK;
    *kappa0_host = 0.5 * log10(value);
    *overflowed_host = 0;
    return SK_OK;
}

}  // extern "C"
