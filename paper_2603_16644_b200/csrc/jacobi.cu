// One-sided Jacobi singular values (diagnostic): jacobi_singular_values
// src/dense.py:365-415 with the circle-method round-robin schedule of
// _round_robin_rounds src/dense.py:345-362, the orthogonality gate
// sqrt(rows) * 2^-52, the tangent formula and the sweep-max-|t| < tol stop rule.
//
// All disjoint pairs of a round are rotated in parallel (one warp per pair, the
// reference batches a round the same way), one grid barrier per round inside a
// cooperative kernel; columns live column-major in the workspace so every dot
// and rotation is a coalesced stream.  Singular values are column norms, sorted
// descending on the device (bitonic, one CTA).
#include <cstdlib>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace sk {
namespace jac {

constexpr int THREADS = 256, WARPS = THREADS / 32;

struct Ctl {
    unsigned long long maxt_bits[2];   // per-sweep max |t| (double bits, >= 0), double-buffered
    int sweeps_done;
    int converged;
};

__device__ __forceinline__ int player(int pos, int r, int k) {   // circle method, k even
    if (pos == 0) return 0;
    int v = (pos - 1 - r) % (k - 1);
    if (v < 0) v += k - 1;
    return 1 + v;
}

__global__ void __launch_bounds__(THREADS)
jacobi_kernel(double *w, int64_t rows, int n, int max_sweeps, double tol, double gate, Ctl *ctl) {
    cg::grid_group grid = cg::this_grid();
    const int lane = threadIdx.x & 31;
    const int gwarp = blockIdx.x * WARPS + (threadIdx.x >> 5);
    const int nwarps = gridDim.x * WARPS;
    const int k = n + (n & 1);          // players incl. the bye (-1 -> index n when n is odd)
    const int npairs = k / 2;
    bool converged = n < 2;
    int sweep = 0;
    for (; sweep < max_sweeps && !converged; ++sweep) {
        const int sb = sweep & 1;
        for (int r = 0; r < k - 1; ++r) {
            for (int pi = gwarp; pi < npairs; pi += nwarps) {
                int p = player(pi, r, k), q = player(k - 1 - pi, r, k);
                if (p > q) { const int t = p; p = q; q = t; }
                if (q >= n) continue;   // bye
                double *cp = w + (int64_t)p * rows, *cq = w + (int64_t)q * rows;
                double app = 0, aqq = 0, apq = 0;
                for (int64_t i = lane; i < rows; i += 32) {
                    const double x = cp[i], y = cq[i];
                    app += x * x;
                    aqq += y * y;
                    apq += x * y;
                }
                app = warp_sum(app);
                aqq = warp_sum(aqq);
                apq = warp_sum(apq);
                const bool rotate = fabs(apq) > gate * sqrt(app) * sqrt(aqq);
                double t = 0.0;
                if (rotate) {
                    const double tau = (aqq - app) / (2.0 * apq);
                    const double sgn = tau >= 0 ? 1.0 : -1.0;
                    t = sgn / (fabs(tau) + hypot(1.0, tau));
                }
                const double c = 1.0 / sqrt(1.0 + t * t), s = t * c;
                if (rotate) {
                    for (int64_t i = lane; i < rows; i += 32) {
                        const double x = cp[i], y = cq[i];
                        cp[i] = c * x - s * y;
                        cq[i] = s * x + c * y;
                    }
                }
                if (lane == 0 && t != 0.0)
                    atomicMax(&ctl->maxt_bits[sb], (unsigned long long)__double_as_longlong(fabs(t)));
            }
            grid.sync();
        }
        const double mt = __longlong_as_double((long long)ctl->maxt_bits[sb]);
        converged = mt < tol;
        if (blockIdx.x == 0 && threadIdx.x == 0) ctl->maxt_bits[sb ^ 1] = 0ull;
        grid.sync();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) { ctl->sweeps_done = sweep; ctl->converged = converged ? 1 : 0; }
}

// One CTA of CT threads per pair (the columns of a pair live in registers between the
// dot products and the rotation: one L2 read and one write per element per round),
// rows <= CT * RPT.  Same schedule, gate, tangent and stop rule as jacobi_kernel; the
// three dot products are summed per thread, per warp, then over the CTA's warps in a
// fixed order.  For the n x n diagnostics (R_s, the R factor of A_p) at n = 2048 this
// is 1024 CTAs, all resident, one grid barrier per round.
constexpr int CT = 128, CT_WARPS = CT / 32;
template <int RPT>
__global__ void __launch_bounds__(CT)
jacobi_cta_kernel(double *w, int64_t rows, int n, int max_sweeps, double tol, double gate, Ctl *ctl) {
    cg::grid_group grid = cg::this_grid();
    __shared__ double red[CT_WARPS][3];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int k = n + (n & 1);
    const int npairs = k / 2;
    bool converged = n < 2;
    int sweep = 0;
    for (; sweep < max_sweeps && !converged; ++sweep) {
        const int sb = sweep & 1;
        for (int r = 0; r < k - 1; ++r) {
            for (int pi = blockIdx.x; pi < npairs; pi += gridDim.x) {
                int p = player(pi, r, k), q = player(k - 1 - pi, r, k);
                if (p > q) { const int t = p; p = q; q = t; }
                if (q >= n) continue;   // bye (uniform per CTA)
                double *cp = w + (int64_t)p * rows, *cq = w + (int64_t)q * rows;
                double x[RPT], y[RPT];
                double app = 0, aqq = 0, apq = 0;
#pragma unroll
                for (int i = 0; i < RPT; ++i) {
                    const int64_t row = tid + (int64_t)i * CT;
                    x[i] = row < rows ? cp[row] : 0.0;
                    y[i] = row < rows ? cq[row] : 0.0;
                }
#pragma unroll
                for (int i = 0; i < RPT; ++i) {
                    app += x[i] * x[i];
                    aqq += y[i] * y[i];
                    apq += x[i] * y[i];
                }
                app = warp_sum(app);
                aqq = warp_sum(aqq);
                apq = warp_sum(apq);
                if (lane == 0) { red[warp][0] = app; red[warp][1] = aqq; red[warp][2] = apq; }
                __syncthreads();
                app = red[0][0]; aqq = red[0][1]; apq = red[0][2];
#pragma unroll
                for (int v = 1; v < CT_WARPS; ++v) { app += red[v][0]; aqq += red[v][1]; apq += red[v][2]; }
                __syncthreads();   // red is reused by the next pair of this CTA
                const bool rotate = fabs(apq) > gate * sqrt(app) * sqrt(aqq);
                double t = 0.0;
                if (rotate) {
                    const double tau = (aqq - app) / (2.0 * apq);
                    const double sgn = tau >= 0 ? 1.0 : -1.0;
                    t = sgn / (fabs(tau) + hypot(1.0, tau));
                    const double c = 1.0 / sqrt(1.0 + t * t), s = t * c;
#pragma unroll
                    for (int i = 0; i < RPT; ++i) {
                        const int64_t row = tid + (int64_t)i * CT;
                        if (row < rows) {
                            cp[row] = c * x[i] - s * y[i];
                            cq[row] = s * x[i] + c * y[i];
                        }
                    }
                }
                if (tid == 0 && t != 0.0)
                    atomicMax(&ctl->maxt_bits[sb], (unsigned long long)__double_as_longlong(fabs(t)));
            }
            grid.sync();
        }
        const double mt = __longlong_as_double((long long)ctl->maxt_bits[sb]);
        converged = mt < tol;
        if (blockIdx.x == 0 && threadIdx.x == 0) ctl->maxt_bits[sb ^ 1] = 0ull;
        grid.sync();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) { ctl->sweeps_done = sweep; ctl->converged = converged ? 1 : 0; }
}

__global__ void to_colmajor(const double *a, int64_t rows, int n, int64_t lda, double *w) {
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < rows * n;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = idx / rows, i = idx % rows;
        w[idx] = a[i * lda + c];
    }
}

// column norms -> bitonic sort descending (single CTA, npow2 <= 8192)
__global__ void colnorm_sort(const double *w, int64_t rows, int n, int npow2, double *sv) {
    extern __shared__ double sh[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int c = warp; c < npow2; c += nw) {
        double s = 0.0;
        if (c < n) {
            for (int64_t i = lane; i < rows; i += 32) s += w[(int64_t)c * rows + i] * w[(int64_t)c * rows + i];
            s = warp_sum(s);
        }
        if (lane == 0) sh[c] = (c < n) ? sqrt(s) : -1.0;
    }
    __syncthreads();
    for (int size = 2; size <= npow2; size <<= 1)
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = threadIdx.x; i < npow2; i += blockDim.x) {
                const int j = i ^ stride;
                if (j > i) {
                    const bool desc = (i & size) == 0;
                    const double a = sh[i], b = sh[j];
                    if (desc ? (a < b) : (a > b)) { sh[i] = b; sh[j] = a; }
                }
            }
            __syncthreads();
        }
    for (int i = threadIdx.x; i < n; i += blockDim.x) sv[i] = sh[i];
}

}  // namespace jac
}  // namespace sk

using namespace sk;

extern "C" {

size_t sk_jacobi_workspace(int64_t rows, int64_t n) {
    return align_up((size_t)rows * n * sizeof(double), 256) + align_up((size_t)n * sizeof(double), 256) + 512;
}

int sk_jacobi_sv_f64(const double *a, int64_t rows, int64_t n, int64_t lda, int max_sweeps, double tol,
                     double *sv_host, void *ws, size_t ws_bytes, sk_stream_t stream) {
    SK_NO_DEFER("sk_jacobi_sv_f64");
    if (!a || !sv_host || rows <= 0 || n <= 0 || lda < n || n > 8192 || !ws || ws_bytes < sk_jacobi_workspace(rows, n)) {
        set_error("sk_jacobi_sv_f64: bad arguments");
        return SK_ERR_ARG;
    }
    cudaStream_t st = (cudaStream_t)stream;
    unsigned char *p = static_cast<unsigned char *>(ws);
    double *w = reinterpret_cast<double *>(p);
    p += align_up((size_t)rows * n * sizeof(double), 256);
    double *sv = reinterpret_cast<double *>(p);
    p += align_up((size_t)n * sizeof(double), 256);
    jac::Ctl *ctl = reinterpret_cast<jac::Ctl *>(p);
    SK_CUDA(cudaMemsetAsync(ctl, 0, sizeof(jac::Ctl), st));
    jac::to_colmajor<<<(unsigned)std::min<int64_t>((rows * n + 255) / 256, 8192), 256, 0, st>>>(a, rows, (int)n, lda, w);
    SK_LAUNCH_CHECK("to_colmajor");
    const double gate = sqrt((double)rows) * ldexp(1.0, -52);
    int ni = (int)n;
    int64_t r64 = rows;
    void *args[] = {&w, &r64, &ni, &max_sweeps, &tol, (void *)&gate, &ctl};
    // pair-per-CTA kernel when a column fits the CTA's registers (SK_JACOBI=warp: the
    // warp-per-pair kernel); the CTA count is capped by co-residency (cooperative launch)
    const char *je = getenv("SK_JACOBI");
    const bool cta = !(je && je[0] == 'w') && rows <= (int64_t)jac::CT * 16;
    if (cta) {
        const void *fn = rows <= jac::CT * 4 ? (const void *)jac::jacobi_cta_kernel<4>
                                            : rows <= jac::CT * 8 ? (const void *)jac::jacobi_cta_kernel<8>
                                                                  : (const void *)jac::jacobi_cta_kernel<16>;
        const int maxb = max_coop_blocks(fn, jac::CT, 0);
        const int blocks = std::max(1, (int)std::min<int64_t>((n + 1) / 2, maxb));
        SK_CUDA(cudaLaunchCooperativeKernel(fn, dim3(blocks), dim3(jac::CT), args, 0, st));
        SK_LAUNCH_CHECK("jacobi_cta_kernel");
    } else {
        int maxb = max_coop_blocks((const void *)jac::jacobi_kernel, jac::THREADS, 0);
        int blocks = (int)std::min<int64_t>((n / 2 + jac::WARPS - 1) / jac::WARPS + 1, maxb);
        if (blocks < 1) blocks = 1;
        SK_CUDA(cudaLaunchCooperativeKernel((const void *)jac::jacobi_kernel, dim3(blocks), dim3(jac::THREADS), args, 0,
                                            st));
        SK_LAUNCH_CHECK("jacobi_kernel");
    }
    int npow2 = 1;
    while (npow2 < n) npow2 <<= 1;
    const size_t smem = (size_t)npow2 * sizeof(double);
    if (smem > 40 * 1024)
        SK_CUDA(cudaFuncSetAttribute(jac::colnorm_sort, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    jac::colnorm_sort<<<1, 1024, smem, st>>>(w, rows, (int)n, npow2, sv);
    SK_LAUNCH_CHECK("colnorm_sort");
    jac::Ctl h;
    SK_CUDA(cudaMemcpyAsync(&h, ctl, sizeof(h), cudaMemcpyDeviceToHost, st));
    SK_CUDA(cudaMemcpyAsync(sv_host, sv, (size_t)n * sizeof(double), cudaMemcpyDeviceToHost, st));
    SK_CUDA(cudaStreamSynchronize(st));
    if (!h.converged) {
        set_error("Jacobi did not converge in %d sweeps", max_sweeps);
        return SK_NO_CONVERGENCE;
    }
    return SK_OK;
}

}  // extern "C"
