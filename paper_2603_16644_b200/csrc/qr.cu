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
// reference uses BLAS there, whose summation order is unspecified; we use a fixed
// per-warp order, deterministic run to run).
//
// GPU structure: one cooperative persistent kernel, one grid barrier per column.
// Column c > j is owned by warp (c mod #warps) for the whole factorisation; step j
// has every owner apply reflector j to its columns (dot, tau*dot, rank-1 update)
// and the owner of column j+1 immediately forms reflector j+1 (look-ahead), so
// reflector j+1 is ready at the barrier.  Reflectors are double-buffered.
// The Q factor is not formed: build_preconditioner only uses R
// (src/solvers.py:196-197).  The reference's non-finite Q check
// (src/precision.py:200) cannot fire without R or tau failing first at these
// scales (|Q| entries are bounded by the reflector norms), see DESIGN.md.
#include "common.cuh"

namespace cg = cooperative_groups;

namespace sk {
namespace qr {

constexpr int THREADS = 256, WARPS = THREADS / 32;

template <typename T>
struct Ctl {
    T tau[2];
    T alpha[2];
    int fail_code;
    int fail_col;
};

// ---- binary16 pairwise tree over L values produced by f(i) (already rounded) --
template <class F>
__device__ __half tree_sum_half(int L, F f, __half *scratch) {
    using H = LevelOps<__half>;
    const int lane = threadIdx.x & 31;
    const int n3 = (L + 7) >> 3;
    for (int i = lane; i < n3; i += 32) {
        const int base = i * 8;
        const int cnt = min(8, L - base);
        __half x[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) x[u] = (u < cnt) ? f(base + u) : H::zero();
        __half y[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) y[k] = (2 * k + 1 < cnt) ? H::add(x[2 * k], x[2 * k + 1]) : x[2 * k];
        const int c1 = (cnt + 1) >> 1;
        __half z0 = (1 < c1) ? H::add(y[0], y[1]) : y[0];
        __half z1 = (3 < c1) ? H::add(y[2], y[3]) : y[2];
        const int c2 = (c1 + 1) >> 1;
        scratch[i] = (1 < c2) ? H::add(z0, z1) : z0;
    }
    __syncwarp();
    int cnt = n3;
    while (cnt > 1) {
        const int nn = (cnt + 1) >> 1;
        for (int base = 0; base < nn; base += 32) {
            const int i = base + lane;
            __half val = H::zero();
            if (i < nn) val = (2 * i + 1 < cnt) ? H::add(scratch[2 * i], scratch[2 * i + 1]) : scratch[2 * i];
            __syncwarp();
            if (i < nn) scratch[i] = val;
            __syncwarp();
        }
        cnt = nn;
    }
    const __half r = scratch[0];
    __syncwarp();
    return r;
}

// ---- native warp dot (fixed order: lane-strided partials, xor-shuffle tree) ----
template <typename T, class F>
__device__ T warp_dot_native(int L, F f) {
    using O = LevelOps<T>;
    const int lane = threadIdx.x & 31;
    T s = O::zero();
    for (int i = lane; i < L; i += 32) s = O::add(s, f(i));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s = O::add(s, __shfl_xor_sync(0xffffffffu, s, o));
    return s;
}

template <typename T, bool HALF>
__device__ T warp_dot(int L, const T *u, const T *v, T *scratch) {
    using O = LevelOps<T>;
    if constexpr (HALF) {
        return tree_sum_half(L, [&](int i) { return O::mul(u[i], v[i]); }, scratch);
    } else {
        return warp_dot_native<T>(L, [&](int i) { return O::mul(u[i], v[i]); });
    }
}

// Form reflector for column j from W[j:, j] (warp-cooperative).  Returns fail code.
template <typename T, bool HALF>
__device__ int make_reflector(T *w, int64_t ld, int d, int j, T *vout, Ctl<T> *ctl, int buf, T *scratch) {
    using O = LevelOps<T>;
    const int lane = threadIdx.x & 31;
    const int L = d - j;
    T *x = w + (int64_t)j * ld + j;
    const T nrm = O::sqrt(warp_dot<T, HALF>(L, x, x, scratch));
    if (O::to_f64(nrm) == 0.0) return SK_RANK_DEFICIENT;
    const T x0 = x[0];
    const T alpha = (O::to_f64(x0) >= 0.0) ? O::sub(O::zero(), nrm) : nrm;   // -norm if x0 >= 0
    // v = x with v0 = x0 - alpha
    for (int i = lane; i < L; i += 32) vout[i] = (i == 0) ? O::sub(x0, alpha) : x[i];
    __syncwarp();
    const T vtv = warp_dot<T, HALF>(L, vout, vout, scratch);
    if (O::to_f64(vtv) == 0.0) return SK_RANK_DEFICIENT;
    const T tau = O::div(O::from_f64(2.0), vtv);
    if (!O::finite(tau)) return SK_RANK_DEFICIENT;
    // column j of the working matrix becomes (alpha, 0, 0, ...)
    for (int i = lane; i < L; i += 32) x[i] = (i == 0) ? alpha : O::zero();
    if (lane == 0) { ctl->tau[buf] = tau; ctl->alpha[buf] = alpha; }
    __syncwarp();
    return SK_OK;
}

// Apply reflector (v, tau) of step j to column c: w[j:, c] -= v * (tau * v.w[j:, c]).
template <typename T, bool HALF>
__device__ void apply_reflector(T *w, int64_t ld, int d, int j, int c, const T *v, T tau, T *scratch) {
    using O = LevelOps<T>;
    const int lane = threadIdx.x & 31;
    const int L = d - j;
    T *col = w + (int64_t)c * ld + j;
    const T t = O::mul(tau, warp_dot<T, HALF>(L, v, col, scratch));
    for (int i = lane; i < L; i += 32) col[i] = O::sub(col[i], O::mul(v[i], t));
    __syncwarp();
}

template <typename T, bool HALF>
__global__ void __launch_bounds__(THREADS)
householder_kernel(T *w, int64_t ld, int d, int n, T *vbuf /* 2 x d */, Ctl<T> *ctl, int scratch_per_warp) {
    extern __shared__ __align__(16) unsigned char qr_smem[];
    cg::grid_group grid = cg::this_grid();
    const int warp = threadIdx.x >> 5;
    const int gwarp = blockIdx.x * WARPS + warp;
    const int nwarps = gridDim.x * WARPS;
    T *scratch = reinterpret_cast<T *>(qr_smem) + warp * scratch_per_warp;

    // reflector 0
    if (gwarp == 0) {
        const int rc = make_reflector<T, HALF>(w, ld, d, 0, vbuf, ctl, 0, scratch);
        if (rc != SK_OK && (threadIdx.x & 31) == 0) { ctl->fail_code = rc; ctl->fail_col = 0; }
    }
    grid.sync();
    for (int j = 0; j < n; ++j) {
        if (ctl->fail_code != SK_OK) return;   // uniform: read after the barrier
        const int buf = j & 1;
        const T *v = vbuf + (size_t)buf * d;
        const T tau = ctl->tau[buf];
        // columns c in (j, n) owned by this warp
        int c = j + 1 + ((gwarp - (j + 1)) % nwarps + nwarps) % nwarps;
        for (; c < n; c += nwarps) {
            apply_reflector<T, HALF>(w, ld, d, j, c, v, tau, scratch);
            if (c == j + 1) {   // look-ahead: reflector j+1 as soon as its column is final
                const int rc = make_reflector<T, HALF>(w, ld, d, j + 1, vbuf + (size_t)(buf ^ 1) * d, ctl,
                                                       buf ^ 1, scratch);
                if (rc != SK_OK && (threadIdx.x & 31) == 0) { ctl->fail_code = rc; ctl->fail_col = j + 1; }
            }
        }
        grid.sync();
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
__global__ void prescale_half(__half *a, int64_t count, double scale) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
        a[i] = __double2half((double)__half2float(a[i]) * scale);   // round_to_precision(work*scale, binary16)
}

// R (row-major f64) = promote(W[:n, :]) upper triangle, / scale; non-finite -> count
template <typename T>
__global__ void extract_r(const T *w, int64_t ld, int n, double inv_scale, double *r, int64_t ldr, int *nonfinite) {
    const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= (int64_t)n * n) return;
    const int i = (int)(idx / n), c = (int)(idx % n);
    double v = 0.0;
    if (c >= i) {
        const T x = w[(int64_t)c * ld + i];
        if (!LevelOps<T>::finite(x)) atomicAdd(nonfinite, 1);
        v = LevelOps<T>::to_f64(x) / inv_scale;
    } else {
        const T x = w[(int64_t)c * ld + i];   // exact zeros written by the factorisation
        v = LevelOps<T>::to_f64(x);
    }
    r[(int64_t)i * ldr + c] = v;
}

template <typename T>
size_t ws_bytes(int64_t d) {
    return align_up(sizeof(Ctl<T>), 256) + align_up(2 * (size_t)d * sizeof(T), 256) + 256;
}

template <typename T, bool HALF>
int run(T *w, int64_t d, int64_t n, double inv_scale, double *r, int64_t ldr, sk_status *status, void *ws,
        size_t wsb, cudaStream_t st) {
    if (wsb < ws_bytes<T>(d)) { set_error("sk_qr_r: workspace too small"); return SK_ERR_ARG; }
    unsigned char *p = static_cast<unsigned char *>(ws);
    Ctl<T> *ctl = reinterpret_cast<Ctl<T> *>(p);
    p += align_up(sizeof(Ctl<T>), 256);
    T *vbuf = reinterpret_cast<T *>(p);
    p += align_up(2 * (size_t)d * sizeof(T), 256);
    int *nonfinite = reinterpret_cast<int *>(p);
    SK_CUDA(cudaMemsetAsync(ctl, 0, sizeof(Ctl<T>), st));
    SK_CUDA(cudaMemsetAsync(nonfinite, 0, sizeof(int), st));

    const int scratch_per_warp = HALF ? (int)((d + 7) / 8 + 8) : 1;
    const size_t smem = (size_t)WARPS * scratch_per_warp * sizeof(T);
    auto kfn = householder_kernel<T, HALF>;
    if (smem > 40 * 1024) SK_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int maxb = max_coop_blocks((const void *)kfn, THREADS, smem);
    if (maxb <= 0) { set_error("sk_qr_r: kernel cannot be co-resident (d too large?)"); return SK_ERR_ARG; }
    int blocks = (int)((n + WARPS - 1) / WARPS);
    if (blocks > maxb) blocks = maxb;
    if (blocks < 1) blocks = 1;
    int di = (int)d, ni = (int)n;
    int64_t ldw = d;
    void *args[] = {&w, &ldw, &di, &ni, &vbuf, &ctl, (void *)&scratch_per_warp};
    SK_CUDA(cudaLaunchCooperativeKernel((const void *)kfn, dim3(blocks), dim3(THREADS), args, smem, st));
    SK_LAUNCH_CHECK("householder_kernel");
    int fail[2];
    SK_CUDA(cudaMemcpyAsync(fail, &ctl->fail_code, 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
    SK_CUDA(cudaStreamSynchronize(st));
    if (fail[0] != SK_OK) {
        set_error("reflector %d collapsed at working precision", fail[1]);
        return fill_status(status, fail[0], fail[1], 0.0, 0.0);
    }
    const int64_t total = n * n;
    extract_r<T><<<(unsigned)((total + 255) / 256), 256, 0, st>>>(w, d, (int)n, inv_scale, r, ldr, nonfinite);
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

}  // namespace qr
}  // namespace sk

using namespace sk;

extern "C" {

size_t sk_qr_workspace(int level, int64_t d, int64_t n) {
    (void)n;
    if (level == 16) return qr::ws_bytes<__half>(d) + 256;
    if (level == 32) return qr::ws_bytes<float>(d);
    return qr::ws_bytes<double>(d);
}

int sk_qr_r(int level, void *a_s, int64_t d, int64_t n, double *r, int64_t ldr, sk_status *status, void *ws,
            size_t ws_bytes, sk_stream_t stream) {
    if (!a_s || !r || !ws || n <= 0 || d < n || ldr < n || d > (1 << 26)) {
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
                                                                      qr::ws_bytes<__half>(d));
    SK_CUDA(cudaMemsetAsync(bits, 0, sizeof(unsigned long long), st));
    const unsigned g = (unsigned)std::min<int64_t>((count + 255) / 256, 4 * sm_count());
    qr::maxabs_half<<<g, 256, 0, st>>>(a, count, bits);
    SK_LAUNCH_CHECK("maxabs_half");
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
    qr::prescale_half<<<g, 256, 0, st>>>(a, count, scale);
    SK_LAUNCH_CHECK("prescale_half");
    // R = float64(R16) / scale  (extract_r divides by its 'inv_scale' argument)
    return qr::run<__half, true>(a, d, n, scale, r, ldr, status, ws, ws_bytes, st);
}

}  // extern "C"
