// Library plumbing: versioning, thread-local error text, device facts.
#include <cstdarg>
#include <atomic>
#include <mutex>
#include <algorithm>
#include <climits>

#include "common.cuh"

namespace sk {

static thread_local char g_err[512] = "";
static std::atomic<unsigned long long> g_launches{0};

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

int cuda_fail(cudaError_t e, const char *where) {
    set_error("CUDA error %d (%s) at %s", (int)e, cudaGetErrorString(e), where);
    return SK_ERR_CUDA;
}

int sm_count() {
    static int cache[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (!cache[dev]) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        cache[dev] = v > 0 ? v : 1;
    }
    return cache[dev];
}

int max_coop_blocks(const void *kernel, int threads, size_t smem) {
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem) != cudaSuccess)
        return 0;
    return per_sm * sm_count();
}

static thread_local DevStatus *g_deferred = nullptr;

DevStatus *deferred_status() { return g_deferred; }

__global__ void note_verdict_kernel(DevStatus *ds, const int *code, int want_code, const int *index,
                                    const double *value, const double *aux) {
    const int c = *code;
    if (c == 0 || ds->code != 0) return;
    ds->code = want_code > 0 ? want_code : c;
    ds->index = index ? *index : -1;
    ds->value = value ? *value : 0.0;
    ds->aux = aux ? *aux : 0.0;
}

int note_verdict(const int *code, int want_code, const int *index, const double *value, const double *aux,
                 cudaStream_t st) {
    note_verdict_kernel<<<1, 1, 0, st>>>(g_deferred, code, want_code, index, value, aux);
    SK_LAUNCH_CHECK("note_verdict_kernel");
    return SK_OK;
}

template <typename T>
__global__ void guard_identity_kernel(const DevStatus *ds, T *a, int64_t rows, int64_t cols, int64_t ld,
                                      bool col_major) {
    if (ds->code == 0) return;   // uniform: the record is only written by earlier kernels
    const int64_t total = rows * cols;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total; k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = k / cols, j = k % cols;
        a[col_major ? j * ld + i : i * ld + j] = T(i == j ? 1.0f : 0.0f);
    }
}

int guard_identity(void *a, int elem_bytes, int64_t rows, int64_t cols, int64_t ld, bool col_major,
                   cudaStream_t st) {
    const unsigned g = (unsigned)std::min<int64_t>((rows * cols + 255) / 256, 2 * (int64_t)sm_count());
    if (elem_bytes == 2)
        guard_identity_kernel<__half><<<g, 256, 0, st>>>(g_deferred, static_cast<__half *>(a), rows, cols, ld, col_major);
    else if (elem_bytes == 4)
        guard_identity_kernel<float><<<g, 256, 0, st>>>(g_deferred, static_cast<float *>(a), rows, cols, ld, col_major);
    else
        guard_identity_kernel<double><<<g, 256, 0, st>>>(g_deferred, static_cast<double *>(a), rows, cols, ld, col_major);
    SK_LAUNCH_CHECK("guard_identity_kernel");
    return SK_OK;
}

__global__ void note_positive_kernel(DevStatus *ds, const double *x, int code) {
    if (*x > 0.0 && ds->code == 0) {
        ds->code = code;
        ds->index = -1;
        ds->value = *x;
        ds->aux = 0.0;
    }
}

// first exactly-zero diagonal entry of a row-major R (one CTA)
__global__ void note_zero_diag_kernel(DevStatus *ds, const double *r, int64_t ldr, int64_t n, int code) {
    long long first = LLONG_MAX;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x)
        if (r[i * ldr + i] == 0.0) { first = i; break; }
    for (int o = 16; o > 0; o >>= 1) first = min(first, __shfl_xor_sync(0xffffffffu, first, o));
    __shared__ long long wmin[32];
    if ((threadIdx.x & 31) == 0) wmin[threadIdx.x >> 5] = first;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int k = 1; k < (int)(blockDim.x >> 5); ++k) first = min(first, wmin[k]);
        first = min(first, wmin[0]);
        if (first != LLONG_MAX && ds->code == 0) {
            ds->code = code;
            ds->index = first;
            ds->value = 0.0;
            ds->aux = 0.0;
        }
    }
}

int note_zero_diagonal(const double *r, int64_t ldr, int64_t n, int code, cudaStream_t st) {
    note_zero_diag_kernel<<<1, 256, 0, st>>>(g_deferred, r, ldr, n, code);
    SK_LAUNCH_CHECK("note_zero_diag_kernel");
    return SK_OK;
}

}  // namespace sk

extern "C" {

int sk_note_positive(const double *x_dev, int code, sk_stream_t stream) {
    if (!sk::g_deferred || !x_dev || code <= 0) {
        sk::set_error("sk_note_positive: bad arguments (needs sk_defer_verdicts)");
        return SK_ERR_ARG;
    }
    sk::note_positive_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(sk::g_deferred, x_dev, code);
    SK_LAUNCH_CHECK("note_positive_kernel");
    return SK_OK;
}

int sk_note_zero_diagonal(const double *r, int64_t ldr, int64_t n, int code, sk_stream_t stream) {
    if (!sk::g_deferred || !r || n <= 0 || ldr < n || code <= 0) {
        sk::set_error("sk_note_zero_diagonal: bad arguments (needs sk_defer_verdicts)");
        return SK_ERR_ARG;
    }
    return sk::note_zero_diagonal(r, ldr, n, code, (cudaStream_t)stream);
}

int sk_defer_verdicts(sk_status *status_dev) {
    sk::g_deferred = reinterpret_cast<sk::DevStatus *>(status_dev);
    return SK_OK;
}

int sk_guard_identity(int elem_bytes, void *a, int64_t rows, int64_t cols, int64_t ld, int col_major,
                      sk_stream_t stream) {
    if (!sk::g_deferred || !a || rows < 0 || cols < 0 || ld < (col_major ? rows : cols) ||
        (elem_bytes != 2 && elem_bytes != 4 && elem_bytes != 8)) {
        sk::set_error("sk_guard_identity: bad arguments (needs sk_defer_verdicts)");
        return SK_ERR_ARG;
    }
    if (rows == 0 || cols == 0) return SK_OK;
    return sk::guard_identity(a, elem_bytes, rows, cols, ld, col_major != 0, (cudaStream_t)stream);
}

int sk_note_flag(const int *flag_dev, int code, sk_stream_t stream) {
    if (!sk::g_deferred || !flag_dev || code <= 0) {
        sk::set_error("sk_note_flag: bad arguments (needs sk_defer_verdicts)");
        return SK_ERR_ARG;
    }
    return sk::note_verdict(flag_dev, code, nullptr, nullptr, nullptr, (cudaStream_t)stream);
}

int sk_version(void) { return 1; }

uint64_t sk_launch_count(void) { return sk::g_launches.load(std::memory_order_relaxed); }

const char *sk_last_error(void) { return sk::g_err; }

int sk_sm_count(int device) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return -1;
    return v;
}

}  // extern "C"
