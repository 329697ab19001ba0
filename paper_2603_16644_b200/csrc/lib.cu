// Library plumbing: versioning, thread-local error text, device facts.
#include <cstdarg>
#include <atomic>
#include <mutex>

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

}  // namespace sk

extern "C" {

int sk_version(void) { return 1; }

uint64_t sk_launch_count(void) { return sk::g_launches.load(std::memory_order_relaxed); }

const char *sk_last_error(void) { return sk::g_err; }

int sk_sm_count(int device) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return -1;
    return v;
}

}  // extern "C"
