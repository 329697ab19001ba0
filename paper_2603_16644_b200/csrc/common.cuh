// Shared device/host helpers for libsklsq (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>

#include "../../include/sklsq.h"

namespace sk {

// ---------------------------------------------------------------- errors ---
void set_error(const char *fmt, ...);
int cuda_fail(cudaError_t e, const char *where);
inline int fill_status(sk_status *st, int code, int64_t index, double value, double aux) {
    if (st) { st->code = code; st->pad = 0; st->index = index; st->value = value; st->aux = aux; }
    return code;
}

#define SK_CUDA(call)                                                   \
    do {                                                                \
        cudaError_t _e = (call);                                        \
        if (_e != cudaSuccess) return ::sk::cuda_fail(_e, #call);      \
    } while (0)

void count_launch();   // every kernel launch site passes through SK_LAUNCH_CHECK

#define SK_LAUNCH_CHECK(where)                                          \
    do {                                                                \
        ::sk::count_launch();                                           \
        cudaError_t _e = cudaGetLastError();                            \
        if (_e != cudaSuccess) return ::sk::cuda_fail(_e, where);      \
    } while (0)

int sm_count();                 // of the current device (cached per device)
int max_coop_blocks(const void *kernel, int threads, size_t smem);

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Device-side status record for kernels that detect numerical failures.
struct DevStatus {
    int code;
    int pad;
    long long index;
    double value;
    double aux;
};

// ------------------------------------------------------ deferred verdicts --
// sk_defer_verdicts (include/sklsq.h): while a device status record is installed on
// the calling host thread, the entry points that would synchronise to read a
// numerical verdict enqueue note_verdict instead and return SK_OK (CUDA-graph capture
// of a whole solve).  The first failure in stream order wins.
DevStatus *deferred_status();
// if *code != 0 (or, with want_code > 0, if *code != 0 then want_code): record it, with
// the optional index / value / aux read from the device
int note_verdict(const int *code, int want_code, const int *index, const double *value, const double *aux,
                 cudaStream_t st);
// entry points whose result is a host value: refused while verdicts are deferred
#define SK_NO_DEFER(name)                                                                      \
    do {                                                                                       \
        if (::sk::deferred_status()) {                                                         \
            ::sk::set_error("%s returns a host value: not available under sk_defer_verdicts", name); \
            return SK_ERR_ARG;                                                                 \
        }                                                                                      \
    } while (0)
// first exactly-zero diagonal entry of the row-major n x n R -> `code` with its index
int note_zero_diagonal(const double *r, int64_t ldr, int64_t n, int code, cudaStream_t st);
// if status->code != 0: overwrite the rows x cols matrix (elements of `elem_bytes`
// bytes, 2 = binary16, 4 = binary32, 8 = binary64; ld elements; col_major or row-major)
// with the identity, so the data-dependent kernels after a recorded failure see a
// well-conditioned operand instead of garbage (their results are never returned)
int guard_identity(void *a, int elem_bytes, int64_t rows, int64_t cols, int64_t ld, bool col_major,
                   cudaStream_t st);

// ------------------------------------------------------------ DMMA (FP64) --
// mma.sync m8n8k4 f64: A 8x4 (row), B 4x8 (col), C/D 8x8.  Lowers to DMMA.8x8x4
// on sm_100a (tcgen05 has no f64 kind).  Fragment ownership, lane = 4*g + t:
//   a = A[g][t], b = B[t][g], c0/c1 = C[g][2t], C[g][2t+1].
__device__ __forceinline__ void dmma884(double &c0, double &c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// ------------------------------------------------------------- cp.async ----
__device__ __forceinline__ unsigned smem_u32(const void *p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
// 16-byte async copy with zero fill of the (16 - src_bytes) tail.
__device__ __forceinline__ void cp_async16(void *dst, const void *src, int src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(dst)), "l"(src),
                 "r"(src_bytes));
}
__device__ __forceinline__ void cp_async8(void *dst, const void *src, int src_bytes) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(dst)), "l"(src),
                 "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// ------------------------------------------------------------ reductions ---
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Level-precision scalar arithmetic.  binary16 follows numpy float16 semantics
// (op in binary32, one round-to-nearest-even to binary16; for + - * / sqrt this
// equals the correctly rounded binary16 op since 24 >= 2*11+2).  The explicit
// _rn intrinsics forbid FMA contraction, which numpy never does.
template <typename T> struct LevelOps;

// binary16 arithmetic.  numpy's float16 ufuncs compute in binary32 and round to
// binary16; for +, -, x that double rounding is innocuous (24 >= 2 * 11 + 2 bits), so the
// native round-to-nearest fp16 instructions give the same bits in one instruction
// instead of two conversions, the op and a pack (_rn: never contracted into an FMA).
template <> struct LevelOps<__half> {
    using T = __half;
    __device__ static __forceinline__ T add(T a, T b) { return __hadd_rn(a, b); }
    __device__ static __forceinline__ T sub(T a, T b) { return __hsub_rn(a, b); }
    __device__ static __forceinline__ T mul(T a, T b) { return __hmul_rn(a, b); }
    __device__ static __forceinline__ T div(T a, T b) { return __float2half_rn(__fdiv_rn(__half2float(a), __half2float(b))); }
    __device__ static __forceinline__ T sqrt(T a) { return __float2half_rn(__fsqrt_rn(__half2float(a))); }
    __device__ static __forceinline__ double to_f64(T a) { return (double)__half2float(a); }
    __device__ static __forceinline__ T from_f64(double a) { return __double2half(a); }
    __device__ static __forceinline__ bool finite(T a) { return isfinite(__half2float(a)); }
    __device__ static __forceinline__ T zero() { return __float2half_rn(0.f); }
};
template <> struct LevelOps<float> {
    using T = float;
    __device__ static __forceinline__ T add(T a, T b) { return __fadd_rn(a, b); }
    __device__ static __forceinline__ T sub(T a, T b) { return __fsub_rn(a, b); }
    __device__ static __forceinline__ T mul(T a, T b) { return __fmul_rn(a, b); }
    __device__ static __forceinline__ T div(T a, T b) { return __fdiv_rn(a, b); }
    __device__ static __forceinline__ T sqrt(T a) { return __fsqrt_rn(a); }
    __device__ static __forceinline__ double to_f64(T a) { return (double)a; }
    __device__ static __forceinline__ T from_f64(double a) { return __double2float_rn(a); }
    __device__ static __forceinline__ bool finite(T a) { return isfinite(a); }
    __device__ static __forceinline__ T zero() { return 0.f; }
};
template <> struct LevelOps<double> {
    using T = double;
    __device__ static __forceinline__ T add(T a, T b) { return __dadd_rn(a, b); }
    __device__ static __forceinline__ T sub(T a, T b) { return __dsub_rn(a, b); }
    __device__ static __forceinline__ T mul(T a, T b) { return __dmul_rn(a, b); }
    __device__ static __forceinline__ T div(T a, T b) { return __ddiv_rn(a, b); }
    __device__ static __forceinline__ T sqrt(T a) { return __dsqrt_rn(a); }
    __device__ static __forceinline__ double to_f64(T a) { return a; }
    __device__ static __forceinline__ T from_f64(double a) { return a; }
    __device__ static __forceinline__ bool finite(T a) { return isfinite(a); }
    __device__ static __forceinline__ T zero() { return 0.0; }
};

// Packed FP32x2 arithmetic (sm_100 FFMA2 / FMUL2): two lanes per instruction.
__device__ __forceinline__ uint64_t f32x2(float lo, float hi) {
    return (uint64_t)__float_as_uint(lo) | ((uint64_t)__float_as_uint(hi) << 32);
}
__device__ __forceinline__ float f32x2_lo(uint64_t v) { return __uint_as_float((uint32_t)v); }
__device__ __forceinline__ float f32x2_hi(uint64_t v) { return __uint_as_float((uint32_t)(v >> 32)); }
__device__ __forceinline__ uint64_t f32x2_fma(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ uint64_t f32x2_mul(uint64_t a, uint64_t b) {
    uint64_t d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}

// Dataflow kernels (co-resident CTAs, cooperative launch): wait until *flag != 0 and
// return it (acquire); -1 after ~seconds instead of hanging if the chain is stuck.
__device__ __forceinline__ int wait_flag(const int *flag) {
    int v;
    long long spins = 0;
    while ((v = *reinterpret_cast<const volatile int *>(flag)) == 0) {
        if (++spins > (1ll << 26)) return -1;
        __nanosleep(64);
    }
    __threadfence();
    return v;
}

}  // namespace sk
