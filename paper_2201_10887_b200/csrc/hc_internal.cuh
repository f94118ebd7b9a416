// hc_internal.cuh -- shared device helpers for libheightcast_cuda (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "heightcast.h"

// ---------------------------------------------------------------------------
// error reporting (thread-local, no other global state)

namespace hc {

void set_error(const char* fmt, ...);
int cuda_status(const char* what);   // HC_OK or HC_ECUDA after a launch

#define HC_REQUIRE(cond, ...)          \
    do {                               \
        if (!(cond)) {                 \
            ::hc::set_error(__VA_ARGS__); \
            return HC_EINVAL;          \
        }                              \
    } while (0)

// ---------------------------------------------------------------------------
// exactly-rounded float64 arithmetic: these intrinsics are never contracted into
// FMA, so expressions below keep the reference's two roundings per a*b+c.

__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }

// ordered-int encoding of float so atomicMin/atomicMax on int order like floats
__device__ __forceinline__ int32_t float_key(float f) {
    int32_t b = __float_as_int(f);
    return b >= 0 ? b : (b ^ 0x7fffffff);
}
__host__ __device__ __forceinline__ float key_float(int32_t k) {
    int32_t b = k >= 0 ? k : (k ^ 0x7fffffff);
#ifdef __CUDA_ARCH__
    return __int_as_float(b);
#else
    float f;
    __builtin_memcpy(&f, &b, 4);
    return f;
#endif
}
constexpr int32_t KEY_POS_INF = 0x7f800000;           // key(+inf)
constexpr int32_t KEY_NEG_INF = (int32_t)0x807fffff;  // key(-inf) = 0xff800000 ^ 0x7fffffff

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

constexpr int kSMs = 148;

}  // namespace hc
