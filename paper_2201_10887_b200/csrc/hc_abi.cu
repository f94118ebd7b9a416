// hc_abi.cu -- ABI version and thread-local error reporting.
#include <stdarg.h>
#include <stdio.h>

#include "hc_internal.cuh"

namespace hc {

static thread_local char g_error[512] = "";

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_error, sizeof(g_error), fmt, ap);
    va_end(ap);
}

int cuda_status(const char* what) {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error("%s: %s", what, cudaGetErrorString(e));
        return HC_ECUDA;
    }
    return HC_OK;
}

}  // namespace hc

extern "C" int hc_abi_version(void) { return HC_ABI_VERSION; }

extern "C" const char* hc_last_error(void) { return hc::g_error; }

// L2 read-bandwidth probe (measurement only): every thread streams float4 words of
// an L2-resident buffer `passes` times (grid-stride, coalesced) and folds them
// into one value so the loads are kept.  bytes read = passes * n4 * 16.
namespace hc {
__global__ void __launch_bounds__(512) k_l2_read(const float4* __restrict__ buf, size_t n4, int passes,
                                                 float* sink) {
    float acc = 0.f;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (int p = 0; p < passes; ++p)
        for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
            const float4 v = __ldcg(buf + i);
            acc += (v.x + v.y) + (v.z + v.w);
        }
    if (acc == 12345.678f) *sink = acc;   // practically never: keeps the loads live
}
}  // namespace hc

extern "C" int hc_bench_l2_read(const void* buf, size_t bytes, int passes, float* sink, hc_stream_t stream) {
    HC_REQUIRE(buf && sink && passes > 0 && bytes >= 16, "hc_bench_l2_read: bad argument");
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    hc::k_l2_read<<<sms * 4, 512, 0, (cudaStream_t)stream>>>((const float4*)buf, bytes / 16, passes, sink);
    return hc::cuda_status("hc_bench_l2_read");
}
