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
