// capi.cu — error reporting and device queries for the C ABI.
#include <stdarg.h>

#include "common.cuh"

namespace wg {

static thread_local char g_err[512] = "";

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

int cuda_fail(cudaError_t e, const char *what) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return WG_ECUDA;
}

int sm_count() {
    static thread_local int dev = -1, count = 0;
    int cur = 0;
    cudaGetDevice(&cur);
    if (cur != dev || count == 0) {
        int c = 0;
        if (cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, cur) != cudaSuccess || c < 1) c = 148;
        dev = cur;
        count = c;
    }
    return count;
}

}  // namespace wg

extern "C" {

const char *wg_last_error(void) { return wg::g_err; }

int wg_abi_version(void) { return WG_ABI_VERSION; }

int wg_device_sm_count(int *out) {
    if (!out) {
        wg::set_error("null argument");
        return WG_EINVAL;
    }
    *out = wg::sm_count();
    return WG_OK;
}

}  // extern "C"
