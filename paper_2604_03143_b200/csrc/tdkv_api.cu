// C-ABI plumbing shared by every tdkv entry point: error strings, launch
// accounting, device facts.
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <mutex>

#include "tdkv_common.cuh"

namespace tdkv {

static thread_local char g_err[512] = "";
static std::atomic<int64_t> g_launches{0};

int32_t set_error(int32_t code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return code;
}

int32_t check_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_error(TDKV_ECUDA, "%s: %s", what, cudaGetErrorString(e));
    return TDKV_OK;
}

void count_launch(int64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

int sm_count() {
    // per-device cached fact (the only cached state in the library)
    static int cache[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (cache[dev] == 0) {
        int n = 0;
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        cache[dev] = n > 0 ? n : 148;
    }
    return cache[dev];
}

}  // namespace tdkv

extern "C" {

int32_t tdkv_version(void) { return (1 << 16) | 0; }

const char* tdkv_last_error(void) { return tdkv::g_err; }

int64_t tdkv_launch_count(void) { return tdkv::g_launches.load(std::memory_order_relaxed); }

}  // extern "C"
