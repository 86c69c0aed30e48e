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

int32_t tdkv_host_is_pinned(const void* p) {
    if (p == nullptr) return 0;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();  // a pageable pointer is not an error to keep
        return 0;
    }
    return a.type == cudaMemoryTypeHost ? 1 : 0;
}

int32_t tdkv_copy_h2d(void* d_dst, const void* h_src, int64_t nbytes, void* stream) {
    if (nbytes < 0) return tdkv::set_error(TDKV_EINVAL, "tdkv_copy_h2d: negative size");
    if (nbytes == 0) return TDKV_OK;
    if (d_dst == nullptr || h_src == nullptr)
        return tdkv::set_error(TDKV_EINVAL, "tdkv_copy_h2d: null pointer");
    cudaError_t e = cudaMemcpyAsync(d_dst, h_src, (size_t)nbytes, cudaMemcpyHostToDevice,
                                    (cudaStream_t)stream);
    if (e != cudaSuccess) return tdkv::set_error(TDKV_ECUDA, "tdkv_copy_h2d: %s", cudaGetErrorString(e));
    return TDKV_OK;
}

}  // extern "C"
