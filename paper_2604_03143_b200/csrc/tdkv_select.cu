// K4 check-layer key difference + per-member top-k selection.
//
// Replaces the "one batched difference pass" of pic.probe_and_select
// (pic.py:268-281): key_diff (pic.py:166-171) -- the per-position L2 norm of
// fresh minus cached check-layer keys over (H, D) -- for every member's
// shared rows at once, then per member the top ceil(r*S) positions with
// nonzero magnitude, ties to the lower index, returned ascending
// (select_important, pic.py:180-189), and the member's deviation score, the
// sum of its magnitudes (pic.py:280).
#include <cfloat>

#include "tdkv_common.cuh"

namespace tdkv {

// One warp per row: sum of squared differences accumulated in float64 (the
// reference accumulates in float32 -- any order difference stays far below
// the float32 rounding of the result), sqrt, rounded to float32.
template <typename T>
__global__ void __launch_bounds__(256)
    keydiff_kernel(const T* __restrict__ fresh, const T* __restrict__ cached,
                   const int64_t* __restrict__ cached_rows, int64_t n_rows, int row_elems,
                   float* __restrict__ mags) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t r = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); r < n_rows;
         r += warps) {
        const T* f = fresh + (size_t)r * row_elems;
        const int64_t cr = cached_rows ? __ldg(cached_rows + r) : r;
        const T* c = cached + (size_t)cr * row_elems;
        double acc = 0.0;
        for (int e = lane; e < row_elems; e += 32) {
            const float d = (float)f[e] - (float)c[e];     // float32 difference, as numpy
            acc += (double)__fmul_rn(d, d);                // float32 product, as numpy
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) mags[r] = (float)sqrt((float)acc);
    }
}

// One CTA per member: bitonic sort of (descending magnitude, ascending
// index) keys in shared memory, keep the first min(budget, nonzero) and emit
// them in ascending index order.
__global__ void __launch_bounds__(512)
    select_kernel(const float* __restrict__ mags, const int64_t* __restrict__ member_off,
                  const int32_t* __restrict__ budget, int32_t* __restrict__ out_idx,
                  int32_t* __restrict__ out_count, float* __restrict__ deviation) {
    extern __shared__ __align__(16) unsigned long long keys[];
    __shared__ double red[32];
    __shared__ int s_nnz;
    __shared__ int s_warp[32];
    const int m = blockIdx.x;
    const int64_t off = member_off[m];
    const int n = (int)(member_off[m + 1] - off);
    int npad = 1;
    while (npad < n) npad <<= 1;
    const int tid = threadIdx.x, nthr = blockDim.x;
    if (tid == 0) s_nnz = 0;
    __syncthreads();

    double sum = 0.0;
    int nnz = 0;
    for (int i = tid; i < npad; i += nthr) {
        unsigned long long key = ~0ull;
        if (i < n) {
            const float v = mags[off + i];
            sum += (double)v;
            // v >= 0: its bit pattern orders like its value; invert for a
            // descending sort, index in the low word breaks ties ascending
            const uint32_t bits = v > 0.f ? __float_as_uint(v) : 0u;
            nnz += v > 0.f;
            key = ((unsigned long long)(~bits) << 32) | (uint32_t)i;
        }
        keys[i] = key;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        sum += __shfl_xor_sync(0xffffffffu, sum, o);
        nnz += __shfl_xor_sync(0xffffffffu, nnz, o);
    }
    if ((tid & 31) == 0) {
        red[tid >> 5] = sum;
        atomicAdd(&s_nnz, nnz);
    }
    __syncthreads();
    if (tid == 0) {
        double s = 0.0;
        for (int w = 0; w < (nthr >> 5); ++w) s += red[w];
        deviation[m] = (float)s;
    }
    // bitonic sort ascending
    for (int k = 2; k <= npad; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = tid; i < npad; i += nthr) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const unsigned long long a = keys[i], b = keys[ixj];
                    const bool up = (i & k) == 0;
                    if ((a > b) == up) {
                        keys[i] = b;
                        keys[ixj] = a;
                    }
                }
            }
            __syncthreads();
        }
    }
    const int take = min(budget[m], s_nnz);
    // mark the selected indices (reuse the tail of the key array as flags is
    // unsafe while reading keys -> two passes through a flag word array)
    __syncthreads();
    uint32_t* flags = reinterpret_cast<uint32_t*>(keys + npad);   // npad words after keys
    for (int i = tid; i < npad; i += nthr) flags[i] = 0u;
    __syncthreads();
    for (int i = tid; i < take; i += nthr) flags[(uint32_t)(keys[i] & 0xffffffffu)] = 1u;
    __syncthreads();
    // block-ordered compaction of the flags (ascending indices)
    int running = 0;
    const int lane = tid & 31, warp = tid >> 5;
    for (int base = 0; base < n; base += nthr) {
        const int i = base + tid;
        const bool f = i < n && flags[i];
        const unsigned bal = __ballot_sync(0xffffffffu, f);
        if (lane == 0) s_warp[warp] = __popc(bal);
        __syncthreads();
        if (tid == 0) {
            int acc = 0;
            for (int w = 0; w < (nthr >> 5); ++w) {
                const int c = s_warp[w];
                s_warp[w] = acc;
                acc += c;
            }
            s_warp[31] = acc;   // nthr <= 512 -> at most 16 warps, slot 31 is free
        }
        __syncthreads();
        if (f) out_idx[off + running + s_warp[warp] + __popc(bal & ((1u << lane) - 1u))] = i;
        running += s_warp[31];
        __syncthreads();
    }
    if (tid == 0) out_count[m] = take;
}

}  // namespace tdkv

using namespace tdkv;

extern "C" int32_t tdkv_keydiff(const void* d_fresh, const void* d_cached,
                                const int64_t* d_cached_rows, int64_t n_rows, int32_t row_elems,
                                int32_t dtype, float* d_mags, void* stream) {
    if (n_rows < 0 || row_elems <= 0) return set_error(TDKV_EINVAL, "tdkv_keydiff: bad sizes");
    if (n_rows == 0) return TDKV_OK;
    if (!d_fresh || !d_cached || !d_mags) return set_error(TDKV_EINVAL, "tdkv_keydiff: null pointer");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    long long grid = (n_rows + 7) / 8;
    if (grid > sm_count() * 16) grid = sm_count() * 16;
    if (dtype == TDKV_F32) {
        keydiff_kernel<float><<<(unsigned)grid, 256, 0, s>>>(
            static_cast<const float*>(d_fresh), static_cast<const float*>(d_cached), d_cached_rows,
            n_rows, row_elems, d_mags);
    } else if (dtype == TDKV_BF16) {
        keydiff_kernel<__nv_bfloat16><<<(unsigned)grid, 256, 0, s>>>(
            static_cast<const __nv_bfloat16*>(d_fresh), static_cast<const __nv_bfloat16*>(d_cached),
            d_cached_rows, n_rows, row_elems, d_mags);
    } else {
        return set_error(TDKV_EUNSUPPORTED, "tdkv_keydiff: dtype %d", dtype);
    }
    count_launch();
    return check_launch("tdkv_keydiff");
}

extern "C" int32_t tdkv_select_important(const float* d_mags, const int64_t* d_member_off,
                                         const int32_t* d_budget, int32_t n_members,
                                         int32_t max_count, int32_t* d_out_idx,
                                         int32_t* d_out_count, float* d_deviation, void* stream) {
    if (n_members < 0 || max_count < 0) return set_error(TDKV_EINVAL, "tdkv_select_important: bad sizes");
    if (n_members == 0) return TDKV_OK;
    if (max_count > 16384)
        return set_error(TDKV_EUNSUPPORTED,
                         "tdkv_select_important: %d positions per member (max 16384)", max_count);
    if (!d_mags || !d_member_off || !d_budget || !d_out_idx || !d_out_count || !d_deviation)
        return set_error(TDKV_EINVAL, "tdkv_select_important: null pointer");
    int npad = 1;
    while (npad < max_count) npad <<= 1;
    const size_t smem = (size_t)npad * 8 + (size_t)npad * 4;
    if (cudaFuncSetAttribute(select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
        return check_launch("tdkv_select_important: cudaFuncSetAttribute");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    select_kernel<<<n_members, 512, smem, s>>>(d_mags, d_member_off, d_budget, d_out_idx,
                                               d_out_count, d_deviation);
    count_launch();
    return check_launch("tdkv_select_important");
}
