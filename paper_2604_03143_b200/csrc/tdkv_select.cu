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
template <typename T, typename V>
__global__ void __launch_bounds__(256)
    keydiff_kernel(const T* __restrict__ fresh, const T* __restrict__ cached,
                   const int64_t* __restrict__ cached_rows, int64_t n_rows, int row_elems,
                   float* __restrict__ mags) {
    constexpr int kE = sizeof(V) / sizeof(T);          // elements per load
    const int lane = threadIdx.x & 31;
    const int upr = row_elems / kE;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t r = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); r < n_rows;
         r += warps) {
        const V* f = reinterpret_cast<const V*>(fresh + (size_t)r * row_elems);
        const int64_t cr = cached_rows ? __ldg(cached_rows + r) : r;
        const V* c = reinterpret_cast<const V*>(cached + (size_t)cr * row_elems);
        double acc = 0.0;
        for (int u = lane; u < upr; u += 32) {
            const V fv = __ldcs(f + u), cv = __ldcs(c + u);
            const T* fe = reinterpret_cast<const T*>(&fv);
            const T* ce = reinterpret_cast<const T*>(&cv);
#pragma unroll
            for (int q = 0; q < kE; ++q) {
                const float d = (float)fe[q] - (float)ce[q];   // float32 difference, as numpy
                acc += (double)__fmul_rn(d, d);                // float32 product, as numpy
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) mags[r] = (float)sqrt((float)acc);
    }
}

__device__ __forceinline__ int block_excl_scan(int v, int* s_warp, int& total) {
    // exclusive block scan of one int per thread (blockDim.x <= 1024)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    if (threadIdx.x == 0) {
        int acc = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            const int c = s_warp[w];
            s_warp[w] = acc;
            acc += c;
        }
        s_warp[32] = acc;
    }
    __syncthreads();
    const int out = s_warp[warp] + x - v;
    total = s_warp[32];
    __syncthreads();
    return out;
}

// ---------------------------------------------------------------------------
// Selection of one member by one CTA: radix select on the magnitudes' bit
// patterns (a non-negative float orders like its bits) -- four 8-bit passes
// find the take-th largest value T; everything above T is selected, plus
// the lowest-index elements equal to T (ties to the lower index), compacted
// in ascending index order.  STAGED: the magnitudes are first copied into
// shared memory (one pass over L2 with 16-byte loads).

// bits(i): the magnitude's bit pattern, 0 for zero / NaN (never selected)
__device__ __forceinline__ uint32_t mag_bits(float v) { return v > 0.f ? __float_as_uint(v) : 0u; }

template <bool STAGED>
__device__ __forceinline__ void select_member_global(const float* __restrict__ mags, int n,
                                                     int budget, int32_t* __restrict__ out_idx,
                                                     int32_t* out_count, float* deviation,
                                                     int* hist, int* s_warp, double* red,
                                                     int& s_nnz, int& s_sel, int& s_rem,
                                                     uint32_t* staged) {
    const int tid = threadIdx.x, nthr = blockDim.x;
    if (tid == 0) s_nnz = 0;
    __syncthreads();
    double sum = 0.0;
    int nnz = 0;
    if (STAGED) {
        // one pass over L2 with 16-byte loads; every later pass reads smem
        const int n4 = ((reinterpret_cast<uintptr_t>(mags) & 15) == 0) ? n / 4 : 0;
        for (int i = tid; i < n4; i += nthr) {
            const float4 v = __ldcg(reinterpret_cast<const float4*>(mags) + i);
            sum += (double)v.x;
            sum += (double)v.y;
            sum += (double)v.z;
            sum += (double)v.w;
            nnz += (v.x > 0.f) + (v.y > 0.f) + (v.z > 0.f) + (v.w > 0.f);
            reinterpret_cast<uint4*>(staged)[i] =
                make_uint4(mag_bits(v.x), mag_bits(v.y), mag_bits(v.z), mag_bits(v.w));
        }
        for (int i = 4 * n4 + tid; i < n; i += nthr) {
            const float v = __ldcg(mags + i);
            sum += (double)v;
            nnz += v > 0.f;
            staged[i] = mag_bits(v);
        }
    } else {
        for (int i = tid; i < n; i += nthr) {
            const float v = __ldcg(mags + i);
            sum += (double)v;
            nnz += v > 0.f;
        }
    }
    auto bits_at = [&](int i) -> uint32_t {
        return STAGED ? staged[i] : mag_bits(__ldcg(mags + i));
    };
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
        double acc = 0.0;
        for (int w = 0; w < (nthr >> 5); ++w) acc += red[w];
        *deviation = (float)acc;
        s_rem = min(budget, s_nnz);
    }
    __syncthreads();
    const int take = s_rem;
    if (take <= 0) {
        if (tid == 0) *out_count = 0;
        __syncthreads();
        return;
    }
    uint32_t prefix = 0u, mask = 0u;
    for (int shift = 24; shift >= 0; shift -= 8) {
        for (int b = tid; b < 256; b += nthr) hist[b] = 0;
        __syncthreads();
        for (int base = 0; base < n; base += nthr) {
            const int i = base + tid;
            const uint32_t x = i < n ? bits_at(i) : 0u;
            const bool live = i < n && (x & mask) == prefix;
            const unsigned bin = live ? (x >> shift) & 255u : 256u;
            const unsigned peers = __match_any_sync(0xffffffffu, bin);
            if (live && (__ffs(peers) - 1) == (tid & 31)) atomicAdd(&hist[bin], __popc(peers));
        }
        __syncthreads();
        if (tid < 32) {
            int c[8], local = 0;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                c[q] = hist[255 - 8 * tid - q];
                local += c[q];
            }
            int incl = local;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (tid >= o) incl += y;
            }
            const int before = incl - local;
            const int rem = s_rem;
            __syncwarp();
            if (before < rem && incl >= rem) {
                int acc = before;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    if (acc + c[q] >= rem) {
                        s_sel = 255 - 8 * tid - q;
                        s_rem = rem - acc;
                        break;
                    }
                    acc += c[q];
                }
            }
        }
        __syncthreads();
        prefix |= (uint32_t)s_sel << shift;
        mask |= 255u << shift;
        __syncthreads();
    }
    // keep everything above the threshold pattern plus the first need_eq
    // elements equal to it (ties to the lower index), compacted ascending:
    // each thread owns a contiguous run of indices, so two block scans place
    // every kept index
    const uint32_t thr = prefix;
    const int need_eq = s_rem;
    const int per = (n + nthr - 1) / nthr;
    const int i0 = min(n, tid * per), i1 = min(n, i0 + per);
    int eq_cnt = 0;
    for (int i = i0; i < i1; ++i) eq_cnt += bits_at(i) == thr;
    int total;
    const int eq_before = block_excl_scan(eq_cnt, s_warp, total);
    int keep_cnt = 0, eqr = eq_before;
    for (int i = i0; i < i1; ++i) {
        const uint32_t x = bits_at(i);
        if (x > thr) {
            ++keep_cnt;
        } else if (x == thr) {
            keep_cnt += eqr < need_eq;
            ++eqr;
        }
    }
    int pos = block_excl_scan(keep_cnt, s_warp, total);
    eqr = eq_before;
    for (int i = i0; i < i1; ++i) {
        const uint32_t x = bits_at(i);
        bool keep = x > thr;
        if (x == thr) keep = eqr++ < need_eq;
        if (keep) out_idx[pos++] = i;
    }
    if (tid == 0) *out_count = take;
    __syncthreads();
}

__global__ void __launch_bounds__(512)
    select_kernel(const float* __restrict__ mags, const int64_t* __restrict__ member_off,
                  const int32_t* __restrict__ budget, const int64_t* __restrict__ out_off,
                  int32_t* __restrict__ out_idx, int32_t* __restrict__ out_count,
                  float* __restrict__ deviation) {
    extern __shared__ __align__(16) uint32_t bits[];
    __shared__ double red[32];
    __shared__ int s_warp[33];
    __shared__ int hist[256];
    __shared__ int s_nnz, s_sel, s_rem;
    const int m = blockIdx.x;
    const int64_t off = member_off[m];
    const int n = (int)(member_off[m + 1] - off);
    select_member_global<true>(mags + off, n, budget[m], out_idx + (out_off ? out_off[m] : off),
                               out_count + m,
                               deviation + m, hist, s_warp, red, s_nnz, s_sel, s_rem, bits);
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
    const bool vec = (row_elems * elt_size(dtype)) % 16 == 0 && aligned(d_fresh, 16) &&
                     aligned(d_cached, 16);
    if (dtype == TDKV_F32) {
        const float* f = static_cast<const float*>(d_fresh);
        const float* c = static_cast<const float*>(d_cached);
        if (vec)
            keydiff_kernel<float, uint4><<<(unsigned)grid, 256, 0, s>>>(f, c, d_cached_rows, n_rows,
                                                                        row_elems, d_mags);
        else
            keydiff_kernel<float, float><<<(unsigned)grid, 256, 0, s>>>(f, c, d_cached_rows, n_rows,
                                                                        row_elems, d_mags);
    } else if (dtype == TDKV_BF16) {
        const __nv_bfloat16* f = static_cast<const __nv_bfloat16*>(d_fresh);
        const __nv_bfloat16* c = static_cast<const __nv_bfloat16*>(d_cached);
        if (vec)
            keydiff_kernel<__nv_bfloat16, uint4><<<(unsigned)grid, 256, 0, s>>>(
                f, c, d_cached_rows, n_rows, row_elems, d_mags);
        else
            keydiff_kernel<__nv_bfloat16, __nv_bfloat16><<<(unsigned)grid, 256, 0, s>>>(
                f, c, d_cached_rows, n_rows, row_elems, d_mags);
    } else {
        return set_error(TDKV_EUNSUPPORTED, "tdkv_keydiff: dtype %d", dtype);
    }
    count_launch();
    return check_launch("tdkv_keydiff");
}

extern "C" int32_t tdkv_select_important(const float* d_mags, const int64_t* d_member_off,
                                         const int32_t* d_budget, const int64_t* d_out_off,
                                         int32_t n_members,
                                         int32_t max_count, int32_t* d_out_idx,
                                         int32_t* d_out_count, float* d_deviation, void* stream) {
    if (n_members < 0 || max_count < 0) return set_error(TDKV_EINVAL, "tdkv_select_important: bad sizes");
    if (n_members == 0) return TDKV_OK;
    if (max_count > 49152)
        return set_error(TDKV_EUNSUPPORTED,
                         "tdkv_select_important: %d positions per member (max 49152)", max_count);
    if (!d_mags || !d_member_off || !d_budget || !d_out_idx || !d_out_count || !d_deviation)
        return set_error(TDKV_EINVAL, "tdkv_select_important: null pointer");
    const size_t smem = (size_t)(max_count > 0 ? max_count : 1) * 4;
    if (cudaFuncSetAttribute(select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
        return check_launch("tdkv_select_important: cudaFuncSetAttribute");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    select_kernel<<<n_members, 512, smem, s>>>(d_mags, d_member_off, d_budget, d_out_off,
                                               d_out_idx,
                                               d_out_count, d_deviation);
    count_launch();
    return check_launch("tdkv_select_important");
}

