// Shared device helpers for the tdkv kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include <utility>

#include "tdkv.h"

namespace tdkv {

// ---------------------------------------------------------------------------
// host-side error plumbing (defined in tdkv_api.cu)

int32_t set_error(int32_t code, const char* fmt, ...);
int32_t check_launch(const char* what);
void count_launch(int64_t n = 1);
int sm_count();

// ---------------------------------------------------------------------------
// element / unit traits
//
// A "unit" is the per-thread memory transaction: 16 bytes on the fast path
// (LDG.128/STG.128), or exactly one rotary pair on the narrow path used when
// a row is not a multiple of 16 bytes.  Units never straddle a rotary pair.

template <typename T> struct Elt;
template <> struct Elt<float> {
    using Table = double2;                 // cos, sin in float64
    static constexpr int kDtype = TDKV_F32;
};
template <> struct Elt<__nv_bfloat16> {
    using Table = float2;                  // cos, sin rounded to float32
    static constexpr int kDtype = TDKV_BF16;
};

template <int UB> struct UnitBits;
template <> struct UnitBits<16> { using V = uint4; };
template <> struct UnitBits<8> { using V = uint2; };
template <> struct UnitBits<4> { using V = uint32_t; };

// ---------------------------------------------------------------------------
// rotation of one interleaved pair (toymodel.py:78-82)

__device__ __forceinline__ void rot_pair(float& x, float& y, double2 cs) {
    // float64 evaluation with explicit roundings (no FMA contraction) so the
    // result is bit-identical to numpy's  x*cos - y*sin  /  x*sin + y*cos.
    const double xd = (double)x, yd = (double)y;
    const double e = __dsub_rn(__dmul_rn(xd, cs.x), __dmul_rn(yd, cs.y));
    const double o = __dadd_rn(__dmul_rn(xd, cs.y), __dmul_rn(yd, cs.x));
    x = __double2float_rn(e);
    y = __double2float_rn(o);
}

__device__ __forceinline__ void rot_pair(__nv_bfloat16& x, __nv_bfloat16& y, float2 cs) {
    const float xf = __bfloat162float(x), yf = __bfloat162float(y);
    const float e = fmaf(xf, cs.x, -(yf * cs.y));
    const float o = fmaf(xf, cs.y, yf * cs.x);
    x = __float2bfloat16_rn(e);
    y = __float2bfloat16_rn(o);
}

// Rotate every pair of a unit.  ``tbl`` points at the cos/sin row of the
// token; ``j0`` is the pair index (within the head) of the unit's first pair.
template <typename T, typename V>
__device__ __forceinline__ void rotate_unit(V& v, const typename Elt<T>::Table* __restrict__ tbl,
                                            int j0) {
    constexpr int kPairs = sizeof(V) / (2 * sizeof(T));
    T* e = reinterpret_cast<T*>(&v);
#pragma unroll
    for (int p = 0; p < kPairs; ++p) {
        const typename Elt<T>::Table cs = tbl[j0 + p];
        rot_pair(e[2 * p], e[2 * p + 1], cs);
    }
}

// float '!=' over a unit (np.array_equal semantics: +0 == -0, NaN != NaN)
template <typename T, typename V>
__device__ __forceinline__ bool unit_differs(const V& a, const V& b) {
    constexpr int kN = sizeof(V) / sizeof(T);
    const T* x = reinterpret_cast<const T*>(&a);
    const T* y = reinterpret_cast<const T*>(&b);
    bool d = false;
#pragma unroll
    for (int i = 0; i < kN; ++i) d |= ((float)x[i] != (float)y[i]);
    return d;
}

// max that propagates NaN like numpy's ndarray.max()
__device__ __forceinline__ float nanmax(float a, float b) {
    return (a != a || b != b) ? __int_as_float(0x7fc00000) : fmaxf(a, b);
}

// The reference's violation magnitude, max(float(|dK|.max()), float(|dV|.max()))
// (diffstore.py:157-160): numpy's max propagates NaN within a plane; Python's
// max(k, v) returns v only when v > k, so a NaN in K wins and a NaN in V alone
// is dropped.
__device__ __forceinline__ float py_max_kv(float k, float v) { return v > k ? v : k; }

template <typename T, typename V>
__device__ __forceinline__ float unit_maxabs_nan(const V& a, const V& b) {
    constexpr int kN = sizeof(V) / sizeof(T);
    const T* x = reinterpret_cast<const T*>(&a);
    const T* y = reinterpret_cast<const T*>(&b);
    float m = 0.f;
#pragma unroll
    for (int i = 0; i < kN; ++i) m = nanmax(m, fabsf((float)x[i] - (float)y[i]));
    return m;
}


// ---------------------------------------------------------------------------
// global memory access with cache hints

template <typename V>
__device__ __forceinline__ V ld_stream(const V* p) { return __ldcs(p); }
template <>
__device__ __forceinline__ uint32_t ld_stream<uint32_t>(const uint32_t* p) {
    return __ldcs(reinterpret_cast<const unsigned int*>(p));
}
template <typename V>
__device__ __forceinline__ void st_stream(V* p, const V& v) { __stcs(p, v); }
template <>
__device__ __forceinline__ void st_stream<uint32_t>(uint32_t* p, const uint32_t& v) {
    __stcs(reinterpret_cast<unsigned int*>(p), v);
}

// ---------------------------------------------------------------------------
// mbarrier + bulk async copy (TMA engine, 1-D form: cp.async.bulk)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* smem_dst, const void* gsrc, uint32_t bytes,
                                         uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(smem_dst)),
        "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// bulk prefetch global -> L2 (no completion mechanism; 16-byte aligned,
// size a multiple of 16)
__device__ __forceinline__ void bulk_prefetch_l2(const void* gsrc, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(gsrc), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "TDKV_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra TDKV_WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}

// TMA bulk store smem -> global (bulk-group completion); the source tile must
// stay untouched until bulk_wait_read<0>() by the issuing thread
__device__ __forceinline__ void bulk_s2g(void* gdst, const void* smem_src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
                 "r"(smem_u32(smem_src)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() {
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
    asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}

// Ampere-style async copies (LDGSTS) for small metadata staging

__device__ __forceinline__ void cp_async_8(void* smem_dst, const void* gsrc) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(smem_dst)), "l"(gsrc)
                 : "memory");
}
__device__ __forceinline__ void cp_async_4(void* smem_dst, const void* gsrc) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(smem_dst)), "l"(gsrc)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
    asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// ---------------------------------------------------------------------------
// programmatic dependent launch (PDL): a kernel launched with the
// programmatic-serialization attribute may start while its predecessor in
// the stream is still running; griddep_wait() blocks until every
// predecessor grid has completed and flushed its memory, and
// griddep_launch_dependents() lets the next kernel start launching.  Both
// are no-ops for a kernel launched without the attribute.

__device__ __forceinline__ void griddep_wait() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
}
__device__ __forceinline__ void griddep_launch_dependents() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_maybe_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                                    cudaStream_t s, bool pdl, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// ---------------------------------------------------------------------------

__host__ __device__ __forceinline__ int ceil_div(int a, int b) { return (a + b - 1) / b; }

inline size_t elt_size(int dtype) { return dtype == TDKV_F32 ? 4 : 2; }

// Unit width usable for a row of ``row_elems`` elements of head_dim D:
// 16 B when both the row and the head are whole 16-byte units, else one
// rotary pair.
inline int pick_unit_bytes(int dtype, int head_dim, int row_elems) {
    const int esz = (int)elt_size(dtype);
    const int epu16 = 16 / esz;
    if (head_dim % epu16 == 0 && (row_elems * esz) % 16 == 0) return 16;
    return 2 * esz;
}

inline bool aligned(const void* p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

}  // namespace tdkv
