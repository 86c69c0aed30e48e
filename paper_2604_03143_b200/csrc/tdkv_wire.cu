// TDDF wire format on the GPU: byte-exact packing of a
// diff into the reference's little-endian wire image (serialize_diff,
// diffstore.py:210-239) and unpacking of a wire image into a device payload
// slab (the data movement of deserialize_diff, diffstore.py:242-306; the
// structural parse and validation stay on the host, they are O(layers)).
//
// The image is a list of byte segments: header / per-layer count+flag /
// trailer literals, u32 block indices, and float32 payload blocks.  The
// one-byte flag makes every later field land at an arbitrary byte offset,
// so each thread builds one ALIGNED 32-bit word of the destination from two
// aligned source words with a funnel shift; only the <= 3 bytes at each end
// of a segment are written byte by byte (neighbouring segments own the other
// bytes of those words).
#include "tdkv_common.cuh"

namespace tdkv {

// logical 32-bit word q of a segment's byte stream
struct PackSrc {
    const uint8_t* p;
    int kind;            // TDKV_WIRE_RAW or TDKV_WIRE_BF16_TO_F32
    uint64_t n;          // stream length in bytes
    __device__ __forceinline__ uint32_t word(long long q) const {
        if (q < 0 || (uint64_t)q * 4 >= n) return 0u;
        if (kind == TDKV_WIRE_BF16_TO_F32)
            return (uint32_t)reinterpret_cast<const uint16_t*>(p)[q] << 16;
        const uint64_t b = (uint64_t)q * 4;
        if (b + 4 <= n && (reinterpret_cast<uintptr_t>(p) & 3) == 0)
            return __ldg(reinterpret_cast<const uint32_t*>(p + b));
        uint32_t w = 0;
        for (int i = 0; i < 4 && b + i < n; ++i) w |= (uint32_t)p[b + i] << (8 * i);
        return w;
    }
    __device__ __forceinline__ uint8_t byte(uint64_t i) const {
        return (uint8_t)(word((long long)(i >> 2)) >> (8 * (i & 3)));
    }
};

__global__ void wire_pack_kernel(const tdkv_wire_seg* __restrict__ segs, int n_segs,
                                 uint8_t* __restrict__ out) {
    for (int si = blockIdx.y; si < n_segs; si += gridDim.y) {
        const tdkv_wire_seg sg = segs[si];
        const uint64_t s = sg.offset, n = sg.nbytes;
        if (n == 0) continue;
        const PackSrc src{static_cast<const uint8_t*>(sg.ptr), sg.kind, n};
        const uint64_t a0 = (s + 3) & ~3ull;                 // first aligned dst byte
        const uint64_t a1 = (s + n) & ~3ull;                 // end of the aligned body
        const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
        const long long nthr = (long long)gridDim.x * blockDim.x;
        if (a0 >= a1) {                                      // shorter than one word
            for (long long i = tid; i < (long long)n; i += nthr) out[s + i] = src.byte(i);
            continue;
        }
        if (tid < (long long)(a0 - s)) out[s + tid] = src.byte(tid);               // head
        if (tid < (long long)(s + n - a1)) out[a1 + tid] = src.byte(a1 - s + tid); // tail
        const uint32_t r = (uint32_t)((a0 - s) & 3);         // stream offset of word 0, mod 4
        const long long q0 = (long long)((a0 - s) >> 2);
        const long long words = (long long)((a1 - a0) >> 2);
        uint32_t* o = reinterpret_cast<uint32_t*>(out + a0);
        for (long long w = tid; w < words; w += nthr) {
            const uint32_t lo = src.word(q0 + w), hi = src.word(q0 + w + 1);
            o[w] = r ? __funnelshift_r(lo, hi, 8 * r) : lo;
        }
    }
}

// dst word q of a segment = stream bytes [4q, 4q+4) of the wire image at
// byte offset ``offset`` (the wire buffer carries >= 4 bytes of padding)
__global__ void wire_unpack_kernel(const tdkv_wire_seg* __restrict__ segs, int n_segs,
                                   const uint8_t* __restrict__ in) {
    for (int si = blockIdx.y; si < n_segs; si += gridDim.y) {
        const tdkv_wire_seg sg = segs[si];
        const uint64_t words = sg.nbytes >> 2;
        const uint64_t base = sg.offset & ~3ull;
        const uint32_t r = (uint32_t)(sg.offset & 3);
        const uint32_t* w32 = reinterpret_cast<const uint32_t*>(in + base);
        for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < (long long)words;
             q += (long long)gridDim.x * blockDim.x) {
            const uint32_t lo = __ldg(w32 + q);
            const uint32_t v = r ? __funnelshift_r(lo, __ldg(w32 + q + 1), 8 * r) : lo;
            if (sg.kind == TDKV_WIRE_F32_TO_BF16) {
                reinterpret_cast<__nv_bfloat16*>(const_cast<void*>(sg.ptr))[q] =
                    __float2bfloat16_rn(__uint_as_float(v));
            } else {
                reinterpret_cast<uint32_t*>(const_cast<void*>(sg.ptr))[q] = v;
            }
        }
    }
}

// grid: y = segment, x = blocks per segment, sized so the largest segment
// gets ~16 words per thread (segments of one image are similar in size:
// payload blocks of one layer)
static int wire_grid_x(const long long max_words) {
    long long g = (max_words + 4095) / 4096;
    if (g > 64) g = 64;
    return (int)(g < 1 ? 1 : g);
}

}  // namespace tdkv

using namespace tdkv;

extern "C" int32_t tdkv_wire_pack(const tdkv_wire_seg* d_segs, int32_t n_segs,
                                  int64_t max_seg_bytes, void* d_out, void* stream) {
    if (n_segs < 0 || max_seg_bytes < 0)
        return set_error(TDKV_EINVAL, "tdkv_wire_pack: bad sizes");
    if (n_segs == 0) return TDKV_OK;
    if (!d_segs || !d_out) return set_error(TDKV_EINVAL, "tdkv_wire_pack: null pointer");
    if (reinterpret_cast<uintptr_t>(d_out) & 3)
        return set_error(TDKV_EINVAL, "tdkv_wire_pack: output must be 4-byte aligned");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const dim3 grid(wire_grid_x(max_seg_bytes / 4 + 1), n_segs < 65535 ? n_segs : 65535);
    wire_pack_kernel<<<grid, 256, 0, s>>>(d_segs, n_segs, static_cast<uint8_t*>(d_out));
    count_launch();
    return check_launch("tdkv_wire_pack");
}

extern "C" int32_t tdkv_wire_unpack(const tdkv_wire_seg* d_segs, int32_t n_segs,
                                    int64_t max_seg_bytes, const void* d_in, void* stream) {
    if (n_segs < 0 || max_seg_bytes < 0)
        return set_error(TDKV_EINVAL, "tdkv_wire_unpack: bad sizes");
    if (n_segs == 0) return TDKV_OK;
    if (!d_segs || !d_in) return set_error(TDKV_EINVAL, "tdkv_wire_unpack: null pointer");
    if (reinterpret_cast<uintptr_t>(d_in) & 3)
        return set_error(TDKV_EINVAL, "tdkv_wire_unpack: input must be 4-byte aligned");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const dim3 grid(wire_grid_x(max_seg_bytes / 4 + 1), n_segs < 65535 ? n_segs : 65535);
    wire_unpack_kernel<<<grid, 256, 0, s>>>(d_segs, n_segs, static_cast<const uint8_t*>(d_in));
    count_launch();
    return check_launch("tdkv_wire_unpack");
}
