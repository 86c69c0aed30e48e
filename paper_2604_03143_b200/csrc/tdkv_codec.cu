// K2 block-diff encoder: compare + stream compaction.
//
// Replaces diffstore.encode_diff (diffstore.py:119-182).  The compare pass
// streams both dense caches once (the reference compares every block,
// diffstore.py:149-165) and reduces a per-block "any element differs" flag
// with float '!=' semantics; the compact pass scans each (pair, layer) row of
// flags in block order and copies the changed mirror blocks, zero-padded,
// into the payload in ascending index order (diffstore.py:166-173).
#include <climits>
#include <cstdlib>

#include "tdkv_common.cuh"

namespace tdkv {

struct CodecGeom {
    int32_t num_layers;
    int32_t num_tokens;
    int32_t row_elems;
    int32_t block_size;
    int32_t nb;
    int32_t n_pairs;
    int32_t pair_minor;   // 1: items ordered (layer, block, pair) -- the family order
};

template <typename T, int UB>
__global__ void __launch_bounds__(256)
    diff_compare_kernel(const tdkv_diff_pair* __restrict__ pairs, const uint8_t* __restrict__ hinted,
                        uint8_t* __restrict__ changed, int32_t* __restrict__ violation,
                        float* __restrict__ viol_maxabs, const CodecGeom g) {
    using V = typename UnitBits<UB>::V;
    constexpr int kUnroll = 2;
    const int item = blockIdx.x;                 // (pair, layer, block)
    const int per_pair = g.num_layers * g.nb;
    const int pi = item / per_pair;
    const int rem = item - pi * per_pair;
    const int layer = rem / g.nb;
    const int b = rem - layer * g.nb;
    const int lo = b * g.block_size;
    const int hi = min(lo + g.block_size, g.num_tokens);
    const int upr = g.row_elems * (int)sizeof(T) / UB;
    const int units = (hi - lo) * upr;
    const size_t off_units = ((size_t)layer * g.num_tokens + lo) * upr;

    const tdkv_diff_pair pr = pairs[pi];
    const V* mk = static_cast<const V*>(pr.master_k) + off_units;
    const V* mv = static_cast<const V*>(pr.master_v) + off_units;
    const V* rk = static_cast<const V*>(pr.mirror_k) + off_units;
    const V* rv = static_cast<const V*>(pr.mirror_v) + off_units;

    bool diff = false;
    int u = threadIdx.x;
    for (; u + (kUnroll - 1) * (int)blockDim.x < units; u += kUnroll * blockDim.x) {
        V a[kUnroll][4];
#pragma unroll
        for (int q = 0; q < kUnroll; ++q) {
            const int w = u + q * blockDim.x;
            a[q][0] = ld_stream(mk + w);
            a[q][1] = ld_stream(rk + w);
            a[q][2] = ld_stream(mv + w);
            a[q][3] = ld_stream(rv + w);
        }
#pragma unroll
        for (int q = 0; q < kUnroll; ++q)
            diff |= unit_differs<T>(a[q][0], a[q][1]) | unit_differs<T>(a[q][2], a[q][3]);
    }
    for (; u < units; u += blockDim.x) {
        diff |= unit_differs<T>(ld_stream(mk + u), ld_stream(rk + u)) |
                unit_differs<T>(ld_stream(mv + u), ld_stream(rv + u));
    }
    const int any = __syncthreads_or(diff);
    if (threadIdx.x == 0) changed[item] = (uint8_t)(any != 0);
    if (!any || hinted[(size_t)pi * g.nb + b]) return;

    // soundness violation (rare): max |mirror - master| per plane, combined
    // as the reference does
    float mk_ = 0.f, mv_ = 0.f;
    for (int w = threadIdx.x; w < units; w += blockDim.x) {
        mk_ = nanmax(mk_, unit_maxabs_nan<T>(mk[w], rk[w]));
        mv_ = nanmax(mv_, unit_maxabs_nan<T>(mv[w], rv[w]));
    }
    __shared__ float red[2][32];
    for (int o = 16; o > 0; o >>= 1) {
        mk_ = nanmax(mk_, __shfl_xor_sync(0xffffffffu, mk_, o));
        mv_ = nanmax(mv_, __shfl_xor_sync(0xffffffffu, mv_, o));
    }
    if ((threadIdx.x & 31) == 0) {
        red[0][threadIdx.x >> 5] = mk_;
        red[1][threadIdx.x >> 5] = mv_;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        float a = 0.f, c = 0.f;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            a = nanmax(a, red[0][w]);
            c = nanmax(c, red[1][w]);
        }
        viol_maxabs[item] = py_max_kv(a, c);
        atomicMin(violation + pi, layer * g.nb + b);
    }
}

// One CTA per (pair, layer): block-ordered scan of the change flags in
// chunks of blockDim.x, then a cooperative copy of each changed block.
template <typename T, int UB>
__global__ void __launch_bounds__(256)
    diff_compact_kernel(const tdkv_diff_pair* __restrict__ pairs, const tdkv_diff_out* __restrict__ outs,
                        const uint8_t* __restrict__ changed, int32_t* __restrict__ counts,
                        const CodecGeom g) {
    using V = typename UnitBits<UB>::V;
    const int pi = blockIdx.x / g.num_layers;
    const int layer = blockIdx.x - pi * g.num_layers;
    const uint8_t* flags = changed + ((size_t)pi * g.num_layers + layer) * g.nb;
    const tdkv_diff_out out = outs[pi];
    const tdkv_diff_pair pr = pairs[pi];
    const int upr = g.row_elems * (int)sizeof(T) / UB;
    const int blk_units = g.block_size * upr;

    __shared__ int s_warp[32];
    __shared__ int s_list[256];
    __shared__ int s_total;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nwarps = blockDim.x >> 5;
    int running = 0;

    for (int base = 0; base < g.nb; base += blockDim.x) {
        const int b = base + threadIdx.x;
        const bool f = b < g.nb && flags[b];
        const unsigned bal = __ballot_sync(0xffffffffu, f);
        if (lane == 0) s_warp[warp] = __popc(bal);
        __syncthreads();
        if (threadIdx.x == 0) {
            int acc = 0;
            for (int w = 0; w < nwarps; ++w) {
                const int c = s_warp[w];
                s_warp[w] = acc;
                acc += c;
            }
            s_total = acc;
        }
        __syncthreads();
        const int local = s_warp[warp] + __popc(bal & ((1u << lane) - 1u));
        if (b < g.nb) {
            if (f) {
                // slots past ``cap`` only occur on a soundness violation (the
                // host reports it); never write outside this layer's region
                const int slot = running + local;
                if (slot < out.cap) {
                    out.indices[layer * out.cap + slot] = b;
                    out.blkmap[layer * g.nb + b] = layer * out.cap + slot;
                } else {
                    out.blkmap[layer * g.nb + b] = -1;
                }
                s_list[local] = b;
            } else {
                out.blkmap[layer * g.nb + b] = -1;
            }
        }
        __syncthreads();
        const int n = s_total;
        // copy the n changed blocks of this chunk
        const int n_copy = max(0, min(n, out.cap - running));
        for (int i = 0; i < n_copy; ++i) {
            const int blk = s_list[i];
            const int lo = blk * g.block_size;
            const int rows = min(g.block_size, g.num_tokens - lo);
            const size_t src = ((size_t)layer * g.num_tokens + lo) * upr;
            const size_t dst = ((size_t)layer * out.cap + running + i) * blk_units;
            const V* sk = static_cast<const V*>(pr.mirror_k) + src;
            const V* sv = static_cast<const V*>(pr.mirror_v) + src;
            V* pk = static_cast<V*>(out.payload_k) + dst;
            V* pv = static_cast<V*>(out.payload_v) + dst;
            const int valid = rows * upr;
            for (int w = threadIdx.x; w < blk_units; w += blockDim.x) {
                V kx, vx;
                if (w < valid) {
                    kx = ld_stream(sk + w);
                    vx = ld_stream(sv + w);
                } else {
                    kx = V{};
                    vx = V{};
                }
                pk[w] = kx;
                pv[w] = vx;
            }
        }
        running += n;
        __syncthreads();
    }
    if (threadIdx.x == 0) counts[pi * g.num_layers + layer] = running;
}

// Single-pass encoder: compare, stream compaction and payload copy in one
// launch.  Tiles are (pair, layer, block) in row-major order and are handed
// out by an atomic ticket, so a CTA only ever waits on tiles that started
// before it (no deadlock).  Each CTA compares its block, publishes
// "unchanged" (1) or "stored" (2) with release semantics, and a stored block
// computes its payload slot as the number of stored blocks before it in the
// same (pair, layer) -- a look-back over the published flags -- then copies
// the mirror block (still L2-resident: it was read microseconds ago) to the
// slot, zero-padded.  DRAM traffic is the algorithmic 2 x dense + payload.
// The violation magnitude of one block (max |mirror - master| per plane,
// combined as the reference does) and the pair's first violating block;
// every thread of the CTA calls it.
template <typename T, typename V>
__device__ __noinline__ void record_violation(const V* mk, const V* mv, const V* rk, const V* rv,
                                              int units, float* maxabs, int32_t* violation,
                                              int block_index) {
    __shared__ float red_k[32], red_v[32];
    float mk_ = 0.f, mv_ = 0.f;
    for (int w = threadIdx.x; w < units; w += blockDim.x) {
        mk_ = nanmax(mk_, unit_maxabs_nan<T>(mk[w], rk[w]));
        mv_ = nanmax(mv_, unit_maxabs_nan<T>(mv[w], rv[w]));
    }
    for (int o = 16; o > 0; o >>= 1) {
        mk_ = nanmax(mk_, __shfl_xor_sync(0xffffffffu, mk_, o));
        mv_ = nanmax(mv_, __shfl_xor_sync(0xffffffffu, mv_, o));
    }
    if ((threadIdx.x & 31) == 0) {
        red_k[threadIdx.x >> 5] = mk_;
        red_v[threadIdx.x >> 5] = mv_;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        float a = 0.f, c = 0.f;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            a = nanmax(a, red_k[w]);
            c = nanmax(c, red_v[w]);
        }
        *maxabs = py_max_kv(a, c);
        atomicMin(violation, block_index);
    }
}

// 128-thread CTAs, 8 per SM, three rounds of 4 loads in flight per thread:
// as many bytes in flight per SM as 4 CTAs of 256, but twice the CTAs, so one
// CTA's barrier / look-back / copy phase overlaps the others' streaming
// (C2 family encode 0.87 -> 0.99 of the copy peak; 64-thread CTAs and 4
// rounds per thread measured lower)
template <typename T, int UB>
__global__ void __launch_bounds__(128, 8)
    diff_encode_kernel(const tdkv_diff_pair* __restrict__ pairs,
                       const tdkv_diff_out* __restrict__ outs, const uint8_t* __restrict__ hinted,
                       int32_t* flags, int32_t* ticket, int32_t* __restrict__ counts,
                       int32_t* __restrict__ violation, float* __restrict__ viol_maxabs,
                       const CodecGeom g) {
    using V = typename UnitBits<UB>::V;
    constexpr int kUnroll = 3;
    __shared__ int s_tile, s_before;
    if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1);
    __syncthreads();
    const int item = s_tile;
    // Family order (default): the P mirrors of one master (layer, block)
    // hold consecutive tickets, so the master tile is read from DRAM once and
    // served from L2 to the other P-1 CTAs comparing against it (DRAM bytes
    // per family: master once + P mirrors + payload).  A (pair, layer)'s
    // lower blocks still hold lower tickets, so the look-back below never
    // waits on a CTA that has not started.
    int pi, layer, b;
    if (g.pair_minor) {
        const int lb = item / g.n_pairs;
        pi = item - lb * g.n_pairs;
        layer = lb / g.nb;
        b = lb - layer * g.nb;
    } else {
        const int per_pair = g.num_layers * g.nb;
        pi = item / per_pair;
        const int rem = item - pi * per_pair;
        layer = rem / g.nb;
        b = rem - layer * g.nb;
    }
    const int lo = b * g.block_size;
    const int hi = min(lo + g.block_size, g.num_tokens);
    const int upr = g.row_elems * (int)sizeof(T) / UB;
    const int units = (hi - lo) * upr;
    const size_t off_units = ((size_t)layer * g.num_tokens + lo) * upr;
    const tdkv_diff_pair pr = pairs[pi];
    const V* mk = static_cast<const V*>(pr.master_k) + off_units;
    const V* mv = static_cast<const V*>(pr.master_v) + off_units;
    const V* rk = static_cast<const V*>(pr.mirror_k) + off_units;
    const V* rv = static_cast<const V*>(pr.mirror_v) + off_units;

    bool diff = false;
    int u = threadIdx.x;
    for (; u + (kUnroll - 1) * (int)blockDim.x < units; u += kUnroll * blockDim.x) {
        V a[kUnroll][4];
#pragma unroll
        for (int q = 0; q < kUnroll; ++q) {
            const int w = u + q * blockDim.x;
            a[q][0] = __ldcg(mk + w);          // master: L2-resident for the family
            a[q][1] = __ldcg(rk + w);          // mirror stays in L2 for the copy
            a[q][2] = __ldcg(mv + w);
            a[q][3] = __ldcg(rv + w);
        }
#pragma unroll
        for (int q = 0; q < kUnroll; ++q)
            diff |= unit_differs<T>(a[q][0], a[q][1]) | unit_differs<T>(a[q][2], a[q][3]);
    }
    for (; u < units; u += blockDim.x)
        diff |= unit_differs<T>(__ldcg(mk + u), __ldcg(rk + u)) |
                unit_differs<T>(__ldcg(mv + u), __ldcg(rv + u));
    const int any = __syncthreads_or(diff);
    const bool is_hinted = hinted[(size_t)pi * g.nb + b] != 0;
    const bool stored = any && is_hinted;
    const size_t row = ((size_t)pi * g.num_layers + layer) * g.nb;
    if (threadIdx.x == 0) {
        __threadfence();
        atomicExch(flags + row + b, stored ? 2 : 1);        // publish
    }
    const tdkv_diff_out out = outs[pi];
    if (any && !is_hinted)   // soundness violation (rare): out of line, off the register budget
        record_violation<T, V>(mk, mv, rk, rv, units, viol_maxabs + row + b, violation + pi,
                               layer * g.nb + b);
    const bool last = b == g.nb - 1;
    if (!stored && !last) {
        if (threadIdx.x == 0) out.blkmap[layer * g.nb + b] = -1;
        return;
    }
    // look-back: stored blocks before b in this (pair, layer); predecessors
    // hold lower tickets, so they are running or done
    int before = 0;
    for (int j = threadIdx.x; j < b; j += blockDim.x) {
        int f;
        volatile int32_t* fp = flags + row + j;
        while ((f = *fp) == 0) {}
        before += f == 2;
    }
    __threadfence();
    for (int o = 16; o > 0; o >>= 1) before += __shfl_xor_sync(0xffffffffu, before, o);
    if (threadIdx.x == 0) s_before = 0;
    __syncthreads();
    if ((threadIdx.x & 31) == 0 && before) atomicAdd(&s_before, before);
    __syncthreads();
    const int slot = s_before;
    if (last && threadIdx.x == 0) counts[pi * g.num_layers + layer] = slot + (stored ? 1 : 0);
    if (!stored) {
        if (threadIdx.x == 0) out.blkmap[layer * g.nb + b] = -1;
        return;
    }
    if (slot >= out.cap) return;                     // only after a violation
    if (threadIdx.x == 0) {
        out.indices[layer * out.cap + slot] = b;
        out.blkmap[layer * g.nb + b] = layer * out.cap + slot;
    }
    const int blk_units = g.block_size * upr;
    const size_t dst = ((size_t)layer * out.cap + slot) * blk_units;
    V* pk = static_cast<V*>(out.payload_k) + dst;
    V* pv = static_cast<V*>(out.payload_v) + dst;
    // the mirror tile was just read with .cg, so these loads mostly hit L2;
    // 4 independent 16-byte loads per plane per thread before any store
    constexpr int kCopy = 4;
    int w = threadIdx.x;
    for (; w + (kCopy - 1) * (int)blockDim.x < units; w += kCopy * blockDim.x) {
        V kx[kCopy], vx[kCopy];
#pragma unroll
        for (int q = 0; q < kCopy; ++q) {
            kx[q] = ld_stream(rk + w + q * blockDim.x);
            vx[q] = ld_stream(rv + w + q * blockDim.x);
        }
#pragma unroll
        for (int q = 0; q < kCopy; ++q) {
            st_stream(pk + w + q * blockDim.x, kx[q]);
            st_stream(pv + w + q * blockDim.x, vx[q]);
        }
    }
    for (; w < blk_units; w += blockDim.x) {
        V kx{}, vx{};
        if (w < units) {
            kx = ld_stream(rk + w);
            vx = ld_stream(rv + w);
        }
        st_stream(pk + w, kx);
        st_stream(pv + w, vx);
    }
}

}  // namespace tdkv

using namespace tdkv;

static int32_t codec_check(const char* who, int32_t n_pairs, int32_t L, int32_t T, int32_t H,
                           int32_t D, int32_t bs, int32_t dtype) {
    if (n_pairs < 0 || L <= 0 || T <= 0 || H <= 0 || D <= 0 || bs <= 0)
        return set_error(TDKV_EINVAL, "%s: bad geometry pairs=%d L=%d T=%d H=%d D=%d bs=%d", who,
                         n_pairs, L, T, H, D, bs);
    if (dtype != TDKV_F32 && dtype != TDKV_BF16)
        return set_error(TDKV_EUNSUPPORTED, "%s: dtype %d", who, dtype);
    return TDKV_OK;
}

// unit width for the codec: 16 B when a row is a whole number of 16-byte
// units (the caller guarantees 16-byte aligned dense planes in that case),
// otherwise 4 bytes (rows are always a multiple of 4 bytes).
// TDKV_ENCODE_ORDER=pair selects the pair-major item order (each mirror's
// blocks in a row; the master is re-read per mirror) for A/B measurement
static int encode_pair_minor() {
    static const int v = [] {
        const char* e = getenv("TDKV_ENCODE_ORDER");
        return (e && e[0] == 'p') ? 0 : 1;
    }();
    return v;
}

static int codec_unit(int32_t dtype, int32_t row_elems) {
    return (row_elems * (int)elt_size(dtype)) % 16 == 0 ? 16 : 4;
}

extern "C" int32_t tdkv_diff_compare(const tdkv_diff_pair* d_pairs, int32_t n_pairs,
                                     const uint8_t* d_hinted, uint8_t* d_changed,
                                     int32_t* d_violation, float* d_viol_maxabs,
                                     int32_t num_layers, int32_t num_tokens, int32_t num_heads,
                                     int32_t head_dim, int32_t block_size, int32_t dtype,
                                     void* stream) {
    int32_t rc = codec_check("tdkv_diff_compare", n_pairs, num_layers, num_tokens, num_heads,
                             head_dim, block_size, dtype);
    if (rc) return rc;
    if (n_pairs == 0) return TDKV_OK;
    if (!d_pairs || !d_hinted || !d_changed || !d_violation || !d_viol_maxabs)
        return set_error(TDKV_EINVAL, "tdkv_diff_compare: null pointer");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    CodecGeom g{num_layers, num_tokens, num_heads * head_dim, block_size,
                ceil_div(num_tokens, block_size), n_pairs, encode_pair_minor()};
    const long long items = (long long)n_pairs * num_layers * g.nb;
    if (items > INT_MAX) return set_error(TDKV_EINVAL, "tdkv_diff_compare: batch too large");
    if (cudaMemsetAsync(d_violation, 0x7f, sizeof(int32_t) * n_pairs, s) != cudaSuccess)
        return check_launch("tdkv_diff_compare: memset");
    const int ub = codec_unit(dtype, g.row_elems);
    const dim3 grid((unsigned)items);
    if (dtype == TDKV_F32) {
        if (ub == 16)
            diff_compare_kernel<float, 16><<<grid, 256, 0, s>>>(d_pairs, d_hinted, d_changed,
                                                                d_violation, d_viol_maxabs, g);
        else
            diff_compare_kernel<float, 4><<<grid, 256, 0, s>>>(d_pairs, d_hinted, d_changed,
                                                               d_violation, d_viol_maxabs, g);
    } else {
        if (ub == 16)
            diff_compare_kernel<__nv_bfloat16, 16><<<grid, 256, 0, s>>>(
                d_pairs, d_hinted, d_changed, d_violation, d_viol_maxabs, g);
        else
            diff_compare_kernel<__nv_bfloat16, 4><<<grid, 256, 0, s>>>(
                d_pairs, d_hinted, d_changed, d_violation, d_viol_maxabs, g);
    }
    count_launch();
    return check_launch("tdkv_diff_compare");
}

extern "C" int32_t tdkv_diff_compact(const tdkv_diff_pair* d_pairs, const tdkv_diff_out* d_outs,
                                     int32_t n_pairs, const uint8_t* d_changed, int32_t* d_counts,
                                     int32_t num_layers, int32_t num_tokens, int32_t num_heads,
                                     int32_t head_dim, int32_t block_size, int32_t dtype,
                                     void* stream) {
    int32_t rc = codec_check("tdkv_diff_compact", n_pairs, num_layers, num_tokens, num_heads,
                             head_dim, block_size, dtype);
    if (rc) return rc;
    if (n_pairs == 0) return TDKV_OK;
    if (!d_pairs || !d_outs || !d_changed || !d_counts)
        return set_error(TDKV_EINVAL, "tdkv_diff_compact: null pointer");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    CodecGeom g{num_layers, num_tokens, num_heads * head_dim, block_size,
                ceil_div(num_tokens, block_size), n_pairs, encode_pair_minor()};
    const int ub = codec_unit(dtype, g.row_elems);
    const dim3 grid((unsigned)(n_pairs * num_layers));
    if (dtype == TDKV_F32) {
        if (ub == 16)
            diff_compact_kernel<float, 16><<<grid, 256, 0, s>>>(d_pairs, d_outs, d_changed, d_counts, g);
        else
            diff_compact_kernel<float, 4><<<grid, 256, 0, s>>>(d_pairs, d_outs, d_changed, d_counts, g);
    } else {
        if (ub == 16)
            diff_compact_kernel<__nv_bfloat16, 16><<<grid, 256, 0, s>>>(d_pairs, d_outs, d_changed,
                                                                        d_counts, g);
        else
            diff_compact_kernel<__nv_bfloat16, 4><<<grid, 256, 0, s>>>(d_pairs, d_outs, d_changed,
                                                                       d_counts, g);
    }
    count_launch();
    return check_launch("tdkv_diff_compact");
}

extern "C" int32_t tdkv_diff_encode(const tdkv_diff_pair* d_pairs, const tdkv_diff_out* d_outs,
                                    int32_t n_pairs, const uint8_t* d_hinted, int32_t* d_flags,
                                    int32_t* d_ticket, int32_t* d_counts, int32_t* d_violation,
                                    float* d_viol_maxabs, int32_t num_layers, int32_t num_tokens,
                                    int32_t num_heads, int32_t head_dim, int32_t block_size,
                                    int32_t dtype, void* stream) {
    int32_t rc = codec_check("tdkv_diff_encode", n_pairs, num_layers, num_tokens, num_heads,
                             head_dim, block_size, dtype);
    if (rc) return rc;
    if (n_pairs == 0) return TDKV_OK;
    if (!d_pairs || !d_outs || !d_hinted || !d_flags || !d_ticket || !d_counts || !d_violation ||
        !d_viol_maxabs)
        return set_error(TDKV_EINVAL, "tdkv_diff_encode: null pointer");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    CodecGeom g{num_layers, num_tokens, num_heads * head_dim, block_size,
                ceil_div(num_tokens, block_size), n_pairs, encode_pair_minor()};
    const long long items = (long long)n_pairs * num_layers * g.nb;
    if (items > INT_MAX) return set_error(TDKV_EINVAL, "tdkv_diff_encode: batch too large");
    if (cudaMemsetAsync(d_flags, 0, sizeof(int32_t) * items, s) != cudaSuccess ||
        cudaMemsetAsync(d_ticket, 0, sizeof(int32_t), s) != cudaSuccess ||
        cudaMemsetAsync(d_violation, 0x7f, sizeof(int32_t) * n_pairs, s) != cudaSuccess)
        return check_launch("tdkv_diff_encode: memset");
    const int ub = codec_unit(dtype, g.row_elems);
    const dim3 grid((unsigned)items);
    if (dtype == TDKV_F32) {
        if (ub == 16)
            diff_encode_kernel<float, 16><<<grid, 128, 0, s>>>(d_pairs, d_outs, d_hinted, d_flags,
                                                               d_ticket, d_counts, d_violation,
                                                               d_viol_maxabs, g);
        else
            diff_encode_kernel<float, 4><<<grid, 128, 0, s>>>(d_pairs, d_outs, d_hinted, d_flags,
                                                              d_ticket, d_counts, d_violation,
                                                              d_viol_maxabs, g);
    } else {
        if (ub == 16)
            diff_encode_kernel<__nv_bfloat16, 16><<<grid, 128, 0, s>>>(
                d_pairs, d_outs, d_hinted, d_flags, d_ticket, d_counts, d_violation, d_viol_maxabs,
                g);
        else
            diff_encode_kernel<__nv_bfloat16, 4><<<grid, 128, 0, s>>>(
                d_pairs, d_outs, d_hinted, d_flags, d_ticket, d_counts, d_violation, d_viol_maxabs,
                g);
    }
    count_launch();
    return check_launch("tdkv_diff_encode");
}
