// K5 selective recompute, non-GEMM stages (reference: toymodel._selective_
// forward, toymodel.py:99-151).  Per layer the host runs
//   tdkv_gemm      qkv = h @ [Wq | Wk | Wv]           (tensor cores)
//   tdkv_qkv_rope  q, k rotated to the fixed rows' positions (float64
//                  rotation, bit-compatible with rope_apply), k and v written
//                  to the layer's output planes
//   tdkv_attention causal softmax attention of every fixed row over the
//                  context, fresh rows overriding cached ones
//   tdkv_gemm      h += mix @ Wm                       (tensor cores)
#include "tdkv_common.cuh"

namespace tdkv {

__global__ void qkv_rope_kernel(const float* __restrict__ qkv, const double2* __restrict__ table,
                                int F, int H, int D, float* __restrict__ q_out,
                                float* __restrict__ k_out, float* __restrict__ v_out) {
    const int hid = H * D;
    const int half = D >> 1;
    const long long pairs = (long long)F * (hid >> 1);
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < pairs;
         i += (long long)gridDim.x * blockDim.x) {
        const int f = (int)(i / (hid >> 1));
        const int p = (int)(i - (long long)f * (hid >> 1));    // pair index within the row
        const int e = 2 * p;
        const int j = (e % D) >> 1;                              // pair index within the head
        const double2 cs = table[(size_t)f * half + j];
        const float* row = qkv + (size_t)f * 3 * hid;
        float qx = row[e], qy = row[e + 1];
        float kx = row[hid + e], ky = row[hid + e + 1];
        rot_pair(qx, qy, cs);
        rot_pair(kx, ky, cs);
        q_out[(size_t)f * hid + e] = qx;
        q_out[(size_t)f * hid + e + 1] = qy;
        k_out[(size_t)f * hid + e] = kx;
        k_out[(size_t)f * hid + e + 1] = ky;
        v_out[(size_t)f * hid + e] = row[2 * hid + e];
        v_out[(size_t)f * hid + e + 1] = row[2 * hid + e + 1];
    }
}

// Attention of one fixed row over its context, for one head (one CTA).
// Keys/values of token t come from the fresh rows when fresh_of[t] >= 0,
// else from the context planes; the row sees t < tn (causal by sequence
// index, tn = fix_idx + 1).  Key and value rows are staged kTile tokens at
// a time in shared memory with coalesced loads (rows padded to an even pitch:
// at most 2-way conflicted column reads); every score is one sequential fmaf chain over
// d and every output one sequential float64 sum over t, so the arithmetic is
// the same whatever the tiling.
constexpr int kAttnTile = 32;

// staged rows are padded to an even pitch: 8-byte async copies stay aligned
// and column reads by 32 lanes (one token each) are at most 2-way conflicted
__host__ __device__ inline int attn_pitch(int D) { return D + 2; }

// Stage head h of rows [t0, t0 + n) of the K or V plane (fresh row when
// fresh_of[t] >= 0, else the context row) into s_tile: one warp per row, each
// lane issuing 8-byte async copies, every copy of the tile in flight at once.
__device__ __forceinline__ void stage_rows(float* s_tile, int pitch, const float* fresh,
                                           const float* ctx, const int32_t* fresh_of, int t0,
                                           int n, int h, int D, int hid) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nwarps = blockDim.x >> 5;
    // the tile's fresh-row map in one coalesced load per warp (n <= 32)
    const int fr_lane = lane < n ? __ldg(fresh_of + t0 + lane) : -1;
    for (int t = warp; t < n; t += nwarps) {
        const int fr = __shfl_sync(0xffffffffu, fr_lane, t);
        const float* src = (fr >= 0 ? fresh + (size_t)fr * hid : ctx + (size_t)(t0 + t) * hid) + h * D;
        float* dst = s_tile + t * pitch;
        for (int d = 2 * lane; d < D; d += 64) cp_async_8(dst + d, src + d);
    }
    cp_async_commit();
    cp_async_wait<0>();
}



__device__ __forceinline__ void attend_row(const float* __restrict__ q_row,
                                           const float* __restrict__ k_fresh,
                                           const float* __restrict__ v_fresh,
                                           const float* __restrict__ ctx_k,
                                           const float* __restrict__ ctx_v,
                                           const int32_t* __restrict__ fresh_of, int tn, int h,
                                           int H, int D, float scale, float* __restrict__ mix_row,
                                           float* s_score, float* s_tile) {
    __shared__ float s_q[256];
    __shared__ float s_red[32];
    __shared__ double s_redd[32];
    const int hid = H * D;
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int pitch = attn_pitch(D);
    for (int d = tid; d < D; d += nthr) s_q[d] = q_row[h * D + d];
    // stage rows [t0, t0 + kAttnTile) of the K or V plane (fresh or cached)
    auto stage = [&](const float* fresh, const float* ctx, int t0) {
        stage_rows(s_tile, pitch, fresh, ctx, fresh_of, t0, min(kAttnTile, tn - t0), h, D, hid);
    };

    float mx = -INFINITY;
    for (int t0 = 0; t0 < tn; t0 += kAttnTile) {
        __syncthreads();                   // s_q ready / previous tile consumed
        stage(k_fresh, ctx_k, t0);
        __syncthreads();
        const int n = min(kAttnTile, tn - t0);
        for (int t = tid; t < n; t += nthr) {
            const float* kr = s_tile + t * pitch;
            float acc = 0.f;
            for (int d = 0; d < D; ++d) acc = fmaf(s_q[d], kr[d], acc);
            const float sc = acc * scale;
            s_score[t0 + t] = sc;
            mx = fmaxf(mx, sc);
        }
    }
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((tid & 31) == 0) s_red[tid >> 5] = mx;
    __syncthreads();
    if (tid == 0) {
        float m = -INFINITY;
        for (int w = 0; w < (nthr >> 5); ++w) m = fmaxf(m, s_red[w]);
        s_red[0] = m;
    }
    __syncthreads();
    mx = s_red[0];
    double sum = 0.0;
    for (int t = tid; t < tn; t += nthr) {
        const float e = expf(s_score[t] - mx);
        s_score[t] = e;
        sum += (double)e;
    }
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    __syncthreads();
    if ((tid & 31) == 0) s_redd[tid >> 5] = sum;
    __syncthreads();
    if (tid == 0) {
        double s = 0.0;
        for (int w = 0; w < (nthr >> 5); ++w) s += s_redd[w];
        s_redd[0] = s;
    }
    __syncthreads();
    const float total = (float)s_redd[0];
    for (int t = tid; t < tn; t += nthr) s_score[t] = s_score[t] / total;
    double acc0 = 0.0, acc1 = 0.0;         // output elements d = tid, tid + nthr (D <= 256)
    const int d0 = tid, d1 = tid + nthr;
    for (int t0 = 0; t0 < tn; t0 += kAttnTile) {
        __syncthreads();                   // probabilities written / previous tile consumed
        stage(v_fresh, ctx_v, t0);
        __syncthreads();
        const int n = min(kAttnTile, tn - t0);
        if (d0 < D)
            for (int t = 0; t < n; ++t)
                acc0 += (double)s_score[t0 + t] * (double)s_tile[t * pitch + d0];
        if (d1 < D)
            for (int t = 0; t < n; ++t)
                acc1 += (double)s_score[t0 + t] * (double)s_tile[t * pitch + d1];
    }
    if (d0 < D) mix_row[h * D + d0] = (float)acc0;
    if (d1 < D) mix_row[h * D + d1] = (float)acc1;
}

// One CTA per (fixed row f, head h) of one context.
__global__ void __launch_bounds__(128)
    attention_kernel(const float* __restrict__ q, const float* __restrict__ k_fresh,
                     const float* __restrict__ v_fresh, const float* __restrict__ ctx_k,
                     const float* __restrict__ ctx_v, const int32_t* __restrict__ fresh_of,
                     const int64_t* __restrict__ fix_idx, int H, int D, float scale,
                     float* __restrict__ mix) {
    extern __shared__ float s_dyn[];      // [tile (kAttnTile x pitch) | scores]
    const int f = blockIdx.x, h = blockIdx.y;
    const size_t hid = (size_t)H * D;
    attend_row(q + f * hid, k_fresh, v_fresh, ctx_k, ctx_v, fresh_of, (int)fix_idx[f] + 1, h, H,
               D, scale, mix + f * hid, s_dyn + kAttnTile * attn_pitch(D), s_dyn);
}

// Several members' fixed rows in one launch (grouped recovery): row r
// belongs to the member whose [row0, row0 + n_rows) holds it; its fresh rows
// are the member's slice of the concatenated fresh planes.
__global__ void __launch_bounds__(128)
    attention_many_kernel(const float* __restrict__ q, const float* __restrict__ k_fresh,
                          const float* __restrict__ v_fresh,
                          const tdkv_attn_member* __restrict__ members, int n_members, int layer,
                          int H, int D, float scale, float* __restrict__ mix) {
    extern __shared__ float s_dyn[];      // [tile (kAttnTile x pitch) | scores]
    const int r = blockIdx.x, h = blockIdx.y;
    int lo = 0, hi = n_members - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (members[mid].row0 <= r) lo = mid; else hi = mid - 1;
    }
    const tdkv_attn_member m = members[lo];
    const size_t hid = (size_t)H * D;
    const size_t lofs = (size_t)layer * m.ctx_layer_stride;
    attend_row(q + r * hid, k_fresh + (size_t)m.row0 * hid, v_fresh + (size_t)m.row0 * hid,
               m.ctx_k + lofs, m.ctx_v + lofs, m.fresh_of, (int)m.fix_idx[r - m.row0] + 1, h, H,
               D, scale, mix + r * hid, s_dyn + kAttnTile * attn_pitch(D), s_dyn);
}

// Query-tiled form of attention_many_kernel: one CTA per (4 * QW consecutive
// fixed rows of one member, head).  Every staged key/value tile serves all
// 4 * QW queries, so staging and index work are amortized that many times and
// each thread carries several independent accumulators.  Warp w owns queries
// w, w + 4, ... (scores, max, softmax); thread i owns outputs (q, d) for
// q * D + d = i, i + 128, ... .  Scores are sequential fmaf chains over d and
// outputs sequential float64 sums over t, as in attend_row.
template <int QW>   // queries per warp; kQ = 4 * QW rows per CTA
__global__ void __launch_bounds__(128)
    attention_tiles_kernel(const float* __restrict__ q, const float* __restrict__ k_fresh,
                           const float* __restrict__ v_fresh,
                           const tdkv_attn_member* __restrict__ members, int n_members, int layer,
                           int H, int D, float scale, int max_tokens, float* __restrict__ mix) {
    constexpr int kAttnQ = 4 * QW;
    extern __shared__ float s_dyn[];   // [tile kAttnTile x pitch | q kAttnQ x D | p kAttnQ x max_tokens]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int h = blockIdx.y;
    int lo = 0, hi = n_members - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (members[mid].tile0 <= (int)blockIdx.x) lo = mid; else hi = mid - 1;
    }
    const tdkv_attn_member m = members[lo];
    const int r0 = ((int)blockIdx.x - m.tile0) * kAttnQ;          // member-local first row
    const int nq = min(kAttnQ, m.n_rows - r0);
    const int hid = H * D;
    const int pitch = attn_pitch(D);
    float* s_tile = s_dyn;
    float* s_q = s_tile + kAttnTile * pitch;
    float* s_p = s_q + kAttnQ * D;
    const size_t lofs = (size_t)layer * m.ctx_layer_stride;
    const float* ctx_k = m.ctx_k + lofs;
    const float* ctx_v = m.ctx_v + lofs;
    const float* kf = k_fresh + (size_t)m.row0 * hid;
    const float* vf = v_fresh + (size_t)m.row0 * hid;
    const int32_t* fresh_of = m.fresh_of;
    int tnq[QW];                                                 // this warp's queries' lengths
#pragma unroll
    for (int j = 0; j < QW; ++j) {
        const int qi = warp + 4 * j;
        tnq[j] = qi < nq ? (int)m.fix_idx[r0 + qi] + 1 : 0;
    }
    const int tn = (int)m.fix_idx[r0 + nq - 1] + 1;              // rows ascend: the longest
    for (int i = tid; i < nq * D; i += blockDim.x) {
        const int qi = i / D, d = i - qi * D;
        s_q[i] = q[(size_t)(m.row0 + r0 + qi) * hid + h * D + d];
    }
    auto stage = [&](const float* fresh, const float* ctx, int t0, int n) {
        stage_rows(s_tile, pitch, fresh, ctx, fresh_of, t0, n, h, D, hid);
    };
    // scores
    float mx[QW];
#pragma unroll
    for (int j = 0; j < QW; ++j) mx[j] = -INFINITY;
    for (int t0 = 0; t0 < tn; t0 += kAttnTile) {
        const int n = min(kAttnTile, tn - t0);
        __syncthreads();
        stage(kf, ctx_k, t0, n);
        __syncthreads();
        if (lane < n) {
            // the warp's queries advance together over d: each key element is
            // read once and the QW chains are independent (each chain is still
            // one sequential fmaf over d)
            const float* kr = s_tile + lane * pitch;
            float acc[QW];
#pragma unroll
            for (int j = 0; j < QW; ++j) acc[j] = 0.f;
            for (int d = 0; d < D; ++d) {
                const float kv = kr[d];
#pragma unroll
                for (int j = 0; j < QW; ++j) acc[j] = fmaf(s_q[(warp + 4 * j) * D + d], kv, acc[j]);
            }
#pragma unroll
            for (int j = 0; j < QW; ++j) {
                const int qi = warp + 4 * j;
                if (t0 + lane < tnq[j]) {
                    const float sc = acc[j] * scale;
                    s_p[qi * max_tokens + t0 + lane] = sc;
                    mx[j] = fmaxf(mx[j], sc);
                }
            }
        }
    }
    // softmax of this warp's queries
#pragma unroll
    for (int j = 0; j < QW; ++j) {
        const int qi = warp + 4 * j;
        if (qi >= nq) continue;
        float mj = mx[j];
        for (int o = 16; o > 0; o >>= 1) mj = fmaxf(mj, __shfl_xor_sync(0xffffffffu, mj, o));
        float* p = s_p + qi * max_tokens;
        double sum = 0.0;
        for (int t = lane; t < tnq[j]; t += 32) {
            const float e = expf(p[t] - mj);
            p[t] = e;
            sum += (double)e;
        }
        for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        const float total = (float)sum;
        for (int t = lane; t < tnq[j]; t += 32) p[t] = p[t] / total;
    }
    // outputs
    // thread outputs i = tid + 128 k < kAttnQ * D (D <= 128: at most kAttnQ)
    double acc[kAttnQ];
#pragma unroll
    for (int k = 0; k < kAttnQ; ++k) acc[k] = 0.0;
    for (int t0 = 0; t0 < tn; t0 += kAttnTile) {
        const int n = min(kAttnTile, tn - t0);
        __syncthreads();
        stage(vf, ctx_v, t0, n);
        __syncthreads();
#pragma unroll
        for (int k = 0; k < kAttnQ; ++k) {
            const int i = tid + k * 128;
            if (i >= nq * D) break;
            const int qi = i / D, d = i - qi * D;
            const int tq = (int)m.fix_idx[r0 + qi] + 1;
            const float* p = s_p + qi * max_tokens + t0;
            const int nn = min(n, tq - t0);
            for (int t = 0; t < nn; ++t) acc[k] += (double)p[t] * (double)s_tile[t * pitch + d];
        }
    }
#pragma unroll
    for (int k = 0; k < kAttnQ; ++k) {
        const int i = tid + k * 128;
        if (i >= nq * D) break;
        const int qi = i / D, d = i - qi * D;
        mix[(size_t)(m.row0 + r0 + qi) * hid + h * D + d] = (float)acc[k];
    }
}

// Online-softmax form of the query-tiled attention (head_dim <= 128): one CTA
// per (32 fixed rows of one member, head) streams the member's keys/values
// once in 32-token tiles (K and V staged together), keeping a running max and
// sum per query and rescaling its float64 output accumulators per tile, so
// no full score row is stored and every staged tile serves 32 queries.
// Warp w owns queries w, w + 4, ..., (QW per warp); thread i owns outputs
// (q, d) for q * D + d = i + 128 k.
template <int QW, int DMAX>   // DMAX: largest head_dim served (64 or 128)
__global__ void __launch_bounds__(128)
    attention_online_kernel(const float* __restrict__ q, const float* __restrict__ k_fresh,
                            const float* __restrict__ v_fresh,
                            const tdkv_attn_member* __restrict__ members, int n_members,
                            int layer, int H, int D, float scale, float* __restrict__ mix) {
    constexpr int kQ = 4 * QW;
    constexpr int kOut = kQ * DMAX / 128;                       // outputs per thread (D <= DMAX)
    extern __shared__ float s_dyn[];   // [K tile | V tile | q kQ x D | p kQ x kAttnTile | corr kQ | l kQ]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int h = blockIdx.y;
    int lo = 0, hi = n_members - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (members[mid].tile0 <= (int)blockIdx.x) lo = mid; else hi = mid - 1;
    }
    const tdkv_attn_member m = members[lo];
    const int r0 = ((int)blockIdx.x - m.tile0) * kQ;
    const int nq = min(kQ, m.n_rows - r0);
    const int hid = H * D;
    const int pitch = attn_pitch(D);
    float* s_k = s_dyn;
    float* s_v = s_k + kAttnTile * pitch;
    float* s_q = s_v + kAttnTile * pitch;
    float* s_pt = s_q + kQ * D;
    float* s_corr = s_pt + kQ * kAttnTile;
    float* s_l = s_corr + kQ;
    const size_t lofs = (size_t)layer * m.ctx_layer_stride;
    const float* ctx_k = m.ctx_k + lofs;
    const float* ctx_v = m.ctx_v + lofs;
    const float* kf = k_fresh + (size_t)m.row0 * hid;
    const float* vf = v_fresh + (size_t)m.row0 * hid;
    for (int i = tid; i < nq * D; i += blockDim.x) {
        const int qi = i / D, d = i - qi * D;
        s_q[i] = q[(size_t)(m.row0 + r0 + qi) * hid + h * D + d];
    }
    int tnq[QW];
    float mrun[QW];
    double lrun[QW];
#pragma unroll
    for (int j = 0; j < QW; ++j) {
        const int qi = warp + 4 * j;
        tnq[j] = qi < nq ? (int)m.fix_idx[r0 + qi] + 1 : 0;
        mrun[j] = -INFINITY;
        lrun[j] = 0.0;
    }
    const int tn = (int)m.fix_idx[r0 + nq - 1] + 1;
    double acc[kOut];
#pragma unroll
    for (int k = 0; k < kOut; ++k) acc[k] = 0.0;
    for (int t0 = 0; t0 < tn; t0 += kAttnTile) {
        const int n = min(kAttnTile, tn - t0);
        __syncthreads();                                     // previous tile consumed
        stage_rows(s_k, pitch, kf, ctx_k, m.fresh_of, t0, n, h, D, hid);
        stage_rows(s_v, pitch, vf, ctx_v, m.fresh_of, t0, n, h, D, hid);
        __syncthreads();
        float sc[QW];
        {
            float a[QW];
#pragma unroll
            for (int j = 0; j < QW; ++j) a[j] = 0.f;
            if (lane < n) {
                const float* kr = s_k + lane * pitch;
                for (int d = 0; d < D; ++d) {
                    const float kv = kr[d];
#pragma unroll
                    for (int j = 0; j < QW; ++j) a[j] = fmaf(s_q[(warp + 4 * j) * D + d], kv, a[j]);
                }
            }
#pragma unroll
            for (int j = 0; j < QW; ++j)
                sc[j] = (lane < n && t0 + lane < tnq[j]) ? a[j] * scale : -INFINITY;
        }
#pragma unroll
        for (int j = 0; j < QW; ++j) {
            const int qi = warp + 4 * j;
            float tmax = sc[j];
            for (int o = 16; o > 0; o >>= 1) tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, o));
            const float mnew = fmaxf(mrun[j], tmax);
            const float corr = (mrun[j] == -INFINITY) ? 1.f : expf(mrun[j] - mnew);
            const float p = sc[j] == -INFINITY ? 0.f : expf(sc[j] - mnew);
            double ps = (double)p;
            for (int o = 16; o > 0; o >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, o);
            lrun[j] = lrun[j] * (double)corr + ps;
            mrun[j] = mnew;
            s_pt[qi * kAttnTile + lane] = p;
            if (lane == 0) s_corr[qi] = corr;
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < kOut; ++k) {
            const int i = tid + k * 128;
            if (i >= nq * D) break;
            const int qi = i / D, d = i - qi * D;
            const float* pq = s_pt + qi * kAttnTile;
            double a = acc[k] * (double)s_corr[qi];
            for (int t = 0; t < n; ++t) a += (double)pq[t] * (double)s_v[t * pitch + d];
            acc[k] = a;
        }
    }
#pragma unroll
    for (int j = 0; j < QW; ++j)
        if (lane == 0 && warp + 4 * j < nq) s_l[warp + 4 * j] = (float)lrun[j];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kOut; ++k) {
        const int i = tid + k * 128;
        if (i >= nq * D) break;
        const int qi = i / D, d = i - qi * D;
        mix[(size_t)(m.row0 + r0 + qi) * hid + h * D + d] = (float)(acc[k] / (double)s_l[qi]);
    }
}

}  // namespace tdkv

using namespace tdkv;

extern "C" int32_t tdkv_qkv_rope(const float* d_qkv, const void* d_table, int32_t n_rows,
                                 int32_t num_heads, int32_t head_dim, float* d_q, float* d_k,
                                 float* d_v, void* stream) {
    if (n_rows < 0 || num_heads <= 0 || head_dim <= 0 || (head_dim & 1))
        return set_error(TDKV_EINVAL, "tdkv_qkv_rope: bad geometry");
    if (n_rows == 0) return TDKV_OK;
    if (!d_qkv || !d_table || !d_q || !d_k || !d_v)
        return set_error(TDKV_EINVAL, "tdkv_qkv_rope: null pointer");
    const long long pairs = (long long)n_rows * num_heads * head_dim / 2;
    long long grid = (pairs + 255) / 256;
    if (grid > sm_count() * 8) grid = sm_count() * 8;
    qkv_rope_kernel<<<(unsigned)grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        d_qkv, static_cast<const double2*>(d_table), n_rows, num_heads, head_dim, d_q, d_k, d_v);
    count_launch();
    return check_launch("tdkv_qkv_rope");
}

extern "C" int32_t tdkv_attention(const float* d_q, const float* d_k_fresh, const float* d_v_fresh,
                                  const float* d_ctx_k, const float* d_ctx_v,
                                  const int32_t* d_fresh_of, const int64_t* d_fix_idx,
                                  int32_t n_fix, int32_t num_tokens, int32_t num_heads,
                                  int32_t head_dim, float scale, float* d_mix, void* stream) {
    if (n_fix < 0 || num_tokens <= 0 || num_heads <= 0 || head_dim <= 0 || head_dim > 256)
        return set_error(TDKV_EINVAL, "tdkv_attention: bad geometry");
    if (n_fix == 0) return TDKV_OK;
    const size_t smem = ((size_t)num_tokens + (size_t)kAttnTile * attn_pitch(head_dim)) * sizeof(float);
    if (smem > 200 * 1024)
        return set_error(TDKV_EUNSUPPORTED, "tdkv_attention: %d tokens exceed shared memory",
                         num_tokens);
    if (cudaFuncSetAttribute(attention_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
        return check_launch("tdkv_attention: cudaFuncSetAttribute");
    dim3 grid(n_fix, num_heads);
    attention_kernel<<<grid, 128, smem, static_cast<cudaStream_t>(stream)>>>(
        d_q, d_k_fresh, d_v_fresh, d_ctx_k, d_ctx_v, d_fresh_of, d_fix_idx, num_heads, head_dim,
        scale, d_mix);
    count_launch();
    return check_launch("tdkv_attention");
}

extern "C" int32_t tdkv_attention_many(const float* d_q, const float* d_k_fresh,
                                       const float* d_v_fresh, const tdkv_attn_member* d_members,
                                       int32_t n_members, int32_t layer, int32_t total_rows,
                                       int32_t n_tiles, int32_t rows_per_tile,
                                       int32_t max_tokens, int32_t num_heads,
                                       int32_t head_dim, float scale, float* d_mix,
                                       void* stream) {
    if (n_members < 0 || total_rows < 0 || n_tiles < 0 || layer < 0 || max_tokens <= 0 ||
        num_heads <= 0 || head_dim <= 0 || head_dim > 256)
        return set_error(TDKV_EINVAL, "tdkv_attention_many: bad geometry");
    if (n_members == 0 || total_rows == 0) return TDKV_OK;
    if (!d_q || !d_k_fresh || !d_v_fresh || !d_members || !d_mix)
        return set_error(TDKV_EINVAL, "tdkv_attention_many: null pointer");
    const size_t smem = ((size_t)max_tokens + (size_t)kAttnTile * attn_pitch(head_dim)) * sizeof(float);
    if (smem > 200 * 1024)
        return set_error(TDKV_EUNSUPPORTED, "tdkv_attention_many: %d tokens exceed shared memory",
                         max_tokens);
    if (n_tiles > 0 && rows_per_tile == 16) {
        if (head_dim > 128)
            return set_error(TDKV_EINVAL, "tdkv_attention_many: 16-row tiles need head_dim <= 128");
        const int pitch = attn_pitch(head_dim);
        const size_t osmem = ((size_t)2 * kAttnTile * pitch + (size_t)16 * head_dim +
                              (size_t)16 * kAttnTile + 2 * 16) * sizeof(float);
        auto kern = head_dim <= 64 ? attention_online_kernel<4, 64> : attention_online_kernel<4, 128>;
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)osmem) !=
            cudaSuccess)
            return check_launch("tdkv_attention_many: cudaFuncSetAttribute");
        dim3 ogrid(n_tiles, num_heads);
        kern<<<ogrid, 128, osmem, static_cast<cudaStream_t>(stream)>>>(
            d_q, d_k_fresh, d_v_fresh, d_members, n_members, layer, num_heads, head_dim, scale,
            d_mix);
        count_launch();
        return check_launch("tdkv_attention_many");
    }
    if (n_tiles > 0) {
        if (rows_per_tile != 8 || head_dim > 128)
            return set_error(TDKV_EINVAL,
                             "tdkv_attention_many: tiles of %d rows with head_dim %d (8 or 16 "
                             "rows, head_dim <= 128)",
                             rows_per_tile, head_dim);
        const int kq = 8;
        const size_t tsmem = ((size_t)kAttnTile * attn_pitch(head_dim) + (size_t)kq * head_dim +
                              (size_t)kq * max_tokens) * sizeof(float);
        if (tsmem > 200 * 1024)
            return set_error(TDKV_EUNSUPPORTED,
                             "tdkv_attention_many: %d tokens exceed shared memory", max_tokens);
        auto kern = attention_tiles_kernel<2>;
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)tsmem) != cudaSuccess)
            return check_launch("tdkv_attention_many: cudaFuncSetAttribute");
        dim3 tgrid(n_tiles, num_heads);
        kern<<<tgrid, 128, tsmem, static_cast<cudaStream_t>(stream)>>>(
            d_q, d_k_fresh, d_v_fresh, d_members, n_members, layer, num_heads, head_dim, scale,
            max_tokens, d_mix);
        count_launch();
        return check_launch("tdkv_attention_many");
    }
    if (cudaFuncSetAttribute(attention_many_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
        return check_launch("tdkv_attention_many: cudaFuncSetAttribute");
    dim3 grid(total_rows, num_heads);
    attention_many_kernel<<<grid, 128, smem, static_cast<cudaStream_t>(stream)>>>(
        d_q, d_k_fresh, d_v_fresh, d_members, n_members, layer, num_heads, head_dim, scale, d_mix);
    count_launch();
    return check_launch("tdkv_attention_many");
}
