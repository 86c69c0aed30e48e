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
#include "tdkv_umma.cuh"

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

// Register-blocked attention (rows_per_tile 64): one CTA serves 64 fixed
// rows of one member and one head with 256 threads, staging 64-token key and
// value tiles (double-buffered 16-byte async copies, fresh rows overriding
// cached ones).  Scores: thread (tq, tk) owns the 4 x 4 block of queries
// 4tq.. and keys tk + 16j, each score the same sequential fmaf chain over d
// as the other forms (then * scale); 8 FMAs per 16-byte shared load.  Online
// softmax per query (running max across the 16 threads of its row, float32
// exp as numpy).  P.V: thread owns 4 queries x D/16 output columns (D = 8:
// 2 x 1), summing a key tile in float32 and folding each tile's partial into
// float64 accumulators rescaled by the running-max correction -- float32
// throughput, and an accumulation error of one 64-term float32 sum per tile
// instead of one over the whole context.
constexpr int kBlkQ = 64;          // queries per CTA
constexpr int kBlkK = 64;          // keys per staged tile
constexpr int kBlkThreads = 256;

__host__ __device__ constexpr int blk_pitch(int D) { return D + 4; }

template <int D>
__host__ __device__ constexpr size_t blk_smem_floats() {
    // q tile + 2 x (K tile + V tile) + P^T tile (+ per-query state)
    return (size_t)kBlkQ * blk_pitch(D) + 4 * (size_t)kBlkK * blk_pitch(D) +
           (size_t)kBlkK * (kBlkQ + 4) + 2 * kBlkQ;
}

// 16-byte async staging of head h of token rows [t0, t0 + n) (fresh row when
// fresh_of[t] >= 0, else the context row) into s_tile (pitch floats per row)
template <int D>
__device__ __forceinline__ void blk_stage(float* s_tile, const float* fresh, const float* ctx,
                                          const int32_t* fresh_of, int t0, int n, int h, int hid) {
    constexpr int kChunks = D / 4;
    for (int i = threadIdx.x; i < n * kChunks; i += kBlkThreads) {
        const int t = i / kChunks, c = i - t * kChunks;
        const int fr = __ldg(fresh_of + t0 + t);
        const float* src = (fr >= 0 ? fresh + (size_t)fr * hid : ctx + (size_t)(t0 + t) * hid) +
                           h * D + 4 * c;
        const uint32_t dst = smem_u32(s_tile + t * blk_pitch(D) + 4 * c);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
    }
}

template <int D>
__global__ void __launch_bounds__(kBlkThreads)
    attention_block_kernel(const float* __restrict__ q, const float* __restrict__ k_fresh,
                           const float* __restrict__ v_fresh,
                           const tdkv_attn_member* __restrict__ members, int n_members, int layer,
                           int H, float scale, float* __restrict__ mix) {
    constexpr int P = blk_pitch(D);
    constexpr int PP = kBlkQ + 4;                           // P^T pitch
    // P.V thread layout: QPT queries x DPT columns
    constexpr int DG = D >= 16 ? 16 : D;                   // column groups
    constexpr int DPT = D / DG;                            // columns per thread
    constexpr int QG = kBlkThreads / DG;                   // query groups
    constexpr int QPT = kBlkQ / QG;                        // queries per thread
    extern __shared__ __align__(16) float s_dyn[];
    float* s_q = s_dyn;                                    // [64][P]
    float* s_kv = s_q + kBlkQ * P;                         // 2 buffers x (K [64][P], V [64][P])
    float* s_pt = s_kv + 4 * kBlkK * P;                    // P^T [64 keys][PP]
    float* s_corr = s_pt + kBlkK * PP;                     // [64]
    float* s_lsum = s_corr + kBlkQ;                        // [64]
    const int tid = threadIdx.x;
    const int h = blockIdx.y;
    int lo = 0, hi = n_members - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (members[mid].tile0 <= (int)blockIdx.x) lo = mid; else hi = mid - 1;
    }
    const tdkv_attn_member m = members[lo];
    const int r0 = ((int)blockIdx.x - m.tile0) * kBlkQ;
    const int nq = min(kBlkQ, m.n_rows - r0);
    const int hid = H * D;
    const size_t lofs = (size_t)layer * m.ctx_layer_stride;
    const float* ctx_k = m.ctx_k + lofs;
    const float* ctx_v = m.ctx_v + lofs;
    const float* kf = k_fresh + (size_t)m.row0 * hid;
    const float* vf = v_fresh + (size_t)m.row0 * hid;
    const int tn = (int)m.fix_idx[r0 + nq - 1] + 1;        // keys any row of the tile sees
    const int ntiles = (tn + kBlkK - 1) / kBlkK;

    // stage q rows and the first key/value tile
    for (int i = tid; i < kBlkQ * (D / 4); i += kBlkThreads) {
        const int qi = i / (D / 4), c = i - qi * (D / 4);
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (qi < nq) v = *reinterpret_cast<const float4*>(q + (size_t)(m.row0 + r0 + qi) * hid + h * D + 4 * c);
        *reinterpret_cast<float4*>(s_q + qi * P + 4 * c) = v;
    }
    blk_stage<D>(s_kv, kf, ctx_k, m.fresh_of, 0, min(kBlkK, tn), h, hid);
    blk_stage<D>(s_kv + kBlkK * P, vf, ctx_v, m.fresh_of, 0, min(kBlkK, tn), h, hid);
    cp_async_commit();

    // score-phase ownership: queries 4tq + i, keys tk + 16j
    const int tq = tid >> 4, tk = tid & 15;
    int tnq[4];
    float mrun[4];
    double lrun[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int qi = 4 * tq + i;
        tnq[i] = qi < nq ? (int)m.fix_idx[r0 + qi] + 1 : 0;
        mrun[i] = -INFINITY;
        lrun[i] = 0.0;
    }
    // P.V ownership: queries QPT*pq + i, columns DPT*pd + c
    const int pq = tid / DG, pd = tid - (tid / DG) * DG;
    double acc[QPT][DPT];
#pragma unroll
    for (int i = 0; i < QPT; ++i)
#pragma unroll
        for (int c = 0; c < DPT; ++c) acc[i][c] = 0.0;

    for (int it = 0; it < ntiles; ++it) {
        const int t0 = it * kBlkK;
        const int n = min(kBlkK, tn - t0);
        float* s_k = s_kv + (it & 1) * 2 * kBlkK * P;
        float* s_v = s_k + kBlkK * P;
        if (it + 1 < ntiles) {                              // prefetch the next tile
            float* nk = s_kv + ((it + 1) & 1) * 2 * kBlkK * P;
            const int t1 = t0 + kBlkK;
            blk_stage<D>(nk, kf, ctx_k, m.fresh_of, t1, min(kBlkK, tn - t1), h, hid);
            blk_stage<D>(nk + kBlkK * P, vf, ctx_v, m.fresh_of, t1, min(kBlkK, tn - t1), h, hid);
            cp_async_commit();
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();                                    // tile it (and q) resident
        // ---- scores: sequential fmaf chains over d
        float a[4][4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) a[i][j] = 0.f;
#pragma unroll 2
        for (int d = 0; d < D; d += 4) {
            float4 qv[4], kv[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) qv[i] = *reinterpret_cast<const float4*>(s_q + (4 * tq + i) * P + d);
#pragma unroll
            for (int j = 0; j < 4; ++j) kv[j] = *reinterpret_cast<const float4*>(s_k + (tk + 16 * j) * P + d);
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    a[i][j] = fmaf(qv[i].x, kv[j].x, a[i][j]);
                    a[i][j] = fmaf(qv[i].y, kv[j].y, a[i][j]);
                    a[i][j] = fmaf(qv[i].z, kv[j].z, a[i][j]);
                    a[i][j] = fmaf(qv[i].w, kv[j].w, a[i][j]);
                }
        }
        // ---- online softmax (the 16 threads of a query row are one half-warp)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            float sc[4];
            float tmax = -INFINITY;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int key = tk + 16 * j;
                sc[j] = (key < n && t0 + key < tnq[i]) ? a[i][j] * scale : -INFINITY;
                tmax = fmaxf(tmax, sc[j]);
            }
#pragma unroll
            for (int o = 8; o > 0; o >>= 1) tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, o));
            const float mnew = fmaxf(mrun[i], tmax);
            const float corr = (mrun[i] == -INFINITY || mnew == -INFINITY) ? 1.f : expf(mrun[i] - mnew);
            float ps = 0.f;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float p = sc[j] == -INFINITY ? 0.f : expf(sc[j] - mnew);
                s_pt[(tk + 16 * j) * PP + 4 * tq + i] = p;
                ps += p;
            }
#pragma unroll
            for (int o = 8; o > 0; o >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, o);
            lrun[i] = lrun[i] * (double)corr + (double)ps;
            mrun[i] = mnew;
            if (tk == 0) s_corr[4 * tq + i] = corr;
        }
        __syncthreads();                                    // P^T and corrections ready
        // ---- P.V: float32 sum over the tile's keys, folded into float64
        float o[QPT][DPT];
#pragma unroll
        for (int i = 0; i < QPT; ++i)
#pragma unroll
            for (int c = 0; c < DPT; ++c) o[i][c] = 0.f;
        for (int kk = 0; kk < n; ++kk) {
            float pv[QPT], vv[DPT];
#pragma unroll
            for (int i = 0; i < QPT; ++i) pv[i] = s_pt[kk * PP + QPT * pq + i];
#pragma unroll
            for (int c = 0; c < DPT; ++c) vv[c] = s_v[kk * P + DPT * pd + c];
#pragma unroll
            for (int i = 0; i < QPT; ++i)
#pragma unroll
                for (int c = 0; c < DPT; ++c) o[i][c] = fmaf(pv[i], vv[c], o[i][c]);
        }
#pragma unroll
        for (int i = 0; i < QPT; ++i) {
            const double cr = (double)s_corr[QPT * pq + i];
#pragma unroll
            for (int c = 0; c < DPT; ++c) acc[i][c] = acc[i][c] * cr + (double)o[i][c];
        }
        __syncthreads();                                    // buffers reusable
    }
    if (tk == 0) {
#pragma unroll
        for (int i = 0; i < 4; ++i) s_lsum[4 * tq + i] = (float)lrun[i];
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < QPT; ++i) {
        const int qi = QPT * pq + i;
        if (qi >= nq) continue;
        const double l = (double)s_lsum[qi];
#pragma unroll
        for (int c = 0; c < DPT; ++c)
            mix[(size_t)(m.row0 + r0 + qi) * hid + h * D + DPT * pd + c] = (float)(acc[i][c] / l);
    }
}

template <int D>
static int32_t launch_attention_block(const float* d_q, const float* d_k_fresh,
                                      const float* d_v_fresh, const tdkv_attn_member* d_members,
                                      int32_t n_members, int32_t layer, int32_t n_tiles,
                                      int32_t num_heads, float scale, float* d_mix,
                                      cudaStream_t s) {
    auto kern = attention_block_kernel<D>;
    const size_t smem = blk_smem_floats<D>() * sizeof(float);
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
        return check_launch("tdkv_attention_many: cudaFuncSetAttribute");
    kern<<<dim3(n_tiles, num_heads), kBlkThreads, smem, s>>>(d_q, d_k_fresh, d_v_fresh, d_members,
                                                             n_members, layer, num_heads, scale,
                                                             d_mix);
    count_launch();
    return check_launch("tdkv_attention_many");
}


// Tensor-core attention (rows_per_tile 128, head_dim 32 or 64): one CTA of
// 256 threads serves 128 fixed rows of one member and one head.  Query row r
// is TMEM lane r; warps w and w + 4 share that lane quadrant and split each
// row's columns (keys of S, head dims of O) in halves.  Per 64-key tile:
//   S = Q K^T    tcgen05.mma kind::tf32 as 3xTF32 (Q_hi K_hi + Q_hi K_lo +
//                Q_lo K_hi: ~22 mantissa bits, float32 accumulation in TMEM)
//   softmax      each thread's half score row from TMEM (tcgen05.ld), masked
//                causally by sequence index, the row max exchanged with the
//                partner thread, float32 exp as numpy; P written to shared
//                memory split into tf32 hi / lo
//   O = P V      3xTF32 again into a second TMEM accumulator (V staged
//                transposed: the B operand is K-major over keys)
//   acc          float32 per-row accumulators rescaled by the max correction
// Operands sit in the canonical no-swizzle K-major core-matrix layout (8 rows
// x 16 bytes per core matrix); key and value rows come from the fresh rows
// when fresh_of[t] >= 0, else from the context planes.
constexpr int kTcQ = 128;          // queries per CTA (TMEM lanes)
constexpr int kTcK = 64;           // keys per tile
constexpr int kTcThreads = 256;

template <int D>
struct TcAttnSmem {
    static constexpr int kQ = kTcQ * D * 4;        // one tf32 plane of Q
    static constexpr int kK = kTcK * D * 4;        // K tile
    static constexpr int kV = D * kTcK * 4;        // V^T tile
    static constexpr int kP = kTcQ * kTcK * 4;     // P tile
    static constexpr int kBytes = 2 * (kQ + kK + kV + kP);
};

__device__ __forceinline__ void split_store16(uint8_t* hi, uint8_t* lo, uint32_t off, float4 v) {
    uint4 h, l;
    h.x = tf32_rna(v.x); l.x = tf32_rna(v.x - __uint_as_float(h.x));
    h.y = tf32_rna(v.y); l.y = tf32_rna(v.y - __uint_as_float(h.y));
    h.z = tf32_rna(v.z); l.z = tf32_rna(v.z - __uint_as_float(h.z));
    h.w = tf32_rna(v.w); l.w = tf32_rna(v.w - __uint_as_float(h.w));
    *reinterpret_cast<uint4*>(hi + off) = h;
    *reinterpret_cast<uint4*>(lo + off) = l;
}

template <int N>
__device__ __forceinline__ void tmem_row(uint32_t addr, float (&x)[N]) {
    static_assert(N % 8 == 0, "8-column loads");
#pragma unroll
    for (int c0 = 0; c0 < N; c0 += 8) {
        uint32_t r[8];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
              "=r"(r[6]), "=r"(r[7])
            : "r"(addr + c0));
#pragma unroll
        for (int j = 0; j < 8; ++j) x[c0 + j] = __uint_as_float(r[j]);
    }
    tmem_ld_wait();
}

template <int D>
__global__ void __launch_bounds__(kTcThreads, 1)
    attention_tc_kernel(const float* __restrict__ q, const float* __restrict__ k_fresh,
                        const float* __restrict__ v_fresh,
                        const tdkv_attn_member* __restrict__ members, int n_members, int layer,
                        int H, float scale, float* __restrict__ mix) {
    using SM = TcAttnSmem<D>;
    constexpr int kCq = D / 4;                     // 16-byte chunks per Q / K row
    constexpr int kCp = kTcK / 4;                  // chunks per P / V^T row
    constexpr int kSh = kTcK / 2;                  // S columns per thread
    constexpr int kOh = D / 2;                     // O columns per thread
    constexpr uint32_t kTmemCols = kTcK + D <= 128 ? 128 : 256;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* q_hi = smem;
    uint8_t* q_lo = q_hi + SM::kQ;
    uint8_t* k_hi = q_lo + SM::kQ;
    uint8_t* k_lo = k_hi + SM::kK;
    uint8_t* v_hi = k_lo + SM::kK;
    uint8_t* v_lo = v_hi + SM::kV;
    uint8_t* p_hi = v_lo + SM::kV;
    uint8_t* p_lo = p_hi + SM::kP;
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t s_tmem;
    __shared__ float s_x[2][kTcQ];                 // partner exchange (row max, row sum)

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int row = tid & (kTcQ - 1);              // query row = TMEM lane
    const int hf = tid >> 7;                       // which half of the columns
    const int h = blockIdx.y;
    int lo = 0, hi = n_members - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (members[mid].tile0 <= (int)blockIdx.x) lo = mid; else hi = mid - 1;
    }
    const tdkv_attn_member m = members[lo];
    const int r0 = ((int)blockIdx.x - m.tile0) * kTcQ;
    const int nq = min(kTcQ, m.n_rows - r0);
    const int hid = H * D;
    const size_t lofs = (size_t)layer * m.ctx_layer_stride;
    const float* ctx_k = m.ctx_k + lofs;
    const float* ctx_v = m.ctx_v + lofs;
    const float* kf = k_fresh + (size_t)m.row0 * hid;
    const float* vf = v_fresh + (size_t)m.row0 * hid;
    const int tn = (int)m.fix_idx[r0 + nq - 1] + 1;        // keys any row of the tile sees
    const int ntiles = (tn + kTcK - 1) / kTcK;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(&s_tmem)),
                     "n"(kTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    // the query rows, split into tf32 hi / lo (each thread half a row)
    const bool valid = row < nq;
    const int tnq = valid ? (int)m.fix_idx[r0 + row] + 1 : 0;
    {
        const float* qrow = q + (size_t)(m.row0 + r0 + row) * hid + h * D;
#pragma unroll
        for (int c = hf * (kCq / 2); c < (hf + 1) * (kCq / 2); ++c) {
            const float4 v = valid ? *reinterpret_cast<const float4*>(qrow + 4 * c)
                                   : make_float4(0.f, 0.f, 0.f, 0.f);
            split_store16(q_hi, q_lo, core_off(row, c, kCq), v);
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = s_tmem;
    const uint32_t lane = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t t_s = tmem + lane + hf * kSh;             // S: columns [0, kTcK)
    const uint32_t t_o = tmem + lane + kTcK + hf * kOh;      // O: columns [kTcK, kTcK + D)
    const uint32_t idesc_s = umma_idesc(2, kTcQ, kTcK);
    const uint32_t idesc_o = umma_idesc(2, kTcQ, D);

    float acc[kOh];
#pragma unroll
    for (int d = 0; d < kOh; ++d) acc[d] = 0.f;
    float mrun = -INFINITY;
    float lrun = 0.f;                               // this half's share of the row sum
    uint32_t phase = 0;

    // K / V rows of a tile: eight consecutive threads take eight keys of one
    // 16-byte column; tile it + 1 is loaded into registers while tile it is
    // multiplied and softmaxed, then split and stored
    constexpr int kPer = kTcK * kCq / kTcThreads;          // chunks per thread
    float4 kreg[kPer], vreg[kPer];
    auto load_tile = [&](int it) {
        const int t0 = it * kTcK;
        const int n = min(kTcK, tn - t0);
#pragma unroll
        for (int i = 0; i < kPer; ++i) {
            const int idx = tid + i * kTcThreads;
            const int key = (idx & 7) + ((idx / (8 * kCq)) << 3);
            const int c = (idx >> 3) % kCq;
            kreg[i] = make_float4(0.f, 0.f, 0.f, 0.f);
            vreg[i] = kreg[i];
            if (key < n) {
                const int t = t0 + key;
                const int fr = __ldg(m.fresh_of + t);
                const size_t off = (size_t)h * D + 4 * c;
                kreg[i] = *reinterpret_cast<const float4*>(
                    (fr >= 0 ? kf + (size_t)fr * hid : ctx_k + (size_t)t * hid) + off);
                vreg[i] = *reinterpret_cast<const float4*>(
                    (fr >= 0 ? vf + (size_t)fr * hid : ctx_v + (size_t)t * hid) + off);
            }
        }
    };
    load_tile(0);

    for (int it = 0; it < ntiles; ++it) {
        const int t0 = it * kTcK;
        const int n = min(kTcK, tn - t0);
        // ---- store K (rows = keys) and V^T (rows = head dims), tf32 hi / lo
#pragma unroll
        for (int i = 0; i < kPer; ++i) {
            const int idx = tid + i * kTcThreads;
            const int key = (idx & 7) + ((idx / (8 * kCq)) << 3);
            const int c = (idx >> 3) % kCq;
            split_store16(k_hi, k_lo, core_off(key, c, kCq), kreg[i]);
            const float vx[4] = {vreg[i].x, vreg[i].y, vreg[i].z, vreg[i].w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint32_t o = core_off(4 * c + j, key >> 2, kCp) + (key & 3) * 4;
                const uint32_t hb = tf32_rna(vx[j]);
                *reinterpret_cast<uint32_t*>(v_hi + o) = hb;
                *reinterpret_cast<uint32_t*>(v_lo + o) = tf32_rna(vx[j] - __uint_as_float(hb));
            }
        }
        fence_proxy_async_smem();
        tc_fence_before();
        __syncthreads();
        if (tid == 0) {
            tc_fence_after();
#pragma unroll
            for (int s = 0; s < D / 8; ++s) {
                const uint32_t koff = s * 256;
                const uint64_t dqh = umma_desc(smem_u32(q_hi) + koff, 128, kCq * 128);
                const uint64_t dql = umma_desc(smem_u32(q_lo) + koff, 128, kCq * 128);
                const uint64_t dkh = umma_desc(smem_u32(k_hi) + koff, 128, kCq * 128);
                const uint64_t dkl = umma_desc(smem_u32(k_lo) + koff, 128, kCq * 128);
                umma<true>(tmem, dqh, dkh, idesc_s, s > 0 ? 1u : 0u);
                umma<true>(tmem, dqh, dkl, idesc_s, 1u);
                umma<true>(tmem, dql, dkh, idesc_s, 1u);
            }
            umma_commit(&bar);
        }
        if (it + 1 < ntiles) load_tile(it + 1);     // in flight over the softmax
        mbar_wait(&bar, phase);
        phase ^= 1;
        tc_fence_after();
        // ---- this half of the score row -> P (online softmax)
        float x[kSh];
        tmem_row<kSh>(t_s, x);
        float tmax = -INFINITY;
#pragma unroll
        for (int j = 0; j < kSh; ++j) {
            const int key = hf * kSh + j;
            x[j] = (key < n && t0 + key < tnq) ? x[j] * scale : -INFINITY;
            tmax = fmaxf(tmax, x[j]);
        }
        s_x[hf][row] = tmax;
        __syncthreads();
        const float mnew = fmaxf(mrun, fmaxf(tmax, s_x[hf ^ 1][row]));
        const float corr = (mrun == -INFINITY || mnew == -INFINITY) ? 1.f : expf(mrun - mnew);
        float psum = 0.f;
#pragma unroll
        for (int j = 0; j < kSh; ++j) {
            x[j] = x[j] == -INFINITY ? 0.f : expf(x[j] - mnew);
            psum += x[j];
        }
        lrun = lrun * corr + psum;
        mrun = mnew;
#pragma unroll
        for (int c = 0; c < kCp / 2; ++c)
            split_store16(p_hi, p_lo, core_off(row, hf * (kCp / 2) + c, kCp),
                          make_float4(x[4 * c], x[4 * c + 1], x[4 * c + 2], x[4 * c + 3]));
        fence_proxy_async_smem();
        tc_fence_before();
        __syncthreads();
        if (tid == 0) {
            tc_fence_after();
#pragma unroll
            for (int s = 0; s < kTcK / 8; ++s) {
                const uint32_t koff = s * 256;
                const uint64_t dph = umma_desc(smem_u32(p_hi) + koff, 128, kCp * 128);
                const uint64_t dpl = umma_desc(smem_u32(p_lo) + koff, 128, kCp * 128);
                const uint64_t dvh = umma_desc(smem_u32(v_hi) + koff, 128, kCp * 128);
                const uint64_t dvl = umma_desc(smem_u32(v_lo) + koff, 128, kCp * 128);
                umma<true>(tmem + kTcK, dph, dvh, idesc_o, s > 0 ? 1u : 0u);
                umma<true>(tmem + kTcK, dph, dvl, idesc_o, 1u);
                umma<true>(tmem + kTcK, dpl, dvh, idesc_o, 1u);
            }
            umma_commit(&bar);
        }
        mbar_wait(&bar, phase);
        phase ^= 1;
        tc_fence_after();
        {
            float o[kOh];
            tmem_row<kOh>(t_o, o);
#pragma unroll
            for (int d = 0; d < kOh; ++d) acc[d] = fmaf(acc[d], corr, o[d]);
        }
        // K / V / P shared memory and both accumulators are reused next tile
        tc_fence_before();
        __syncthreads();
        tc_fence_after();
    }
    s_x[hf][row] = lrun;
    __syncthreads();
    if (valid) {
        const float l = s_x[0][row] + s_x[1][row];
        float* out = mix + (size_t)(m.row0 + r0 + row) * hid + h * D + hf * kOh;
#pragma unroll
        for (int c = 0; c < kOh / 4; ++c)
            *reinterpret_cast<float4*>(out + 4 * c) =
                make_float4(acc[4 * c] / l, acc[4 * c + 1] / l, acc[4 * c + 2] / l,
                            acc[4 * c + 3] / l);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                     "n"(kTmemCols)
                     : "memory");
    }
}

template <int D>
static int32_t launch_attention_tc(const float* d_q, const float* d_k_fresh,
                                   const float* d_v_fresh, const tdkv_attn_member* d_members,
                                   int32_t n_members, int32_t layer, int32_t n_tiles,
                                   int32_t num_heads, float scale, float* d_mix, cudaStream_t s) {
    auto kern = attention_tc_kernel<D>;
    const size_t smem = TcAttnSmem<D>::kBytes;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
        return check_launch("tdkv_attention_many: cudaFuncSetAttribute");
    kern<<<dim3(n_tiles, num_heads), kTcThreads, smem, s>>>(d_q, d_k_fresh, d_v_fresh, d_members,
                                                     n_members, layer, num_heads, scale, d_mix);
    count_launch();
    return check_launch("tdkv_attention_many");
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
    if (n_tiles > 0 && (rows_per_tile == kTcQ || rows_per_tile == kBlkQ) &&
        (!aligned(d_q, 16) || !aligned(d_k_fresh, 16) || !aligned(d_v_fresh, 16) ||
         !aligned(d_mix, 16) || (num_heads * head_dim) % 4))
        return set_error(TDKV_EINVAL, "tdkv_attention_many: %d-row tiles read and write "
                         "16-byte vectors: row planes must be 16-byte aligned with H*D %% 4 == 0",
                         rows_per_tile);
    if (n_tiles > 0 && rows_per_tile == kTcQ) {
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        switch (head_dim) {
            case 32: return launch_attention_tc<32>(d_q, d_k_fresh, d_v_fresh, d_members, n_members, layer, n_tiles, num_heads, scale, d_mix, s);
            case 64: return launch_attention_tc<64>(d_q, d_k_fresh, d_v_fresh, d_members, n_members, layer, n_tiles, num_heads, scale, d_mix, s);
            default:
                return set_error(TDKV_EINVAL, "tdkv_attention_many: 128-row tensor-core tiles "
                                 "need head_dim 32 or 64, got %d", head_dim);
        }
    }
    if (n_tiles > 0 && rows_per_tile == kBlkQ) {
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        switch (head_dim) {
            case 8: return launch_attention_block<8>(d_q, d_k_fresh, d_v_fresh, d_members, n_members, layer, n_tiles, num_heads, scale, d_mix, s);
            case 16: return launch_attention_block<16>(d_q, d_k_fresh, d_v_fresh, d_members, n_members, layer, n_tiles, num_heads, scale, d_mix, s);
            case 32: return launch_attention_block<32>(d_q, d_k_fresh, d_v_fresh, d_members, n_members, layer, n_tiles, num_heads, scale, d_mix, s);
            case 64: return launch_attention_block<64>(d_q, d_k_fresh, d_v_fresh, d_members, n_members, layer, n_tiles, num_heads, scale, d_mix, s);
            case 128: return launch_attention_block<128>(d_q, d_k_fresh, d_v_fresh, d_members, n_members, layer, n_tiles, num_heads, scale, d_mix, s);
            default:
                return set_error(TDKV_EINVAL, "tdkv_attention_many: 64-row tiles need head_dim "
                                 "in {8, 16, 32, 64, 128}, got %d", head_dim);
        }
    }
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
