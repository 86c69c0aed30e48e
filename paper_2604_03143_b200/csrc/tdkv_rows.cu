// K3 row mover: gather -> diff overlay -> rotate -> scatter.
//
// One kernel serves the fused decoder (restore.fused_restore,
// restore.py:50-104): for every (job, layer, block) the source block is the
// diff payload when the block changed, else the master rows; the overlay
// happens before rotation (restore.py:5-8); rotated K and V go straight to
// the job's pool slots.  With no diff map it is rope_apply / rope_recover
// (toymodel.py:60-96) or a plain write_rows / read_rows (paged_pool.py:150-
// 164); with rotate == 0 and identity destinations it is diff_decode_dense
// (diffstore.py:185-203).  No dense mirror is ever materialized on the fused
// path.
#include <cstdlib>

#include "tdkv_common.cuh"

namespace tdkv {

struct RowsGeom {
    int32_t num_layers;
    int32_t row_elems;
    int32_t head_dim;
    int32_t block_size;
    int32_t nb_max;
    int32_t n_jobs;
    int32_t job_minor;    // TDKV_ROWS_JOB_MINOR: items ordered (layer, block, tile, job)
};

// item -> (job, layer, tile-in-layer) for ``per_layer`` tiles per layer
__device__ __forceinline__ void rows_item(long long it, const RowsGeom& g, long long per_job,
                                          int per_layer, int& ji, int& layer, int& r2) {
    long long rem;
    if (g.job_minor) {
        const long long lt = it / g.n_jobs;
        ji = (int)(it - lt * g.n_jobs);
        rem = lt;
    } else {
        ji = (int)(it / per_job);
        rem = it - (long long)ji * per_job;
    }
    layer = (int)(rem / per_layer);
    r2 = (int)(rem - (long long)layer * per_layer);
}

template <typename T, int UB>
__global__ void __launch_bounds__(256, 3)
    rows_kernel(const tdkv_rows_job* __restrict__ jobs, const void* __restrict__ table_v,
                const RowsGeom g) {
    using V = typename UnitBits<UB>::V;
    using Tbl = typename Elt<T>::Table;
    constexpr int kEpu = UB / (int)sizeof(T);
    constexpr int kPairs = kEpu / 2;
    constexpr int kRows = 4;                       // rows in flight per thread
    const Tbl* __restrict__ table = static_cast<const Tbl*>(table_v);
    const int upr = g.row_elems * (int)sizeof(T) / UB;
    const int half = g.head_dim >> 1;
    // fixed thread -> column mapping (as in K1): a warp covers consecutive
    // 16-byte units of one row, so every load/store is a full 512-byte run
    const int nthr = blockDim.x;
    const int tx_n = upr < nthr ? upr : nthr;
    const int rows_per_pass = nthr / tx_n;
    const int tx = threadIdx.x % tx_n;
    const int ty = threadIdx.x / tx_n;
    const int per_job = g.num_layers * g.nb_max;
    const long long n_items = (long long)g.n_jobs * per_job;
    if (ty >= rows_per_pass) return;               // no barriers below

    for (long long item = blockIdx.x; item < n_items; item += gridDim.x) {
        int ji, layer, b;
        rows_item(item, g, per_job, g.nb_max, ji, layer, b);
        const tdkv_rows_job* job = jobs + ji;
        const int T_ = job->num_tokens;
        const int lo = b * g.block_size;
        if (lo >= T_) continue;                    // uniform across the CTA
        const int rows = min(g.block_size, T_ - lo);
        const int nbj = (T_ + g.block_size - 1) / g.block_size;

        const int mk_i = job->map_k ? __ldg(job->map_k + layer * nbj + b) : -1;
        const int mv_i = job->map_v ? __ldg(job->map_v + layer * nbj + b) : -1;
        const size_t re = (size_t)g.row_elems;
        const T* k_base = mk_i >= 0 ? static_cast<const T*>(job->pay_k) + (size_t)mk_i * g.block_size * re
                                    : static_cast<const T*>(job->src_k) + (size_t)layer * job->src_layer_stride;
        const T* v_base = mv_i >= 0 ? static_cast<const T*>(job->pay_v) + (size_t)mv_i * g.block_size * re
                                    : static_cast<const T*>(job->src_v) + (size_t)layer * job->src_layer_stride;
        // payload rows are block-relative and contiguous; master rows go
        // through src_rows (or are the token index)
        const bool k_pay = mk_i >= 0, v_pay = mv_i >= 0;
        T* dst_k_l = static_cast<T*>(job->dst_k) + (size_t)layer * job->dst_layer_stride;
        T* dst_v_l = static_cast<T*>(job->dst_v) + (size_t)layer * job->dst_layer_stride;
        const int64_t* srows = job->src_rows;
        const int64_t* drows = job->dst_rows;
        const int rotate = job->rotate;
        const int tbl_row = job->tbl_row, tbl_stride = job->tbl_stride;
        const bool has_v = job->dst_v != nullptr;  // K-only jobs (rope_apply)

        for (int c = tx; c < upr; c += tx_n) {
            const int j0 = ((c * kEpu) % g.head_dim) >> 1;
            Tbl cs[kPairs];
            if (rotate && tbl_stride == 0) {
                const Tbl* trow = table + (size_t)tbl_row * half + j0;
#pragma unroll
                for (int q = 0; q < kPairs; ++q) cs[q] = __ldg(trow + q);
            }
            for (int r0 = ty; r0 < rows; r0 += kRows * rows_per_pass) {
                V kx[kRows], vx[kRows];
                int64_t drow[kRows];
#pragma unroll
                for (int q = 0; q < kRows; ++q) {
                    const int r = r0 + q * rows_per_pass;
                    if (r < rows) {
                        const int t = lo + r;
                        const int64_t srow = srows ? __ldg(srows + t) : t;
                        drow[q] = drows ? __ldg(drows + t) : t;
                        const T* ks = k_base + (k_pay ? (size_t)r : (size_t)srow) * re;
                        kx[q] = ld_stream(reinterpret_cast<const V*>(ks) + c);
                        if (has_v) {
                            const T* vs = v_base + (v_pay ? (size_t)r : (size_t)srow) * re;
                            vx[q] = ld_stream(reinterpret_cast<const V*>(vs) + c);
                        }
                    }
                }
#pragma unroll
                for (int q = 0; q < kRows; ++q) {
                    const int r = r0 + q * rows_per_pass;
                    if (r < rows) {
                        if (rotate) {
                            if (tbl_stride != 0) {
                                const Tbl* trow =
                                    table + (size_t)(tbl_row + (lo + r) * tbl_stride) * half + j0;
#pragma unroll
                                for (int p = 0; p < kPairs; ++p) cs[p] = __ldg(trow + p);
                            }
                            T* e = reinterpret_cast<T*>(&kx[q]);
#pragma unroll
                            for (int p = 0; p < kPairs; ++p) rot_pair(e[2 * p], e[2 * p + 1], cs[p]);
                        }
                        st_stream(reinterpret_cast<V*>(dst_k_l + (size_t)drow[q] * re) + c, kx[q]);
                        if (has_v)
                            st_stream(reinterpret_cast<V*>(dst_v_l + (size_t)drow[q] * re) + c, vx[q]);
                    }
                }
            }
        }
    }
}

// TMA-staged variant (contiguous sources), warp-specialized: warp 8 is the
// producer -- it resolves each work item (job fields, block-map entry,
// source/destination addresses), loads the tile's destination rows into the
// stage's metadata and issues the bulk copies of the tile's K and V rows
// (never straddling a diff block) -- while warps 0-7 rotate and scatter the
// tiles of earlier stages.  A kStages ring with full/empty mbarriers links
// them, so the dependent metadata loads and the copies run ahead of the
// consumers and the loop has no CTA-wide barrier.
// 4 consumer warps + the producer: more, smaller CTAs per SM overlap one
// CTA's ring waits with another's stores (C3 family restore 0.73 -> 0.70 ms,
// C2 per-mirror 2.83 -> 2.74 ms vs 8 consumer warps; 2 warps measured lower
// at C3)
constexpr int kRowsConsumers = 128;

struct RowsItem {
    int valid;                // 0 = no more items (sentinel stage)
    int lo, n;                // token range of the tile
    int rotate, tbl_row, tbl_stride;
    void* dk;                 // destination planes of the item's layer
    void* dv;
};

template <typename T, int S>
__global__ void __launch_bounds__(kRowsConsumers + 32)
    rows_tma_kernel(const tdkv_rows_job* __restrict__ jobs, const void* __restrict__ table_v,
                    const RowsGeom g, const int tile_rows) {
    using V = uint4;
    using Tbl = typename Elt<T>::Table;
    constexpr int kEpu = 16 / (int)sizeof(T);
    constexpr int kPairs = kEpu / 2;
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ __align__(8) uint64_t full[S], empty[S];
    __shared__ __align__(16) int64_t s_drow[S][32];
    __shared__ RowsItem s_it[S];

    const Tbl* __restrict__ table = static_cast<const Tbl*>(table_v);
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int row_bytes = g.row_elems * (int)sizeof(T);
    const int upr = row_bytes / 16;
    const int tile_bytes = tile_rows * row_bytes;
    const int half = g.head_dim >> 1;
    const int tpb = (g.block_size + tile_rows - 1) / tile_rows;     // tiles per block
    const long long per_job = (long long)g.num_layers * g.nb_max * tpb;
    const long long n_items = (long long)g.n_jobs * per_job;
    const size_t re = (size_t)g.row_elems;

    if (tid == 0) {
        for (int i = 0; i < S; ++i) {
            mbar_init(&full[i], 32);                        // every producer lane arrives
            mbar_init(&empty[i], kRowsConsumers);          // every consumer thread arrives
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == kRowsConsumers / 32) {                      // ---- producer warp
        int k = 0;
        for (long long it = blockIdx.x;; it += gridDim.x) {
            // next valid item (tiles past a job's last token are skipped)
            int ji = 0, layer = 0, b = 0, lo = 0, n = 0, T_ = 0;
            const tdkv_rows_job* job = nullptr;
            for (; it < n_items; it += gridDim.x) {
                int r2;
                rows_item(it, g, per_job, g.nb_max * tpb, ji, layer, r2);
                b = r2 / tpb;
                job = jobs + ji;
                T_ = job->num_tokens;
                const int blo = b * g.block_size;
                lo = blo + (r2 - b * tpb) * tile_rows;
                n = min(tile_rows, min(blo + g.block_size, T_) - lo);
                if (n > 0) break;
            }
            const int st = k % S;
            if (k >= S) mbar_wait(&empty[st], (uint32_t)((k / S - 1) & 1));
            if (it >= n_items) {                             // sentinel: consumers stop
                if (lane == 0) s_it[st].valid = 0;
                __syncwarp();
                mbar_arrive(&full[st]);
                break;
            }
            const int nbj = (T_ + g.block_size - 1) / g.block_size;
            if (lane < n) s_drow[st][lane] = job->dst_rows ? __ldg(job->dst_rows + lo + lane) : lo + lane;
            if (lane == 0) {
                const int mk_i = job->map_k ? job->map_k[layer * nbj + b] : -1;
                const int mv_i = job->map_v ? job->map_v[layer * nbj + b] : -1;
                const int in_blk = lo - b * g.block_size;
                const T* ks = mk_i >= 0
                    ? static_cast<const T*>(job->pay_k) + ((size_t)mk_i * g.block_size + in_blk) * re
                    : static_cast<const T*>(job->src_k) + (size_t)layer * job->src_layer_stride + (size_t)lo * re;
                RowsItem& o = s_it[st];
                o.valid = 1;
                o.lo = lo;
                o.n = n;
                o.rotate = job->rotate;
                o.tbl_row = job->tbl_row;
                o.tbl_stride = job->tbl_stride;
                o.dk = static_cast<T*>(job->dst_k) + (size_t)layer * job->dst_layer_stride;
                o.dv = job->dst_v ? static_cast<T*>(job->dst_v) + (size_t)layer * job->dst_layer_stride
                                  : nullptr;
                const uint32_t bytes = (uint32_t)n * row_bytes;
                uint8_t* dst = smem + (size_t)st * 2 * tile_bytes;
                fence_proxy_async_smem();                    // consumers' reads of this stage done
                mbar_arrive_expect_tx(&full[st], (job->dst_v ? 2u : 1u) * bytes);
                bulk_g2s(dst, ks, bytes, &full[st]);
                if (job->dst_v) {
                    const T* vs = mv_i >= 0
                        ? static_cast<const T*>(job->pay_v) + ((size_t)mv_i * g.block_size + in_blk) * re
                        : static_cast<const T*>(job->src_v) + (size_t)layer * job->src_layer_stride + (size_t)lo * re;
                    bulk_g2s(dst + tile_bytes, vs, bytes, &full[st]);
                }
            } else {
                mbar_arrive(&full[st]);
            }
            ++k;
        }
        return;
    }

    // ---- consumer warps 0-7
    const int tx_n = upr < kRowsConsumers ? upr : kRowsConsumers;
    const int rows_per_pass = kRowsConsumers / tx_n;
    const int tx = tid % tx_n, ty = tid / tx_n;
    for (int k = 0;; ++k) {
        const int st = k % S;
        mbar_wait(&full[st], (uint32_t)((k / S) & 1));
        const RowsItem x = s_it[st];
        if (!x.valid) break;
        const V* sk = reinterpret_cast<const V*>(smem + (size_t)st * 2 * tile_bytes);
        const V* sv = reinterpret_cast<const V*>(smem + (size_t)st * 2 * tile_bytes + tile_bytes);
        T* dk = static_cast<T*>(x.dk);
        T* dv = static_cast<T*>(x.dv);
        const bool has_v = dv != nullptr;
        if (ty < rows_per_pass) {
            for (int c = tx; c < upr; c += tx_n) {
                const int j0 = ((c * kEpu) % g.head_dim) >> 1;
                Tbl cs[kPairs];
                if (x.rotate && x.tbl_stride == 0) {
                    const Tbl* trow = table + (size_t)x.tbl_row * half + j0;
#pragma unroll
                    for (int q = 0; q < kPairs; ++q) cs[q] = __ldg(trow + q);
                }
                for (int r = ty; r < x.n; r += rows_per_pass) {
                    const int64_t drow = s_drow[st][r];
                    V kx = sk[r * upr + c];
                    if (x.rotate) {
                        if (x.tbl_stride != 0) {
                            const Tbl* trow =
                                table + (size_t)(x.tbl_row + (x.lo + r) * x.tbl_stride) * half + j0;
#pragma unroll
                            for (int q = 0; q < kPairs; ++q) cs[q] = __ldg(trow + q);
                        }
                        T* e = reinterpret_cast<T*>(&kx);
#pragma unroll
                        for (int q = 0; q < kPairs; ++q) rot_pair(e[2 * q], e[2 * q + 1], cs[q]);
                    }
                    st_stream(reinterpret_cast<V*>(dk + (size_t)drow * re) + c, kx);
                    if (has_v) st_stream(reinterpret_cast<V*>(dv + (size_t)drow * re) + c, sv[r * upr + c]);
                }
            }
        }
        // every consumer thread releases the stage itself (its own reads are
        // then ordered before the producer's refill without relying on a warp
        // barrier; measured at no cost)
        mbar_arrive(&empty[st]);
    }
}

template <typename T, int S>
static int32_t launch_rows_tma_s(const tdkv_rows_job* jobs, const void* table, const RowsGeom& g,
                                 int tile_rows, int grid_limit, cudaStream_t s) {
    auto kern = rows_tma_kernel<T, S>;
    const size_t smem = (size_t)2 * S * tile_rows * g.row_elems * sizeof(T);
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
        return check_launch("tdkv_rows: cudaFuncSetAttribute");
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kRowsConsumers + 32, smem);
    if (per_sm < 1) per_sm = 1;
    const int tpb = (g.block_size + tile_rows - 1) / tile_rows;
    const long long items = (long long)g.n_jobs * g.num_layers * g.nb_max * tpb;
    long long grid = (long long)sm_count() * per_sm;
    if (grid_limit > 0 && grid > grid_limit) grid = grid_limit;
    if (grid > items) grid = items;
    kern<<<(unsigned)grid, kRowsConsumers + 32, smem, s>>>(jobs, table, g, tile_rows);
    return TDKV_OK;
}

// ring depth: TDKV_ROWS_STAGES (2-4, default 2) stages of tile_rows K+V rows
template <typename T>
static int32_t launch_rows_tma(const tdkv_rows_job* jobs, const void* table, const RowsGeom& g,
                               int tile_rows, int grid_limit, cudaStream_t s) {
    static const int stages = [] {
        const char* e = getenv("TDKV_ROWS_STAGES");
        const int v = e ? atoi(e) : 2;
        return v < 2 ? 2 : v > 4 ? 4 : v;
    }();
    if (stages == 4) return launch_rows_tma_s<T, 4>(jobs, table, g, tile_rows, grid_limit, s);
    if (stages == 3) return launch_rows_tma_s<T, 3>(jobs, table, g, tile_rows, grid_limit, s);
    return launch_rows_tma_s<T, 2>(jobs, table, g, tile_rows, grid_limit, s);
}

template <typename T>
__global__ void fill_rows_kernel(T* __restrict__ plane, int64_t layer_stride, int num_layers,
                                 const int64_t* __restrict__ rows, int64_t n_rows, int row_elems,
                                 T value) {
    const long long total = (long long)num_layers * n_rows * row_elems;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const long long per_layer = n_rows * row_elems;
        const int layer = (int)(i / per_layer);
        const long long rem = i - layer * per_layer;
        const long long r = rem / row_elems;
        const int e = (int)(rem - r * row_elems);
        plane[(size_t)layer * layer_stride + (size_t)rows[r] * row_elems + e] = value;
    }
}

template <typename T, int UB>
static void launch_rows(const tdkv_rows_job* jobs, const void* table, const RowsGeom& g,
                        int grid_limit, cudaStream_t s) {
    const long long items = (long long)g.n_jobs * g.num_layers * g.nb_max;
    long long grid = (long long)sm_count() * 8;
    if (grid_limit > 0 && grid > grid_limit) grid = grid_limit;
    if (grid > items) grid = items;
    rows_kernel<T, UB><<<(unsigned)grid, 256, 0, s>>>(jobs, table, g);
}

}  // namespace tdkv

using namespace tdkv;

extern "C" int32_t tdkv_rows(const tdkv_rows_job* d_jobs, int32_t n_jobs, int32_t max_tokens,
                             const void* d_table, int32_t num_layers, int32_t num_heads,
                             int32_t head_dim, int32_t block_size, int32_t dtype, int32_t flags,
                             int32_t tile_rows, int32_t grid_limit, void* stream) {
    if (n_jobs < 0 || num_layers <= 0 || num_heads <= 0 || head_dim <= 0 || (head_dim & 1) ||
        block_size <= 0 || max_tokens < 0)
        return set_error(TDKV_EINVAL, "tdkv_rows: bad geometry");
    if (n_jobs == 0 || max_tokens == 0) return TDKV_OK;
    if (!d_jobs) return set_error(TDKV_EINVAL, "tdkv_rows: null job array");
    if (dtype != TDKV_F32 && dtype != TDKV_BF16)
        return set_error(TDKV_EUNSUPPORTED, "tdkv_rows: dtype %d", dtype);
    RowsGeom g{num_layers, num_heads * head_dim, head_dim, block_size,
               ceil_div(max_tokens, block_size), n_jobs, (flags & TDKV_ROWS_JOB_MINOR) ? 1 : 0};
    // the caller (host wrapper) promises 16-byte aligned planes/strides when
    // rows are whole 16-byte units; pick_unit_bytes encodes the row test
    const int ub = pick_unit_bytes(dtype, head_dim, g.row_elems);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if ((flags & TDKV_ROWS_CONTIGUOUS) && ub == 16) {
        if (tile_rows <= 0 || tile_rows > block_size) tile_rows = block_size;
        if (tile_rows > 32) tile_rows = 32;        // staged destination rows per tile
        if ((size_t)4 * tile_rows * g.row_elems * elt_size(dtype) > 227 * 1024)
            return set_error(TDKV_EINVAL, "tdkv_rows: tile of %d rows exceeds shared memory",
                             tile_rows);
        const int32_t rc = dtype == TDKV_F32
                               ? launch_rows_tma<float>(d_jobs, d_table, g, tile_rows, grid_limit, s)
                               : launch_rows_tma<__nv_bfloat16>(d_jobs, d_table, g, tile_rows,
                                                                grid_limit, s);
        if (rc) return rc;
        count_launch();
        return check_launch("tdkv_rows");
    }
    if (dtype == TDKV_F32) {
        if (ub == 16) launch_rows<float, 16>(d_jobs, d_table, g, grid_limit, s);
        else launch_rows<float, 8>(d_jobs, d_table, g, grid_limit, s);
    } else {
        if (ub == 16) launch_rows<__nv_bfloat16, 16>(d_jobs, d_table, g, grid_limit, s);
        else launch_rows<__nv_bfloat16, 4>(d_jobs, d_table, g, grid_limit, s);
    }
    count_launch();
    return check_launch("tdkv_rows");
}

extern "C" int32_t tdkv_fill_rows(void* d_plane, int64_t layer_stride, int32_t num_layers,
                                  const int64_t* d_rows, int64_t n_rows, int32_t row_elems,
                                  int32_t dtype, uint32_t value_bits, void* stream) {
    if (n_rows < 0 || num_layers <= 0 || row_elems <= 0)
        return set_error(TDKV_EINVAL, "tdkv_fill_rows: bad geometry");
    if (n_rows == 0) return TDKV_OK;
    if (!d_plane || !d_rows) return set_error(TDKV_EINVAL, "tdkv_fill_rows: null pointer");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const long long total = (long long)num_layers * n_rows * row_elems;
    long long grid = (total + 255) / 256;
    if (grid > sm_count() * 8) grid = sm_count() * 8;
    if (dtype == TDKV_F32) {
        float v;
        memcpy(&v, &value_bits, 4);
        fill_rows_kernel<float><<<(unsigned)grid, 256, 0, s>>>(static_cast<float*>(d_plane),
                                                               layer_stride, num_layers, d_rows,
                                                               n_rows, row_elems, v);
    } else if (dtype == TDKV_BF16) {
        const uint16_t bits = (uint16_t)value_bits;
        __nv_bfloat16 v;
        memcpy(&v, &bits, 2);
        fill_rows_kernel<__nv_bfloat16><<<(unsigned)grid, 256, 0, s>>>(
            static_cast<__nv_bfloat16*>(d_plane), layer_stride, num_layers, d_rows, n_rows,
            row_elems, v);
    } else {
        return set_error(TDKV_EUNSUPPORTED, "tdkv_fill_rows: dtype %d", dtype);
    }
    count_launch();
    return check_launch("tdkv_fill_rows");
}
