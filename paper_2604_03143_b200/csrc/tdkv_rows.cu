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
#include "tdkv_common.cuh"

namespace tdkv {

struct RowsGeom {
    int32_t num_layers;
    int32_t row_elems;
    int32_t head_dim;
    int32_t block_size;
    int32_t nb_max;
    int32_t n_jobs;
};

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
        const int ji = (int)(item / per_job);
        const int rem = (int)(item - (long long)ji * per_job);
        const int layer = rem / g.nb_max;
        const int b = rem - layer * g.nb_max;
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

// TMA-staged variant (contiguous sources): a persistent CTA double-buffers
// row tiles of <= tile_rows rows (never straddling a diff block) into shared
// memory with cp.async.bulk while the threads rotate and scatter the
// previous tile -- loads are decoupled from the scattered stores exactly as
// in K1.
template <typename T>
__global__ void __launch_bounds__(256)
    rows_tma_kernel(const tdkv_rows_job* __restrict__ jobs, const void* __restrict__ table_v,
                    const RowsGeom g, const int tile_rows) {
    using V = uint4;
    using Tbl = typename Elt<T>::Table;
    constexpr int kEpu = 16 / (int)sizeof(T);
    constexpr int kPairs = kEpu / 2;
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ __align__(8) uint64_t bars[2];

    const Tbl* __restrict__ table = static_cast<const Tbl*>(table_v);
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int row_bytes = g.row_elems * (int)sizeof(T);
    const int upr = row_bytes / 16;
    const int tile_bytes = tile_rows * row_bytes;
    const int half = g.head_dim >> 1;
    const int tx_n = upr < nthr ? upr : nthr;
    const int rows_per_pass = nthr / tx_n;
    const int tx = tid % tx_n, ty = tid / tx_n;
    const int tpb = (g.block_size + tile_rows - 1) / tile_rows;     // tiles per block
    const long long per_job = (long long)g.num_layers * g.nb_max * tpb;
    const long long n_items = (long long)g.n_jobs * per_job;
    const size_t re = (size_t)g.row_elems;

    if (tid == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        fence_mbar_init();
    }
    __syncthreads();

    struct Item {
        int ji, layer, b, lo, n;
    };
    auto decode = [&](long long it, Item& x) -> bool {
        x.ji = (int)(it / per_job);
        long long rem = it - (long long)x.ji * per_job;
        const int per_layer = g.nb_max * tpb;
        x.layer = (int)(rem / per_layer);
        const int r2 = (int)(rem - (long long)x.layer * per_layer);
        x.b = r2 / tpb;
        const int sub = r2 - x.b * tpb;
        const int T_ = __ldg(&jobs[x.ji].num_tokens);
        const int blo = x.b * g.block_size;
        const int bhi = min(blo + g.block_size, T_);
        x.lo = blo + sub * tile_rows;
        x.n = min(tile_rows, bhi - x.lo);
        return x.n > 0;
    };
    auto next_valid = [&](long long it, Item& x) -> long long {
        while (it < n_items && !decode(it, x)) it += gridDim.x;
        return it;
    };
    // thread 0 only: stage an item's K (and V) rows into buffer ``bi``
    auto issue = [&](const Item& x, int bi) {
        const tdkv_rows_job* job = jobs + x.ji;
        const int T_ = job->num_tokens;
        const int nbj = (T_ + g.block_size - 1) / g.block_size;
        const int mk_i = job->map_k ? job->map_k[x.layer * nbj + x.b] : -1;
        const int mv_i = job->map_v ? job->map_v[x.layer * nbj + x.b] : -1;
        const int in_blk = x.lo - x.b * g.block_size;
        const T* ks = mk_i >= 0
            ? static_cast<const T*>(job->pay_k) + ((size_t)mk_i * g.block_size + in_blk) * re
            : static_cast<const T*>(job->src_k) + (size_t)x.layer * job->src_layer_stride + (size_t)x.lo * re;
        const uint32_t bytes = (uint32_t)x.n * row_bytes;
        uint8_t* dst = smem + (size_t)bi * 2 * tile_bytes;
        const bool has_v = job->dst_v != nullptr;
        mbar_arrive_expect_tx(&bars[bi], (has_v ? 2u : 1u) * bytes);
        bulk_g2s(dst, ks, bytes, &bars[bi]);
        if (has_v) {
            const T* vs = mv_i >= 0
                ? static_cast<const T*>(job->pay_v) + ((size_t)mv_i * g.block_size + in_blk) * re
                : static_cast<const T*>(job->src_v) + (size_t)x.layer * job->src_layer_stride + (size_t)x.lo * re;
            bulk_g2s(dst + tile_bytes, vs, bytes, &bars[bi]);
        }
    };

    // the tile's destination rows are staged in shared memory with cp.async
    // (issued with the next tile's bulk copy), so the scatter loop never
    // waits on a dependent global load
    __shared__ __align__(16) int64_t s_drow[2][32];
    auto stage_rows = [&](const Item& x, int b) {
        const int64_t* dr = jobs[x.ji].dst_rows;
        if (tid < x.n) {
            if (dr) cp_async_8(&s_drow[b][tid], dr + x.lo + tid);
            else s_drow[b][tid] = x.lo + tid;
        }
        cp_async_commit();
    };

    Item cur, nxt;
    long long it = next_valid(blockIdx.x, cur);
    if (tid == 0 && it < n_items) issue(cur, 0);
    if (it < n_items) stage_rows(cur, 0);
    uint32_t phase0 = 0, phase1 = 0;
    int bi = 0;
    while (it < n_items) {
        const long long nx = next_valid(it + gridDim.x, nxt);
        if (tid == 0 && nx < n_items) {
            fence_proxy_async_smem();
            issue(nxt, bi ^ 1);
        }
        if (nx < n_items) {
            stage_rows(nxt, bi ^ 1);
            cp_async_wait<1>();            // this tile's rows (the older group) landed
        } else {
            cp_async_wait<0>();
        }
        mbar_wait(&bars[bi], bi ? phase1 : phase0);
        if (bi) phase1 ^= 1u; else phase0 ^= 1u;
        __syncthreads();                   // staged rows visible to every thread

        const tdkv_rows_job* job = jobs + cur.ji;
        const V* sk = reinterpret_cast<const V*>(smem + (size_t)bi * 2 * tile_bytes);
        const V* sv = reinterpret_cast<const V*>(smem + (size_t)bi * 2 * tile_bytes + tile_bytes);
        T* dk = static_cast<T*>(job->dst_k) + (size_t)cur.layer * job->dst_layer_stride;
        T* dv = static_cast<T*>(job->dst_v) + (size_t)cur.layer * job->dst_layer_stride;
        const bool has_v = job->dst_v != nullptr;
        const int rotate = job->rotate, tbl_row = job->tbl_row, tbl_stride = job->tbl_stride;
        if (ty < rows_per_pass) {
            for (int c = tx; c < upr; c += tx_n) {
                const int j0 = ((c * kEpu) % g.head_dim) >> 1;
                Tbl cs[kPairs];
                if (rotate && tbl_stride == 0) {
                    const Tbl* trow = table + (size_t)tbl_row * half + j0;
#pragma unroll
                    for (int q = 0; q < kPairs; ++q) cs[q] = __ldg(trow + q);
                }
                for (int r = ty; r < cur.n; r += rows_per_pass) {
                    const int t = cur.lo + r;
                    const int64_t drow = s_drow[bi][r];
                    V kx = sk[r * upr + c];
                    if (rotate) {
                        if (tbl_stride != 0) {
                            const Tbl* trow = table + (size_t)(tbl_row + t * tbl_stride) * half + j0;
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
        __syncthreads();
        it = nx;
        cur = nxt;
        bi ^= 1;
    }
}

template <typename T>
static int32_t launch_rows_tma(const tdkv_rows_job* jobs, const void* table, const RowsGeom& g,
                               int tile_rows, int grid_limit, cudaStream_t s) {
    auto kern = rows_tma_kernel<T>;
    const size_t smem = (size_t)4 * tile_rows * g.row_elems * sizeof(T);
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
        return check_launch("tdkv_rows: cudaFuncSetAttribute");
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, smem);
    if (per_sm < 1) per_sm = 1;
    const int tpb = (g.block_size + tile_rows - 1) / tile_rows;
    const long long items = (long long)g.n_jobs * g.num_layers * g.nb_max * tpb;
    long long grid = (long long)sm_count() * per_sm;
    if (grid_limit > 0 && grid > grid_limit) grid = grid_limit;
    if (grid > items) grid = items;
    kern<<<(unsigned)grid, 256, smem, s>>>(jobs, table, g, tile_rows);
    return TDKV_OK;
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
               ceil_div(max_tokens, block_size), n_jobs};
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
