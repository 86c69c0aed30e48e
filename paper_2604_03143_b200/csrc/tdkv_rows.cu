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
__global__ void __launch_bounds__(256)
    rows_kernel(const tdkv_rows_job* __restrict__ jobs, const void* __restrict__ table_v,
                const RowsGeom g) {
    using V = typename UnitBits<UB>::V;
    using Tbl = typename Elt<T>::Table;
    constexpr int kEpu = UB / (int)sizeof(T);
    constexpr int kPairs = kEpu / 2;
    constexpr int kUnroll = 4;
    const Tbl* __restrict__ table = static_cast<const Tbl*>(table_v);
    const int upr = g.row_elems * (int)sizeof(T) / UB;
    const int half = g.head_dim >> 1;
    const int per_job = g.num_layers * g.nb_max;
    const long long n_items = (long long)g.n_jobs * per_job;

    for (long long item = blockIdx.x; item < n_items; item += gridDim.x) {
        const int ji = (int)(item / per_job);
        const int rem = (int)(item - (long long)ji * per_job);
        const int layer = rem / g.nb_max;
        const int b = rem - layer * g.nb_max;
        const tdkv_rows_job& job = jobs[ji];
        const int T_ = job.num_tokens;
        const int lo = b * g.block_size;
        if (lo >= T_) continue;                    // uniform across the CTA
        const int rows = min(g.block_size, T_ - lo);
        const int nbj = (T_ + g.block_size - 1) / g.block_size;

        const int mk_i = job.map_k ? job.map_k[layer * nbj + b] : -1;
        const int mv_i = job.map_v ? job.map_v[layer * nbj + b] : -1;
        const T* src_k_l = static_cast<const T*>(job.src_k) + (size_t)layer * job.src_layer_stride;
        const T* src_v_l = static_cast<const T*>(job.src_v) + (size_t)layer * job.src_layer_stride;
        T* dst_k_l = static_cast<T*>(job.dst_k) + (size_t)layer * job.dst_layer_stride;
        T* dst_v_l = static_cast<T*>(job.dst_v) + (size_t)layer * job.dst_layer_stride;
        const int64_t* srows = job.src_rows;
        const int64_t* drows = job.dst_rows;
        const int rotate = job.rotate;
        const int tbl_row = job.tbl_row, tbl_stride = job.tbl_stride;
        const T* pay_k = static_cast<const T*>(job.pay_k);
        const T* pay_v = static_cast<const T*>(job.pay_v);
        const bool has_v = job.dst_v != nullptr;   // K-only jobs (rope_apply)

        const int units = rows * upr;
        for (int u0 = threadIdx.x; u0 < units; u0 += kUnroll * blockDim.x) {
            V kx[kUnroll], vx[kUnroll];
            int64_t drow[kUnroll];
            int tt[kUnroll], cc[kUnroll];
#pragma unroll
            for (int q = 0; q < kUnroll; ++q) {
                const int u = u0 + q * blockDim.x;
                if (u < units) {
                    const int r = u / upr;
                    const int c = u - r * upr;
                    const int t = lo + r;
                    tt[q] = t;
                    cc[q] = c;
                    const int64_t srow = srows ? __ldg(srows + t) : t;
                    drow[q] = drows ? __ldg(drows + t) : t;
                    const T* ks = mk_i >= 0
                                      ? pay_k + ((size_t)mk_i * g.block_size + r) * g.row_elems
                                      : src_k_l + (size_t)srow * g.row_elems;
                    const T* vs = mv_i >= 0
                                      ? pay_v + ((size_t)mv_i * g.block_size + r) * g.row_elems
                                      : src_v_l + (size_t)srow * g.row_elems;
                    kx[q] = ld_stream(reinterpret_cast<const V*>(ks) + c);
                    if (has_v) vx[q] = ld_stream(reinterpret_cast<const V*>(vs) + c);
                }
            }
#pragma unroll
            for (int q = 0; q < kUnroll; ++q) {
                const int u = u0 + q * blockDim.x;
                if (u < units) {
                    if (rotate) {
                        const int j0 = ((cc[q] * kEpu) % g.head_dim) >> 1;
                        const Tbl* trow =
                            table + (size_t)(tbl_row + tt[q] * tbl_stride) * half + j0;
                        T* e = reinterpret_cast<T*>(&kx[q]);
#pragma unroll
                        for (int p = 0; p < kPairs; ++p) rot_pair(e[2 * p], e[2 * p + 1], trow[p]);
                    }
                    st_stream(reinterpret_cast<V*>(dst_k_l + (size_t)drow[q] * g.row_elems) + cc[q],
                              kx[q]);
                    if (has_v)
                        st_stream(reinterpret_cast<V*>(dst_v_l + (size_t)drow[q] * g.row_elems) + cc[q],
                                  vx[q]);
                }
            }
        }
    }
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
                             int32_t head_dim, int32_t block_size, int32_t dtype, int32_t grid_limit,
                             void* stream) {
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
