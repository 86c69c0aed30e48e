// K0 rotary table + K1 KV Collector.
//
// K1 replaces pic.align_cached (pic.py:208-235) + the _skeleton V copy
// (pic.py:203-204) + PagedPool.write_rows (paged_pool.py:150-156): each
// master tile (one segment, <= max_rows rows, K and V) is staged ONCE in
// shared memory by the TMA engine (cp.async.bulk, double-buffered across the
// persistent loop) and then rotated/copied to every agent that holds the
// segment, straight into that agent's paged-pool slots.  HBM traffic is the
// algorithmic minimum M + N*M (master read once, N agent copies written).
#include <cstdlib>

#include "tdkv_common.cuh"

namespace tdkv {

// ---------------------------------------------------------------------------
// K0

template <typename Tbl>
__global__ void rope_table_kernel(const int64_t* __restrict__ deltas, int64_t n_rows,
                                  const double* __restrict__ inv_freq, int half,
                                  Tbl* __restrict__ out) {
    const int64_t total = n_rows * half;
    // under PDL (tdkv_collect_round): the previous round's K1 may still read
    // the table -- wait for every predecessor, then let this round's K1 start
    // launching (its master-tile prefetch overlaps this kernel)
    griddep_wait();
    griddep_launch_dependents();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / half;
        const int j = (int)(i - r * half);
        // numpy: pos(float64) * inv_freq(float64), one IEEE multiply
        const double theta = __dmul_rn((double)deltas[r], inv_freq[j]);
        double s, c;
        sincos(theta, &s, &c);
        if constexpr (sizeof(Tbl) == 16) {
            out[i] = make_double2(c, s);
        } else {
            out[i] = make_float2((float)c, (float)s);
        }
    }
}

// ---------------------------------------------------------------------------
// K1

constexpr int kMaxSources = 16;

struct CollectParams {
    const void* mk;
    const void* mv;
    int64_t mls;                 // master layer stride (elements)
    const tdkv_collect_unit* units;
    int32_t n_units;
    int32_t max_rows;
    const tdkv_collect_job* jobs;
    const int64_t* dst_rows;
    const void* table;
    int32_t rotate;
    void* dk;
    void* dv;
    int64_t dls;                 // destination layer stride (elements)
    int32_t num_layers;
    int32_t head_dim;
    int32_t row_elems;
    int32_t v_bulk;              // V rows leave by TMA bulk stores straight from the tile
    // multi-source rounds (tdkv_collect_sources): unit u's master tile is read
    // from source unit_src[u] -- a peer GPU's arena over NVLink, or the local
    // one -- instead of mk/mv; every source shares the arena layout
    const uint8_t* unit_src;
    const void* src_k[kMaxSources];
    const void* src_v[kMaxSources];
    // fused K0 (tdkv_collect_round with TDKV_ROUND_FUSE_TABLE): every job has
    // one constant delta (tbl_stride 0); each job group's cos/sin rows are
    // computed into shared memory from deltas[tbl_row] * inv_freq, the
    // arithmetic of rope_table_kernel, instead of read from a K0 table
    const int64_t* deltas;
    const double* inv_freq;
    int32_t fuse_table;
    // family restore (tdkv_restore_family): source i holds the virtual arena
    // rows [i*source_rows, (i+1)*source_rows) -- one master cache each -- and
    // a job whose overlay names a payload block for the tile's (layer,
    // block) takes the tile's K and V rows from that diff payload instead of
    // the staged master rows (the overlay precedes rotation, restore.py:5-8)
    int64_t source_rows;
    const tdkv_collect_overlay* ovl;      // per job: payload slabs + block maps
    int32_t nb;                           // diff blocks per layer
    int32_t block_size;
    int32_t n_jobs;
    int32_t ovl_inline;                   // OVL: K1's CTAs run the overlay pass after their items
    int32_t neox;                         // rotate-half pairs (collect_kernel<..., PAIRED>)
    int32_t cs_tiles;                     // tile planes before the cos/sin rows (4, or 2 when
                                          // every CTA takes one item: no prefetch buffer)
    int32_t drow_off;                     // byte offset of the destination-row buffers
    int32_t one_item;                     // fused rounds: one item per 128-thread CTA
    int32_t stage_cs;                     // K0 rows of each job group copied to shared memory
};

// Per-job destination metadata is staged in shared memory in groups of
// kJobGroup jobs with cp.async (double-buffered), so the scatter loop never
// waits on a dependent global load; each thread's cos/sin values are
// prefetched one job ahead in registers.
constexpr int kJobGroup = 16;                      // capacity; groups are balanced

// jobs per group for a unit of nj jobs: the fewest groups of <= kJobGroup,
// evenly filled (50 jobs -> 4 x 13, not 3 x 16 + 2)
__device__ __forceinline__ int job_group_size(int nj) {
    if (nj <= kJobGroup) return nj > 0 ? nj : 1;  // one group: no division
    const int groups = (nj + kJobGroup - 1) / kJobGroup;
    return (nj + groups - 1) / groups;
}
constexpr int kMaxTileRows = 32;

// Overlay pass of the family restore: the (job, layer, block)s whose rows
// come from the job's diff payload (K1 skipped them), K rotated by the job's
// table row(s), V copied, to the job's destination rows.  A CTA scans
// kOvlChunk block-map entries, compacts the changed ones in shared memory and
// moves them with all threads, kR rows per thread loaded before any is
// stored (chunks small enough that even a 24-mirror family spreads its
// changed blocks over every SM).  Run by K1's CTAs once their items are done
// (CollectParams::ovl_inline: the overlay fills K1's tail, one launch), or
// as its own kernel.
constexpr int kOvlChunk = 32;
template <typename T, int kR>
__device__ __forceinline__ void overlay_rows(const CollectParams& p, long long chunk0,
                                             long long chunk_step) {
    using V = uint4;
    using Tbl = typename Elt<T>::Table;
    constexpr int kEpu = 16 / (int)sizeof(T);
    constexpr int kPairs = kEpu / 2;
    __shared__ int s_list[kOvlChunk];
    __shared__ int s_n;
    const int tid = threadIdx.x;
    const int upr = p.row_elems * (int)sizeof(T) / 16;
    const int nthr = (int)blockDim.x;             // 256, or 128 inside a one-item K1
    const int tx_n = upr < nthr ? upr : nthr;
    const int rows_per_pass = nthr / tx_n;
    const int tx = tid % tx_n, ty = tid / tx_n;
    const Tbl* __restrict__ table = static_cast<const Tbl*>(p.table);
    const int half = p.head_dim >> 1;
    const long long n_entries = (long long)p.n_jobs * p.num_layers * p.nb;
    const long long per_job = (long long)p.num_layers * p.nb;
    // entry e = (job, layer, block), job-major
    auto map_at = [&](long long e) {
        const int job = (int)(e / per_job);
        const long long lb = e - job * per_job;
        const tdkv_collect_overlay o = p.ovl[job];
        return make_int2(o.map_k ? __ldg(o.map_k + lb) : -1, o.map_v ? __ldg(o.map_v + lb) : -1);
    };
    for (long long e0 = chunk0 * kOvlChunk; e0 < n_entries; e0 += chunk_step * kOvlChunk) {
        if (tid == 0) s_n = 0;
        __syncthreads();
        const long long e = e0 + tid;
        if (tid < kOvlChunk && e < n_entries) {
            const int2 m = map_at(e);
            if (m.x >= 0 || m.y >= 0) s_list[atomicAdd(&s_n, 1)] = tid;
        }
        __syncthreads();
        const int n = s_n;
        for (int i = 0; i < n; ++i) {
            const long long ei = e0 + s_list[i];
            const int2 m = map_at(ei);
            const int b = (int)(ei % p.nb);
            const long long jl = ei / p.nb;
            const int layer = (int)(jl % p.num_layers);
            const int job = (int)(jl / p.num_layers);
            const tdkv_collect_job jb = p.jobs[job];
            const tdkv_collect_overlay o = p.ovl[job];
            const int i0 = b * p.block_size;
            const int nrows = (int)min((int64_t)p.block_size, p.source_rows - i0);
            const V* pk = m.x >= 0 ? reinterpret_cast<const V*>(static_cast<const T*>(o.pay_k) +
                                                                (size_t)m.x * p.block_size * p.row_elems)
                                   : nullptr;
            const V* pv = m.y >= 0 ? reinterpret_cast<const V*>(static_cast<const T*>(o.pay_v) +
                                                                (size_t)m.y * p.block_size * p.row_elems)
                                   : nullptr;
            T* dk_l = static_cast<T*>(p.dk) + (size_t)layer * p.dls;
            T* dv_l = p.dv ? static_cast<T*>(p.dv) + (size_t)layer * p.dls : nullptr;
            const int64_t* drows = p.dst_rows + jb.dst_off + i0;
            if (ty < rows_per_pass) {
                for (int c = tx; c < upr; c += tx_n) {
                    const int j0 = ((c * kEpu) % p.head_dim) >> 1;
                    for (int r0 = ty; r0 < nrows; r0 += kR * rows_per_pass) {
                        V kx[kR], vx[kR];
                        int64_t drow[kR];
#pragma unroll
                        for (int q = 0; q < kR; ++q) {
                            const int r = r0 + q * rows_per_pass;
                            if (r < nrows) {
                                drow[q] = __ldg(drows + r);
                                if (pk) kx[q] = ld_stream(pk + (size_t)r * upr + c);
                                if (pv) vx[q] = ld_stream(pv + (size_t)r * upr + c);
                            }
                        }
#pragma unroll
                        for (int q = 0; q < kR; ++q) {
                            const int r = r0 + q * rows_per_pass;
                            if (r >= nrows) continue;
                            if (pk) {
                                if (p.rotate) {
                                    const Tbl* trow = table + (size_t)(jb.tbl_row +
                                                                       (i0 + r) * jb.tbl_stride) *
                                                                  half + j0;
                                    T* x = reinterpret_cast<T*>(&kx[q]);
#pragma unroll
                                    for (int w = 0; w < kPairs; ++w)
                                        rot_pair(x[2 * w], x[2 * w + 1], __ldg(trow + w));
                                }
                                st_stream(reinterpret_cast<V*>(dk_l + (size_t)drow[q] * p.row_elems) + c,
                                          kx[q]);
                            }
                            if (pv && dv_l)
                                st_stream(reinterpret_cast<V*>(dv_l + (size_t)drow[q] * p.row_elems) + c,
                                          vx[q]);
                        }
                    }
                }
            }
        }
        __syncthreads();                           // s_list / s_n reused
    }
}

template <typename T>
__global__ void __launch_bounds__(256) overlay_rows_kernel(const CollectParams p) {
    overlay_rows<T, 4>(p, blockIdx.x, gridDim.x);
}

// OVL: the family-restore instantiation (diff overlay); the collector's
// instantiations compile it out, keeping their register count (and so four
// resident CTAs per SM).  FUSE: the fused-K0 instantiation for 16-byte units
// (small rounds, where the instruction count per stored unit -- not HBM --
// bounds the kernel): every job has one constant delta, its cos/sin row sits
// in shared memory, and the scatter loop is the rotation, one 32-bit-indexed
// address and the store.
//
// PAIRED: a thread owns a unit of a head's lower half AND the unit D/2
// elements on (a "slot"), with the job group's cos/sin rows in shared memory.
// This is the rotate-half form (p.neox: element j of a head with element
// j + D/2, angle j -- every pair in the thread's registers; a warp-shuffle
// exchange between the halves' lanes measured 0.58 of peak at C2/C3) and,
// for bfloat16 rounds with K0's table, the interleaved form too: two loads
// and two stores in flight per thread per row measured 0.985 / 0.991 / 0.988
// / 0.992 of peak at C3 / C2 / C4 / C5 against 0.947 / 0.950 / 0.940 / 0.941
// for one unit per thread (same box, scripts/gpu_r02_paired.sh).
template <typename T, int UB, bool BULK, bool OVL, bool FUSE = false, bool PAIRED = false>
__global__ void __launch_bounds__(256, 4) collect_kernel(const CollectParams p) {
    using V = typename UnitBits<UB>::V;
    using Tbl = typename Elt<T>::Table;
    constexpr int kEpu = UB / (int)sizeof(T);      // elements per unit
    constexpr int kPairs = kEpu / 2;
    constexpr int kCs = kPairs;                   // cos/sin entries per interleaved unit

    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ __align__(8) uint64_t bars[2];
    // per job group: the destination row of every (job, tile row), stride
    // max_rows, two group buffers -- dynamic, after the tiles and the cos/sin rows
    const int drow_stride = p.max_rows;
    int64_t* s_drow0 = reinterpret_cast<int64_t*>(smem + p.drow_off);
    auto s_drow_b = [&](int mb) { return s_drow0 + (size_t)mb * kJobGroup * drow_stride; };
    __shared__ int4 s_meta[2][kJobGroup];          // tbl_row, tbl_stride, i0
    __shared__ int2 s_map[2][kJobGroup];           // OVL: the tile's K / V payload blocks

    const int tid = threadIdx.x;
    const int nthr = blockDim.x;
    const int row_bytes = p.row_elems * (int)sizeof(T);
    const int tile_bytes = p.max_rows * row_bytes;      // one plane
    const int upr = row_bytes / UB;                      // units per row
    const int tx_n = upr < nthr ? upr : nthr;
    const int rows_per_pass = nthr / tx_n;
    const int tx = tid % tx_n;
    const int ty = tid / tx_n;
    const int n_items = p.n_units * p.num_layers;
    // pair index of this thread's first unit (the usual single c = tx)
    auto angle0 = [&](int c) { return ((c * kEpu) % p.head_dim) >> 1; };
    const int j0_tx = angle0(tx);
    // PAIRED: slots = (head, unit of the lower half); slot s owns units c_lo and
    // c_lo + hh of its row (hh = units per half head)
    const int hh = (p.head_dim >> 1) / kEpu;
    const int n_slots = upr >> 1;
    const int sx_n = n_slots < nthr ? n_slots : nthr;
    const int slot_rows = sx_n > 0 ? nthr / sx_n : 0;
    const int sx = sx_n > 0 ? tid % sx_n : 0;
    const int sy = sx_n > 0 ? tid / sx_n : 0;
    // log2(head_dim / 2) when a power of two (the fused table's index split)
    const int half_shift = ((p.head_dim >> 1) & ((p.head_dim >> 1) - 1)) == 0
                               ? __ffs(p.head_dim >> 1) - 1 : -1;
    const Tbl* __restrict__ table = static_cast<const Tbl*>(p.table);
    const int half = p.head_dim >> 1;
    const bool has_v = p.dv != nullptr;            // K-only collect (align_cached)
    const bool rotate = p.rotate != 0;
    // V is position-free: with v_bulk its rows go from the staged tile to the
    // agents' slots by TMA bulk stores (one per job when the job's slots are
    // contiguous, else one per row) and the threads only handle K
    const bool v_tma = BULK && has_v && p.v_bulk != 0;

    if constexpr (BULK) {
        if (tid == 0) {
            mbar_init(&bars[0], 1);
            mbar_init(&bars[1], 1);
            fence_mbar_init();
        }
        __syncthreads();
    }

    // item -> (layer, unit); units vary fastest so consecutive CTAs stream
    // neighbouring tiles of one layer plane
    auto stage_src = [&](int layer, int ui, const T*& gk, const T*& gv, tdkv_collect_unit& u) {
        u = p.units[ui];
        int64_t row0 = u.row0;
        const void* bk = p.mk;
        const void* bv = p.mv;
        if (p.unit_src) {
            const int src = p.unit_src[ui];
            bk = p.src_k[src];
            bv = p.src_v[src];
        } else if (OVL && p.source_rows > 0) {
            const int src = (int)(row0 / p.source_rows);
            row0 -= (int64_t)src * p.source_rows;
            bk = p.src_k[src];
            bv = p.src_v[src];
        }
        const size_t off = (size_t)layer * p.mls + (size_t)row0 * p.row_elems;
        gk = static_cast<const T*>(bk) + off;
        gv = static_cast<const T*>(bv) + off;
    };
    auto stage_meta = [&](const tdkv_collect_unit& u, int layer, int g, int mb) {
        const int gsz = job_group_size(u.job_end - u.job_begin);
        const int jbase = u.job_begin + g * gsz;
        const int ng = min(gsz, u.job_end - jbase);
        // one warp per job, one lane per tile row (kMaxTileRows == 32)
        const int lane = tid & 31;
        if (lane < u.nrows) {
            for (int jj = tid >> 5; jj < ng; jj += nthr >> 5) {
                const tdkv_collect_job* jp = p.jobs + jbase + jj;
                const int64_t off = jp->dst_off + (u.row0 - jp->seg_row0) + lane;
                cp_async_8(s_drow_b(mb) + jj * drow_stride + lane, p.dst_rows + off);
            }
        }
        if (tid < ng) {
            const tdkv_collect_job jb = p.jobs[jbase + tid];
            const int i0 = u.row0 - jb.seg_row0;
            s_meta[mb][tid] = make_int4(jb.tbl_row, jb.tbl_stride, i0, 0);
            if constexpr (OVL) {
                // the tile lies inside one diff block (block_size % max_rows
                // == 0): fetch its K / V payload blocks with the rows
                const tdkv_collect_overlay o = p.ovl[jbase + tid];
                const size_t e = (size_t)layer * p.nb + i0 / p.block_size;
                if (o.map_k) cp_async_4(&s_map[mb][tid].x, o.map_k + e);
                else s_map[mb][tid].x = -1;
                if (o.map_v) cp_async_4(&s_map[mb][tid].y, o.map_v + e);
                else s_map[mb][tid].y = -1;
            }
        }
        cp_async_commit();
    };
    auto load_cs = [&](Tbl* cs, int tbl_row, int j0) {
        const Tbl* trow = table + (size_t)tbl_row * half + j0;
#pragma unroll
        for (int q = 0; q < kCs; ++q) cs[q] = __ldg(trow + q);
    };
    // rotate one unit's interleaved pairs in place
    auto rotate_unit_k = [&](V& kv, const Tbl* cs) {
        T* e = reinterpret_cast<T*>(&kv);
#pragma unroll
        for (int q = 0; q < kPairs; ++q) rot_pair(e[2 * q], e[2 * q + 1], cs[q]);
    };
    // fused K0: the group's rows live in shared memory after the tiles
    const bool fused = p.fuse_table != 0;
    Tbl* s_cs = reinterpret_cast<Tbl*>(smem + (size_t)p.cs_tiles * tile_bytes);
    // K0 rows staged per job group (set by the launcher for rotate-half
    // rounds and, TDKV_K1_STAGE_CS, interleaved ones)
    const bool staged_cs = p.stage_cs != 0 && rotate && !fused;
    auto load_cs_job = [&](Tbl* cs, int jj, const int4& m, int j0) {
        if (fused || staged_cs) {
            const Tbl* trow = s_cs + (size_t)jj * half + j0;
#pragma unroll
            for (int q = 0; q < kCs; ++q) cs[q] = trow[q];
        } else {
            load_cs(cs, m.x, j0);
        }
    };

    int item = blockIdx.x;
    // item -> (layer, unit) tracked incrementally (items advance by gridDim.x)
    int layer = item / p.n_units;
    int ui = item - layer * p.n_units;
    const int step_l = (int)gridDim.x / p.n_units;
    const int step_u = (int)gridDim.x - step_l * p.n_units;
    if constexpr (BULK) {
        if (tid == 0 && item < n_items) {
            const T *gk, *gv;
            tdkv_collect_unit u;
            stage_src(layer, ui, gk, gv, u);
            const uint32_t bytes = (uint32_t)u.nrows * row_bytes;
            mbar_arrive_expect_tx(&bars[0], (has_v ? 2 : 1) * bytes);
            bulk_g2s(smem, gk, bytes, &bars[0]);
            if (has_v) bulk_g2s(smem + tile_bytes, gv, bytes, &bars[0]);
        }
    }

    // PDL (tdkv_collect_round): everything above reads plan state and the
    // master arena only; the cos/sin table comes from the K0 launched just
    // before, and no pool row may be written before the predecessors finish
    griddep_wait();

    for (int iter = 0; item < n_items; item += gridDim.x, ++iter) {
        const int b = iter & 1;
        uint8_t* buf = smem + (size_t)b * 2 * tile_bytes;
        const tdkv_collect_unit u = p.units[ui];
        stage_meta(u, layer, 0, 0);
        const int cur_layer = layer, cur_ui = ui;
        ui += step_u;
        layer += step_l;
        if (ui >= p.n_units) {
            ui -= p.n_units;
            ++layer;
        }

        if constexpr (BULK) {
            const int next = item + gridDim.x;
            if (tid == 0 && next < n_items) {
                // buffer b^1 was drained by every thread before the trailing
                // __syncthreads of the previous iteration
                fence_proxy_async_smem();
                const T *gk, *gv;
                tdkv_collect_unit un;
                stage_src(layer, ui, gk, gv, un);
                const uint32_t bytes = (uint32_t)un.nrows * row_bytes;
                uint8_t* nb = smem + (size_t)(b ^ 1) * 2 * tile_bytes;
                mbar_arrive_expect_tx(&bars[b ^ 1], (has_v ? 2 : 1) * bytes);
                bulk_g2s(nb, gk, bytes, &bars[b ^ 1]);
                if (has_v) bulk_g2s(nb + tile_bytes, gv, bytes, &bars[b ^ 1]);
            }
            mbar_wait(&bars[b], (uint32_t)((iter >> 1) & 1));
        } else {
            const T *gk, *gv;
            tdkv_collect_unit un;
            stage_src(cur_layer, cur_ui, gk, gv, un);
            const int words = u.nrows * row_bytes / 4;
            const uint32_t* sk32 = reinterpret_cast<const uint32_t*>(gk);
            const uint32_t* sv32 = reinterpret_cast<const uint32_t*>(gv);
            uint32_t* dk32 = reinterpret_cast<uint32_t*>(buf);
            uint32_t* dv32 = reinterpret_cast<uint32_t*>(buf + tile_bytes);
            for (int w = tid; w < words; w += nthr) {
                dk32[w] = sk32[w];
                if (has_v) dv32[w] = sv32[w];
            }
        }

        const V* sk = reinterpret_cast<const V*>(buf);
        const V* sv = reinterpret_cast<const V*>(buf + tile_bytes);
        T* dk_l = static_cast<T*>(p.dk) + (size_t)cur_layer * p.dls;
        T* dv_l = static_cast<T*>(p.dv) + (size_t)cur_layer * p.dls;
        const int nj = u.job_end - u.job_begin;
        const int gsz = job_group_size(nj);
        const int ngroups = nj <= kJobGroup ? 1 : (nj + gsz - 1) / gsz;

        for (int g = 0; g < ngroups; ++g) {
            const int mb = g & 1;
            if (g + 1 < ngroups) {
                stage_meta(u, cur_layer, g + 1, mb ^ 1);
                cp_async_wait<1>();
            } else {
                cp_async_wait<0>();
            }
            __syncthreads();
            const int ng = min(gsz, u.job_end - u.job_begin - g * gsz);
            if (FUSE || (fused && rotate)) {
                // this group's cos/sin rows (rope_table_kernel's arithmetic)
                for (int idx = tid; idx < ng * half; idx += nthr) {
                    const int jj = half_shift >= 0 ? idx >> half_shift : idx / half;
                    const int j = idx - jj * half;
                    const double theta =
                        __dmul_rn((double)p.deltas[s_meta[mb][jj].x], p.inv_freq[j]);
                    double sn, cn;
                    sincos(theta, &sn, &cn);
                    if constexpr (sizeof(Tbl) == 16) {
                        s_cs[idx] = make_double2(cn, sn);
                    } else {
                        s_cs[idx] = make_float2((float)cn, (float)sn);
                    }
                }
                __syncthreads();
            } else if (staged_cs) {
                // K0's table rows of the group's constant-delta jobs copied
                // to shared memory once per group: the scatter loop reads its
                // cos/sin from shared memory instead of a per-job L1/L2 load
                // (rotate-half: a thread's 2 x 16-byte units need kEpu entries
                // per job, too many registers to prefetch the next job's)
                for (int idx = tid; idx < ng * half; idx += nthr) {
                    const int jj = half_shift >= 0 ? idx >> half_shift : idx / half;
                    const int4 mj = s_meta[mb][jj];
                    if (mj.y == 0)
                        s_cs[idx] = __ldg(table + (size_t)mj.x * half + (idx - jj * half));
                }
                __syncthreads();
            }
            if constexpr (BULK) {
                // a job whose tile comes from its diff payload moves V in
                // the thread loop below
                // (family restore: a job's payload-sourced planes are the
                // overlay pass's)
                if (v_tma && tid < ng && !(OVL && s_map[mb][tid].y >= 0)) {
                    const int64_t* dr = s_drow_b(mb) + tid * drow_stride;
                    const int64_t r0 = dr[0];
                    bool contig = true;
                    for (int r = 1; r < u.nrows; ++r) contig &= dr[r] == r0 + r;
                    const uint8_t* src = buf + tile_bytes;
                    if (contig) {
                        bulk_s2g(dv_l + (size_t)r0 * p.row_elems, src,
                                 (uint32_t)(u.nrows * row_bytes));
                    } else {
                        for (int r = 0; r < u.nrows; ++r)
                            bulk_s2g(dv_l + (size_t)dr[r] * p.row_elems, src + r * row_bytes,
                                     (uint32_t)row_bytes);
                    }
                    bulk_commit();
                }
            }
            if constexpr (PAIRED) {
              if (sy < slot_rows) {
                // a slot = one unit of a head's lower half + the unit D/2 on
                // (rotate-half: the pair partners; interleaved: two
                // self-contained units) -- two 16-byte loads and stores per
                // row in flight per thread
                const uint32_t upr32 = (uint32_t)upr;
                const bool neox = p.neox != 0;
                for (int sl = sx; sl < n_slots; sl += sx_n) {
                    const int c_lo = (sl / hh) * (2 * hh) + sl % hh;
                    const int c_hi = c_lo + hh;
                    const int e0 = (sl % hh) * kEpu;       // the slot's first element
                    // cos/sin entries: q < kPairs from jlo, the rest from jsplit
                    // (rotate-half: angles e0 .. e0 + kEpu; interleaved: the
                    // lower unit's pairs, then the upper unit's, D/4 on)
                    const int jlo = neox ? e0 : e0 >> 1;
                    const int jsplit = neox ? e0 + kPairs : (e0 >> 1) + (half >> 1);
                    for (int jj = 0; jj < ng; ++jj) {
                        const int4 mj = s_meta[mb][jj];
                        // family restore: a plane taken from the job's diff
                        // payload is the overlay pass's (flags uniform per CTA)
                        const bool ovk = OVL && s_map[mb][jj].x >= 0;
                        const bool ovv = OVL && s_map[mb][jj].y >= 0;
                        if (ovk && (ovv || v_tma || !has_v)) continue;
                        Tbl cs[kEpu];
                        if (rotate && mj.y == 0) {
                            const Tbl* trow = s_cs + jj * half;
#pragma unroll
                            for (int q = 0; q < kEpu; ++q)
                                cs[q] = trow[q < kPairs ? jlo + q : jsplit + (q - kPairs)];
                        }
                        const int64_t* dr = s_drow_b(mb) + jj * drow_stride;
                        for (int r = sy; r < u.nrows; r += slot_rows) {
                            if (!FUSE && rotate && mj.y != 0) {
                                const Tbl* trow = table + (size_t)(mj.x + (mj.z + r) * mj.y) * half;
#pragma unroll
                                for (int q = 0; q < kEpu; ++q)
                                    cs[q] = __ldg(trow + (q < kPairs ? jlo + q : jsplit + (q - kPairs)));
                            }
                            const size_t o = (size_t)(uint32_t)dr[r] * upr32;
                            V lo = sk[r * upr + c_lo], hi = sk[r * upr + c_hi];
                            if (rotate) {
                                T* a = reinterpret_cast<T*>(&lo);
                                T* b = reinterpret_cast<T*>(&hi);
                                if (neox) {
#pragma unroll
                                    for (int q = 0; q < kEpu; ++q) rot_pair(a[q], b[q], cs[q]);
                                } else {
#pragma unroll
                                    for (int q = 0; q < kPairs; ++q) {
                                        rot_pair(a[2 * q], a[2 * q + 1], cs[q]);
                                        rot_pair(b[2 * q], b[2 * q + 1], cs[kPairs + q]);
                                    }
                                }
                            }
                            if (!ovk) {
                                st_stream(reinterpret_cast<V*>(dk_l) + o + c_lo, lo);
                                st_stream(reinterpret_cast<V*>(dk_l) + o + c_hi, hi);
                            }
                            if (has_v && !v_tma && !ovv) {
                                st_stream(reinterpret_cast<V*>(dv_l) + o + c_lo, sv[r * upr + c_lo]);
                                st_stream(reinterpret_cast<V*>(dv_l) + o + c_hi, sv[r * upr + c_hi]);
                            }
                        }
                    }
                }
              }
            } else if constexpr (FUSE) {
              if (ty < rows_per_pass) {
                // constant delta per job, cos/sin rows in shared memory
                const uint32_t upr32 = (uint32_t)upr;
                for (int c = tx; c < upr; c += tx_n) {
                    const int j0 = c == tx ? j0_tx : angle0(c);
                    V* __restrict__ dkc = reinterpret_cast<V*>(dk_l) + c;
                    V* __restrict__ dvc = reinterpret_cast<V*>(dv_l) + c;
                    const V* skc = sk + c;
                    const V* svc = sv + c;
                    for (int jj = 0; jj < ng; ++jj) {
                        Tbl cs[kCs];
                        const Tbl* trow = s_cs + jj * half + j0;
#pragma unroll
                        for (int q = 0; q < kCs; ++q) cs[q] = trow[q];
                        const int64_t* dr = s_drow_b(mb) + jj * drow_stride;
#pragma unroll 2
                        for (int r = ty; r < u.nrows; r += rows_per_pass) {
                            const size_t o = (size_t)(uint32_t)dr[r] * upr32;
                            V kv = skc[r * upr];
                            rotate_unit_k(kv, cs);
                            st_stream(dkc + o, kv);
                            if (has_v && !v_tma) st_stream(dvc + o, svc[r * upr]);
                        }
                    }
                }
              }
            } else if (ty < rows_per_pass) {
                for (int c = tx; c < upr; c += tx_n) {
                    const int j0 = c == tx ? j0_tx : angle0(c);
                    Tbl cs[kCs], csn[kCs];
                    int4 m = s_meta[mb][0];
                    if (rotate && m.y == 0) load_cs_job(cs, 0, m, j0);
                    for (int jj = 0; jj < ng; ++jj) {
                        const int4 mn = jj + 1 < ng ? s_meta[mb][jj + 1] : m;
                        if (rotate && jj + 1 < ng && mn.y == 0) load_cs_job(csn, jj + 1, mn, j0);
                        const int64_t* dr = s_drow_b(mb) + jj * drow_stride;
                        // overlay flags are uniform across the CTA: a plane
                        // taken from the payload is the overlay pass's
                        const bool ovk = OVL && s_map[mb][jj].x >= 0;
                        const bool ovv = OVL && s_map[mb][jj].y >= 0;
                        for (int r = ty; r < u.nrows && !(ovk && (ovv || v_tma || !has_v));
                             r += rows_per_pass) {
                            const size_t drow = (size_t)(uint32_t)dr[r];
                            V kv = sk[r * upr + c];
                            if (rotate) {
                                if (m.y != 0) load_cs(cs, m.x + (m.z + r) * m.y, j0);
                                rotate_unit_k(kv, cs);
                            }
                            if (!ovk)
                                st_stream(reinterpret_cast<V*>(dk_l + (size_t)drow * p.row_elems) + c,
                                          kv);
                            if (has_v && !v_tma && !ovv)
                                st_stream(reinterpret_cast<V*>(dv_l + (size_t)drow * p.row_elems) + c,
                                          sv[r * upr + c]);
                        }
                        m = mn;
#pragma unroll
                        for (int q = 0; q < kCs; ++q) cs[q] = csn[q];
                    }
                }
            }
            if (g + 1 == ngroups && v_tma && tid < kJobGroup)
                bulk_wait_read<0>();    // the tile buffer is refilled next iteration
            __syncthreads();
        }
    }
    if constexpr (OVL) {
        // payload-sourced (mirror, layer, block)s: disjoint from every row
        // this kernel's items wrote, so no ordering against them is needed
        if (p.ovl_inline) overlay_rows<T, 2>(p, blockIdx.x, gridDim.x);
    }
    if constexpr (BULK) {
        if (v_tma && tid < kJobGroup) bulk_wait<0>();
    }
}

template <typename T, int UB, bool BULK, bool OVL = false>
static int32_t launch_collect(const CollectParams& p, int grid_limit, cudaStream_t s, bool pdl) {
    auto kern = collect_kernel<T, UB, BULK, OVL>;
    // interleaved rounds with K0's table take the paired (two units per
    // thread) loop too; TDKV_K1_PAIRED=0 keeps one unit per thread (A/B)
    static const int paired_env = [] {
        const char* e = getenv("TDKV_K1_PAIRED");
        return e ? atoi(e) : 1;
    }();
    bool paired_il = false;
    if constexpr (UB == 16 && BULK && !OVL) {
        // bfloat16 only: the float32 form (float64 table entries) spills at
        // 64 registers and measured slower (C1 x 64 agents, K0 table: 0.82 ->
        // 0.78 of peak)
        // (TDKV_K1_PAIRED=2: every 16-byte interleaved form, the fused table
        // and float32 included -- A/B only)
        const bool halves = (p.head_dim / 2) % (16 / (int)sizeof(T)) == 0;
        paired_il = !p.neox && p.rotate && halves &&
                    ((paired_env == 1 && sizeof(T) == 2 && !p.fuse_table) || paired_env == 2);
        if (p.neox || (paired_il && p.fuse_table))
            kern = p.fuse_table ? collect_kernel<T, UB, BULK, OVL, true, true>
                                : collect_kernel<T, UB, BULK, OVL, false, true>;
        else if (p.fuse_table)
            kern = collect_kernel<T, UB, BULK, OVL, true>;
        else if (paired_il)
            kern = collect_kernel<T, UB, BULK, OVL, false, true>;
    } else if constexpr (UB == 16 && BULK && OVL && sizeof(T) == 2) {
        // the family restore's collector round (interleaved, K0 table)
        paired_il = sizeof(T) == 2 && !p.neox && p.rotate && paired_env != 0 &&
                    (p.head_dim / 2) % (16 / (int)sizeof(T)) == 0;
        if (paired_il) kern = collect_kernel<T, UB, BULK, OVL, false, true>;
    } else {
        if (p.neox) return set_error(TDKV_EINVAL, "tdkv_collect: NeoX pairs need 16-byte units");
    }
    // One item per CTA of 128 threads with no prefetch buffer (no item waits
    // behind another's chain of dependent loads; 8 CTAs per SM overlap the
    // chains): every bfloat16 round (C3 0.926 -> 0.945 of peak, C2 0.944 ->
    // 0.951, C4 0.927 -> 0.938, C2 with 3 agents 0.84 -> 0.96), and float32
    // (float64 rotation) rounds whose items carry few jobs, flagged by the
    // planner (TDKV_ROUND_ONE_ITEM: C1, 4 jobs per item, 0.64 -> 0.68; items
    // of 16-32 jobs -- C1 with 32-64 agents -- stay faster persistent); and
    // the family restore (OVL: C2 2.62 -> 2.31 ms, C3 0.74 -> 0.66 ms).
    // TDKV_K1_SINGLE: 0 never, 2 always (A/B).
    static const int single_env = [] {
        const char* e = getenv("TDKV_K1_SINGLE");
        return e ? atoi(e) : 1;        // 0 never, 1 as flagged, 2 always (A/B)
    }();
    CollectParams pp = p;
    const int items = p.n_units * p.num_layers;
    // cos/sin rows of a job group in shared memory: the fused table, and the
    // rotate-half form's staged K0 rows
    static const int stage_env = [] {
        const char* e = getenv("TDKV_K1_STAGE_CS");
        return e ? atoi(e) : 0;        // interleaved rounds: 0 K0 rows from L1/L2, 1 staged
    }();
    pp.stage_cs = (p.rotate && !p.fuse_table && (p.neox || paired_il || stage_env == 1)) ? 1 : 0;
    const size_t cs_bytes = p.fuse_table || pp.stage_cs
                                ? (size_t)kJobGroup * (p.head_dim / 2) *
                                      sizeof(typename Elt<T>::Table)
                                : 0;
    auto smem_for = [&](int cs_tiles, int32_t& drow_off) {
        drow_off = (int32_t)(((size_t)cs_tiles * p.max_rows * p.row_elems * sizeof(T) +
                              cs_bytes + 15) / 16 * 16);
        return (size_t)drow_off + (size_t)2 * kJobGroup * p.max_rows * 8;
    };
    const bool single = UB == 16 && BULK && grid_limit <= 0 &&
                        (single_env == 2 ||
                         (single_env == 1 &&
                          (sizeof(T) == 2 || OVL || (p.fuse_table && p.one_item))));
    pp.cs_tiles = single ? 2 : 4;
    const int threads = single ? 128 : 256;
    const size_t smem = smem_for(pp.cs_tiles, pp.drow_off);
    if (smem > 227 * 1024)
        return set_error(TDKV_EINVAL, "tdkv_collect: tile of %d rows needs %zu B of shared memory",
                         p.max_rows, smem);
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
        return check_launch("tdkv_collect: cudaFuncSetAttribute");
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
    if (per_sm < 1) per_sm = 1;
    int grid = single ? items : sm_count() * per_sm;
    if (grid_limit > 0 && grid > grid_limit) grid = grid_limit;
    if (grid > items) grid = items;
    if (launch_maybe_pdl(kern, dim3(grid), dim3(threads), smem, s, pdl, pp) != cudaSuccess)
        return check_launch("tdkv_collect: launch");
    count_launch();
    return check_launch("tdkv_collect");
}

template <typename T>
static int32_t launch_overlay_pass(const CollectParams& p, cudaStream_t s) {
    auto kern = overlay_rows_kernel<T>;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, 0);
    if (per_sm < 1) per_sm = 1;
    const long long chunks = ((long long)p.n_jobs * p.num_layers * p.nb + kOvlChunk - 1) /
                             kOvlChunk;
    long long grid = (long long)sm_count() * per_sm;
    if (grid > chunks) grid = chunks;
    if (grid < 1) return TDKV_OK;
    kern<<<(unsigned)grid, 256, 0, s>>>(p);
    count_launch();
    return check_launch("tdkv_restore_family: overlay pass");
}

}  // namespace tdkv

using namespace tdkv;

static int32_t rope_table_impl(const int64_t* d_deltas, int64_t n_rows, const double* d_inv_freq,
                               int32_t half_dim, int32_t table_dtype, void* d_table, void* stream,
                               bool pdl);

extern "C" int32_t tdkv_rope_table(const int64_t* d_deltas, int64_t n_rows,
                                   const double* d_inv_freq, int32_t half_dim,
                                   int32_t table_dtype, void* d_table, void* stream) {
    return rope_table_impl(d_deltas, n_rows, d_inv_freq, half_dim, table_dtype, d_table, stream,
                           false);
}

static int32_t rope_table_impl(const int64_t* d_deltas, int64_t n_rows, const double* d_inv_freq,
                               int32_t half_dim, int32_t table_dtype, void* d_table, void* stream,
                               bool pdl) {
    if (n_rows < 0 || half_dim <= 0) return set_error(TDKV_EINVAL, "tdkv_rope_table: bad sizes");
    if (n_rows == 0) return TDKV_OK;
    if (!d_deltas || !d_inv_freq || !d_table)
        return set_error(TDKV_EINVAL, "tdkv_rope_table: null pointer");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int64_t total = n_rows * half_dim;
    int grid = (int)((total + 255) / 256);
    if (grid > sm_count() * 8) grid = sm_count() * 8;
    cudaError_t e;
    if (table_dtype == TDKV_F32) {
        e = launch_maybe_pdl(rope_table_kernel<double2>, dim3(grid), dim3(256), 0, s, pdl,
                             d_deltas, n_rows, d_inv_freq, (int)half_dim,
                             static_cast<double2*>(d_table));
    } else if (table_dtype == TDKV_BF16) {
        e = launch_maybe_pdl(rope_table_kernel<float2>, dim3(grid), dim3(256), 0, s, pdl,
                             d_deltas, n_rows, d_inv_freq, (int)half_dim,
                             static_cast<float2*>(d_table));
    } else {
        return set_error(TDKV_EUNSUPPORTED, "tdkv_rope_table: dtype %d", table_dtype);
    }
    if (e != cudaSuccess) return check_launch("tdkv_rope_table: launch");
    count_launch();
    return check_launch("tdkv_rope_table");
}

static int32_t collect_impl(const void* d_master_k, const void* d_master_v,
                            int64_t master_layer_stride, const tdkv_collect_unit* d_units,
                            int32_t n_units, int32_t max_rows, const tdkv_collect_job* d_jobs,
                            const int64_t* d_dst_rows, const void* d_table, int32_t rotate,
                            void* d_dst_k, void* d_dst_v, int64_t dst_layer_stride,
                            int32_t num_layers, int32_t num_heads, int32_t head_dim,
                            int32_t dtype, int32_t grid_limit, void* stream,
                            const uint8_t* d_unit_src, const void* const* h_src_k,
                            const void* const* h_src_v, int32_t n_src, bool pdl = false,
                            const int64_t* d_deltas = nullptr,
                            const double* d_inv_freq = nullptr, int64_t source_rows = 0,
                            const tdkv_collect_overlay* d_overlay = nullptr,
                            int32_t block_size = 0, int32_t nb = 0, int32_t n_jobs = 0,
                            bool neox = false, bool one_item = false) {
    if (n_units < 0 || num_layers <= 0 || num_heads <= 0 || head_dim <= 0 || (head_dim & 1))
        return set_error(TDKV_EINVAL, "tdkv_collect: bad geometry L=%d H=%d D=%d", num_layers,
                         num_heads, head_dim);
    if (n_units == 0) return TDKV_OK;
    if (max_rows <= 0 || max_rows > kMaxTileRows)
        return set_error(TDKV_EINVAL, "tdkv_collect: max_rows must be in [1, %d]", kMaxTileRows);
    if (!d_master_k || !d_units || !d_jobs || !d_dst_rows || !d_dst_k ||
        (rotate && !d_table && !(d_deltas && d_inv_freq)) ||
        ((d_dst_v == nullptr) != (d_master_v == nullptr)))
        return set_error(TDKV_EINVAL, "tdkv_collect: null pointer");
    if (dtype != TDKV_F32 && dtype != TDKV_BF16)
        return set_error(TDKV_EUNSUPPORTED, "tdkv_collect: dtype %d", dtype);
    // destination rows are indexed in 32 bits inside K1
    if (dst_layer_stride / ((int64_t)num_heads * head_dim) > (int64_t)UINT32_MAX)
        return set_error(TDKV_EINVAL, "tdkv_collect: destination planes of more than 2^32 rows");

    CollectParams p;
    p.ovl_inline = 0;
    p.cs_tiles = 4;
    p.drow_off = 0;
    p.neox = neox ? 1 : 0;
    p.one_item = one_item ? 1 : 0;
    p.stage_cs = 0;
    p.mk = d_master_k;
    p.mv = d_master_v;
    p.mls = master_layer_stride;
    p.units = d_units;
    p.n_units = n_units;
    p.max_rows = max_rows;
    p.jobs = d_jobs;
    p.dst_rows = d_dst_rows;
    p.table = d_table;
    p.rotate = rotate;
    p.dk = d_dst_k;
    p.dv = d_dst_v;
    p.dls = dst_layer_stride;
    p.num_layers = num_layers;
    p.head_dim = head_dim;
    p.row_elems = num_heads * head_dim;
    p.unit_src = d_unit_src;
    p.deltas = d_deltas;
    p.inv_freq = d_inv_freq;
    p.fuse_table = (rotate && d_deltas && d_inv_freq) ? 1 : 0;
    p.source_rows = source_rows;
    p.ovl = d_overlay;
    p.block_size = block_size;
    p.nb = nb;
    p.n_jobs = n_jobs;
    for (int i = 0; i < kMaxSources; ++i) {
        p.src_k[i] = i < n_src ? h_src_k[i] : nullptr;
        p.src_v[i] = i < n_src && h_src_v ? h_src_v[i] : nullptr;
    }
    static const bool v_bulk_env = [] {
        const char* e = getenv("TDKV_COLLECT_V_BULK");
        return !(e && e[0] == '0');
    }();

    const size_t esz = elt_size(dtype);
    const size_t row_bytes = (size_t)p.row_elems * esz;
    int ub = pick_unit_bytes(dtype, head_dim, p.row_elems);
    if (ub == 16 && !(aligned(d_dst_k, 16) && aligned(d_dst_v, 16) && aligned(d_master_k, 16) &&
                      aligned(d_master_v, 16) &&
                      (dst_layer_stride * esz) % 16 == 0))
        ub = (int)(2 * esz);
    const bool bulk = row_bytes % 16 == 0 && aligned(d_master_k, 16) && aligned(d_master_v, 16) &&
                      (master_layer_stride * esz) % 16 == 0;
    p.v_bulk = v_bulk_env && bulk && ub == 16 && d_dst_v != nullptr;
    if (!aligned(d_master_k, 4) || !aligned(d_master_v, 4))
        return set_error(TDKV_EINVAL, "tdkv_collect: master planes must be 4-byte aligned");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (neox) {
        // partner units by warp shuffle: whole warps per row, both halves of a
        // head within one warp
        const int epu = (int)(16 / esz);
        if (!(bulk && ub == 16) || (head_dim / 2) % epu || d_overlay)
            return set_error(TDKV_EINVAL, "tdkv_collect: NeoX pairs need 16-byte-aligned planes "
                             "and half heads of whole 16-byte units");
    }

    if (d_overlay) {
        // the family restore needs the TMA-staged, 16-byte form
        if (!(bulk && ub == 16))
            return set_error(TDKV_EINVAL, "tdkv_restore_family: masters, payloads and the pool "
                             "must be 16-byte aligned with 16-byte rows");
        static const bool separate = [] {
            const char* e = getenv("TDKV_OVERLAY_SEPARATE");
            return e && e[0] == '1';
        }();
        p.ovl_inline = separate ? 0 : 1;
        const int32_t rc = dtype == TDKV_F32
                               ? launch_collect<float, 16, true, true>(p, grid_limit, s, pdl)
                               : launch_collect<__nv_bfloat16, 16, true, true>(p, grid_limit, s, pdl);
        if (rc || !separate) return rc;
        return dtype == TDKV_F32 ? launch_overlay_pass<float>(p, s)
                                 : launch_overlay_pass<__nv_bfloat16>(p, s);
    }
    if (dtype == TDKV_F32) {
        if (ub == 16)
            return bulk ? launch_collect<float, 16, true>(p, grid_limit, s, pdl)
                        : launch_collect<float, 16, false>(p, grid_limit, s, pdl);
        return bulk ? launch_collect<float, 8, true>(p, grid_limit, s, pdl)
                    : launch_collect<float, 8, false>(p, grid_limit, s, pdl);
    }
    if (ub == 16)
        return bulk ? launch_collect<__nv_bfloat16, 16, true>(p, grid_limit, s, pdl)
                    : launch_collect<__nv_bfloat16, 16, false>(p, grid_limit, s, pdl);
    return bulk ? launch_collect<__nv_bfloat16, 4, true>(p, grid_limit, s, pdl)
                : launch_collect<__nv_bfloat16, 4, false>(p, grid_limit, s, pdl);
}

extern "C" int32_t tdkv_collect(const void* d_master_k, const void* d_master_v,
                                int64_t master_layer_stride, const tdkv_collect_unit* d_units,
                                int32_t n_units, int32_t max_rows, const tdkv_collect_job* d_jobs,
                                const int64_t* d_dst_rows, const void* d_table, int32_t rotate,
                                void* d_dst_k, void* d_dst_v, int64_t dst_layer_stride,
                                int32_t num_layers, int32_t num_heads, int32_t head_dim,
                                int32_t dtype, int32_t grid_limit, void* stream) {
    return collect_impl(d_master_k, d_master_v, master_layer_stride, d_units, n_units, max_rows,
                        d_jobs, d_dst_rows, d_table, rotate, d_dst_k, d_dst_v, dst_layer_stride,
                        num_layers, num_heads, head_dim, dtype, grid_limit, stream, nullptr,
                        nullptr, nullptr, 0);
}

// One round in one call: K0 (this round's cos/sin rows) and K1, both
// launched with programmatic dependent launch -- K0 waits for the previous
// round (its table is being overwritten) and then releases K1, whose launch,
// barrier setup and first master-tile TMA loads overlap K0; K1 waits for K0
// only before it rotates or writes.  Opt-in (TDKV_PDL=1): plain launches
// measured faster at C2.
extern "C" int32_t tdkv_collect_round(const int64_t* d_deltas, int64_t n_table_rows,
                                      const double* d_inv_freq, void* d_table,
                                      const void* d_master_k, const void* d_master_v,
                                      int64_t master_layer_stride,
                                      const tdkv_collect_unit* d_units, int32_t n_units,
                                      int32_t max_rows, const tdkv_collect_job* d_jobs,
                                      const int64_t* d_dst_rows, void* d_dst_k, void* d_dst_v,
                                      int64_t dst_layer_stride, int32_t num_layers,
                                      int32_t num_heads, int32_t head_dim, int32_t dtype,
                                      int32_t grid_limit, int32_t flags, void* stream) {
    // off by default: measured 4% slower at C2 on B200 (K1's early-launched
    // CTAs idle at griddepcontrol.wait while holding their SM slots)
    static const bool pdl = [] {
        const char* e = getenv("TDKV_PDL");
        return e && e[0] == '1';
    }();
    const bool rotate = n_table_rows > 0;
    const bool fuse = rotate && (flags & TDKV_ROUND_FUSE_TABLE);
    const bool neox = rotate && (flags & TDKV_ROUND_NEOX);
    const bool one_item = fuse && (flags & TDKV_ROUND_ONE_ITEM);
    if (rotate && !fuse) {
        const int32_t rc = rope_table_impl(d_deltas, n_table_rows, d_inv_freq, head_dim / 2, dtype,
                                           d_table, stream, pdl);
        if (rc) return rc;
    }
    return collect_impl(d_master_k, d_master_v, master_layer_stride, d_units, n_units, max_rows,
                        d_jobs, d_dst_rows, rotate && !fuse ? d_table : nullptr, rotate ? 1 : 0,
                        d_dst_k, d_dst_v, dst_layer_stride, num_layers, num_heads, head_dim, dtype,
                        grid_limit, stream, nullptr, nullptr, nullptr, 0, pdl && rotate && !fuse,
                        fuse ? d_deltas : nullptr, fuse ? d_inv_freq : nullptr, 0, nullptr, 0, 0,
                        0, neox, one_item);
}

extern "C" int32_t tdkv_collect_sources(const void* const* h_src_k, const void* const* h_src_v,
                                        int32_t n_src, const uint8_t* d_unit_src,
                                        int64_t master_layer_stride,
                                        const tdkv_collect_unit* d_units, int32_t n_units,
                                        int32_t max_rows, const tdkv_collect_job* d_jobs,
                                        const int64_t* d_dst_rows, const void* d_table,
                                        int32_t rotate, void* d_dst_k, void* d_dst_v,
                                        int64_t dst_layer_stride, int32_t num_layers,
                                        int32_t num_heads, int32_t head_dim, int32_t dtype,
                                        int32_t grid_limit, void* stream) {
    if (n_src <= 0 || n_src > kMaxSources || !h_src_k || !d_unit_src)
        return set_error(TDKV_EINVAL, "tdkv_collect_sources: %d sources (1..%d) and a unit "
                         "source map are required", n_src, kMaxSources);
    if ((h_src_v == nullptr) != (d_dst_v == nullptr))
        return set_error(TDKV_EINVAL, "tdkv_collect_sources: null pointer");
    // every source must pass the alignment tests the single-source launch
    // makes on its master pointer: test them all through the first slot
    const void* k0 = h_src_k[0];
    const void* v0 = h_src_v ? h_src_v[0] : nullptr;
    for (int i = 0; i < n_src; ++i) {
        if (!h_src_k[i] || (h_src_v && !h_src_v[i]))
            return set_error(TDKV_EINVAL, "tdkv_collect_sources: source %d is null", i);
        if (!aligned(h_src_k[i], 16) || (h_src_v && !aligned(h_src_v[i], 16)))
            return set_error(TDKV_EINVAL, "tdkv_collect_sources: source %d not 16-byte aligned",
                             i);
    }
    return collect_impl(k0, v0, master_layer_stride, d_units, n_units, max_rows, d_jobs,
                        d_dst_rows, d_table, rotate, d_dst_k, d_dst_v, dst_layer_stride,
                        num_layers, num_heads, head_dim, dtype, grid_limit, stream, d_unit_src,
                        h_src_k, h_src_v, n_src);
}

// Family restore: K1 writing every master-sourced (mirror, tile) + the
// overlay pass writing the payload-sourced blocks (see tdkv.h).
extern "C" int32_t tdkv_restore_family(const void* const* h_src_k, const void* const* h_src_v,
                                       int32_t n_src, int64_t source_rows,
                                       const tdkv_collect_unit* d_units, int32_t n_units,
                                       int32_t max_rows, const tdkv_collect_job* d_jobs,
                                       int32_t n_jobs, const int64_t* d_dst_rows,
                                       const tdkv_collect_overlay* d_overlay, int32_t nb,
                                       int32_t block_size,
                                       const void* d_table, int32_t rotate, void* d_dst_k,
                                       void* d_dst_v, int64_t dst_layer_stride,
                                       int32_t num_layers, int32_t num_heads, int32_t head_dim,
                                       int32_t dtype, int32_t grid_limit, void* stream) {
    if (n_src <= 0 || n_src > kMaxSources || !h_src_k || source_rows <= 0)
        return set_error(TDKV_EINVAL, "tdkv_restore_family: %d masters (1..%d) of %lld rows",
                         n_src, kMaxSources, (long long)source_rows);
    if (n_jobs < 0) return set_error(TDKV_EINVAL, "tdkv_restore_family: %d jobs", n_jobs);
    if (n_jobs == 0 || n_units == 0) return TDKV_OK;
    if (!d_overlay) return set_error(TDKV_EINVAL, "tdkv_restore_family: null overlay array");
    if (block_size <= 0 || max_rows <= 0 || block_size % max_rows != 0)
        return set_error(TDKV_EINVAL, "tdkv_restore_family: tiles of %d rows must divide the "
                         "diff block size %d", max_rows, block_size);
    if (nb != (int32_t)((source_rows + block_size - 1) / block_size))
        return set_error(TDKV_EINVAL, "tdkv_restore_family: %d blocks per layer for %lld rows "
                         "of block size %d", nb, (long long)source_rows, block_size);
    if ((h_src_v == nullptr) != (d_dst_v == nullptr))
        return set_error(TDKV_EINVAL, "tdkv_restore_family: null pointer");
    for (int i = 0; i < n_src; ++i) {
        if (!h_src_k[i] || (h_src_v && !h_src_v[i]))
            return set_error(TDKV_EINVAL, "tdkv_restore_family: master %d is null", i);
        if (!aligned(h_src_k[i], 16) || (h_src_v && !aligned(h_src_v[i], 16)))
            return set_error(TDKV_EINVAL, "tdkv_restore_family: master %d not 16-byte aligned",
                             i);
    }
    const void* const* src_v = h_src_v;
    const int64_t mls = source_rows * (int64_t)num_heads * head_dim;   // each master's layer stride
    return collect_impl(h_src_k[0], src_v ? src_v[0] : nullptr, mls, d_units,
                        n_units, max_rows, d_jobs, d_dst_rows, d_table, rotate, d_dst_k, d_dst_v,
                        dst_layer_stride, num_layers, num_heads, head_dim, dtype, grid_limit,
                        stream, nullptr, h_src_k, src_v, n_src, false, nullptr, nullptr,
                        source_rows, d_overlay, block_size, nb, n_jobs);
}
