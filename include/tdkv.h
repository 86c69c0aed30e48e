/*
 * tdkv.h -- C-ABI of the B200 KV Collector + block-sparse diff codec.
 *
 * Drop-in boundary for the hot path of TokenDance's reference package
 * ``roundkv`` 0.1.0 (paths below are relative to /root/reference/pkg/src/roundkv).
 * The reference has no FFI layer (it is pure Python + numpy);
 * each entry point below is what a binding for the named Python function
 * would call.  INTEGRATION.md shows the ctypes binding.
 *
 * Conventions
 *   - Plain pointers and sizes only.  Pointers prefixed ``d_`` are device
 *     pointers; everything else is host memory.  ``stream`` is a cudaStream_t
 *     passed as void* (NULL = legacy default stream).
 *   - Every function returns 0 on success or a TDKV_E* code; a message for
 *     the most recent failure on the calling thread is available from
 *     tdkv_last_error().  No call synchronizes the stream.
 *   - KV planes are (num_layers, rows, num_heads, head_dim) with a given
 *     layer stride in ELEMENTS; a "row" is one token's H*D elements.
 *   - dtype: TDKV_F32 (rotation evaluated in float64 with one final
 *     round-to-nearest, bit-compatible with toymodel.py:60-83) or TDKV_BF16
 *     (rotation in float32 with float32 cos/sin derived from the float64
 *     angle, result rounded to bf16).
 *   - Rotary pairs are interleaved (2j, 2j+1) (toymodel.py:78-82).
 *   - Reentrant: no global mutable state except a launch counter.
 */
#ifndef TDKV_H
#define TDKV_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TDKV_F32 0
#define TDKV_BF16 1

#define TDKV_OK 0
#define TDKV_EINVAL 1     /* bad argument (shape, pointer, alignment) */
#define TDKV_EUNSUPPORTED 2
#define TDKV_ECUDA 3      /* a CUDA launch/runtime error */
#define TDKV_ENOSLOTS 4   /* allocator: not enough free slots */

#define TDKV_NO_VIOLATION 0x7f7f7f7f

/* Library version, (major << 16) | minor. */
int32_t tdkv_version(void);
/* Message for the last failing call on this thread ("" if none). */
const char* tdkv_last_error(void);
/* Number of kernels this library has launched in the process so far. */
int64_t tdkv_launch_count(void);
/* 1 when p lies in page-locked host memory (cudaHostAlloc / cudaHostRegister),
 * else 0.  Lets a caller holding a wire image in pinned memory skip the
 * staging copy of deserialize_to_device (diffstore.py:242-306 parses from a
 * bytes object; the GPU form moves the image over PCIe). */
int32_t tdkv_host_is_pinned(const void* p);
/* Asynchronous host -> device copy of nbytes on `stream` (full PCIe rate
 * only from page-locked memory). */
int32_t tdkv_copy_h2d(void* d_dst, const void* h_src, int64_t nbytes, void* stream);

/* ------------------------------------------------------------------------
 * K0  rotary table.  Replaces the angle/cos/sin part of rope_apply
 * (toymodel.py:73-77).  For each row r and pair j:
 *     theta = (double)d_deltas[r] * d_inv_freq[j]         (IEEE mul)
 *     table[r][j] = (cos theta, sin theta)
 * stored as double2 (table_dtype TDKV_F32) or float2 (TDKV_BF16).
 * d_inv_freq holds base^(-2j/D) computed by the caller (toymodel.py:74).
 * ---------------------------------------------------------------------- */
int32_t tdkv_rope_table(const int64_t* d_deltas, int64_t n_rows,
                        const double* d_inv_freq, int32_t half_dim,
                        int32_t table_dtype, void* d_table, void* stream);

/* ------------------------------------------------------------------------
 * K1  KV Collector.  Replaces pic.align_cached (pic.py:208-235) fused with
 * the _skeleton V copy (pic.py:203-204) and PagedPool.write_rows
 * (paged_pool.py:150-156, reached via trace._write_cache trace.py:148-152).
 *
 * The master arena holds every shared segment's cached rows:
 * d_master_{k,v}[layer * master_layer_stride + row * H * D + e].
 * A unit is a tile of <= max_rows consecutive arena rows of ONE segment
 * plus a range of jobs [job_begin, job_end) that hold that segment; the
 * tile is staged once in shared memory (cp.async.bulk) and written to every
 * job.  For job j and segment-relative token i the destination row is
 * d_dst_rows[job.dst_off + i] and the cos/sin row is
 * job.tbl_row + i * job.tbl_stride.  rotate == 0 copies K unchanged (the
 * reference skips rope_apply when every delta is zero, pic.py:228).
 * ---------------------------------------------------------------------- */
typedef struct {
    int64_t dst_off;     /* index of token 0 of this job in d_dst_rows */
    int32_t seg_row0;    /* arena row of token 0 of the job's segment */
    int32_t tbl_row;     /* cos/sin row of token 0 */
    int32_t tbl_stride;  /* 0: one delta for the whole job, 1: per token */
    int32_t pad_;
} tdkv_collect_job;

typedef struct {
    int32_t row0;        /* first arena row of the tile */
    int32_t nrows;       /* rows in the tile (<= max_rows) */
    int32_t job_begin;
    int32_t job_end;
} tdkv_collect_unit;

int32_t tdkv_collect(const void* d_master_k, const void* d_master_v,
                     int64_t master_layer_stride,
                     const tdkv_collect_unit* d_units, int32_t n_units,
                     int32_t max_rows,
                     const tdkv_collect_job* d_jobs, const int64_t* d_dst_rows,
                     const void* d_table, int32_t rotate,
                     void* d_dst_k, void* d_dst_v, int64_t dst_layer_stride,
                     int32_t num_layers, int32_t num_heads, int32_t head_dim,
                     int32_t dtype, int32_t grid_limit, void* stream);

/* One round in one call (replaces the K0 + K1 pair of a collector round,
 * pic.py:208-235): tdkv_rope_table over d_deltas[n_table_rows] into d_table
 * (n_table_rows = 0: no rotation, K1 alone), then tdkv_collect with that
 * table.  With TDKV_PDL=1 both kernels are launched with programmatic
 * dependent launch (K1's launch and first master-tile loads overlap K0, K0
 * waits for the previous kernels before overwriting the table); by default
 * they are plain launches (measured faster at C2).  Capturable into a CUDA
 * graph. */
int32_t tdkv_collect_round(const int64_t* d_deltas, int64_t n_table_rows,
                           const double* d_inv_freq, void* d_table, const void* d_master_k,
                           const void* d_master_v, int64_t master_layer_stride,
                           const tdkv_collect_unit* d_units, int32_t n_units, int32_t max_rows,
                           const tdkv_collect_job* d_jobs, const int64_t* d_dst_rows,
                           void* d_dst_k, void* d_dst_v, int64_t dst_layer_stride,
                           int32_t num_layers, int32_t num_heads, int32_t head_dim,
                           int32_t dtype, int32_t grid_limit, int32_t flags, void* stream);
/* flags of tdkv_collect_round: TDKV_ROUND_FUSE_TABLE computes each job
 * group's cos/sin rows inside K1 (shared memory, the K0 arithmetic) instead
 * of launching K0 -- one kernel per round, for launch-bound small rounds.
 * Requires one table row per job (every job's delta constant: tbl_stride 0,
 * tbl_row indexing d_deltas). */
#define TDKV_ROUND_FUSE_TABLE 1
/* TDKV_ROUND_NEOX rotates rotate-half pairs (element j of a head with element
 * j + D/2, angle index j; GPT-NeoX / Llama layout) instead of the reference's
 * interleaved pairs (toymodel.py:78-82): a thread owns a 16-byte unit of a
 * head's lower half and the unit D/2 elements on, so both members of every
 * pair are in its registers.  Requires 16-byte-aligned planes and half heads
 * of whole 16-byte units. */
#define TDKV_ROUND_NEOX 2
/* TDKV_ROUND_ONE_ITEM (with TDKV_ROUND_FUSE_TABLE): one work item per CTA of
 * 128 threads, no persistent prefetch -- for rounds whose items carry few
 * jobs (the planner sets it for <= 8 jobs per tile). */
#define TDKV_ROUND_ONE_ITEM 4
/* d_master_v == d_dst_v == NULL makes a K-only collect (align_cached alone;
 * the reference copies V in _skeleton). */

/* K1 over several master sources: the All-Gather round fused with the
 * collector.  Replaces the exchange the reference does not have
 * (every segment master sits in one process, trace.py:161-184) followed by
 * align_cached (pic.py:208-235) + the _skeleton V copy (pic.py:203-204) +
 * write_rows (paged_pool.py:150-156): unit u's master tile is read from
 * source d_unit_src[u], whose K/V bases are h_src_k/h_src_v[d_unit_src[u]]
 * (host arrays of n_src <= 16 device pointers, each an arena of the same
 * layout -- typically a peer GPU's arena mapped over NVLink by CUDA IPC, or
 * the local one).  Every other argument is tdkv_collect's; the tiles are
 * TMA-staged from the peer straight into shared memory, so no received copy
 * of the masters is ever written to local HBM.  All sources must be 16-byte
 * aligned. */
int32_t tdkv_collect_sources(const void* const* h_src_k, const void* const* h_src_v,
                             int32_t n_src, const uint8_t* d_unit_src,
                             int64_t master_layer_stride,
                             const tdkv_collect_unit* d_units, int32_t n_units,
                             int32_t max_rows,
                             const tdkv_collect_job* d_jobs, const int64_t* d_dst_rows,
                             const void* d_table, int32_t rotate,
                             void* d_dst_k, void* d_dst_v, int64_t dst_layer_stride,
                             int32_t num_layers, int32_t num_heads, int32_t head_dim,
                             int32_t dtype, int32_t grid_limit, void* stream);

/* Family restore: the fused decoder of a whole family as the collector
 * round of its master.  Replaces fused_restore (restore.py:50-104) over every
 * mirror of one or more families -- DiffStore.encode_family's output restored
 * the way trace._verify_family_restores (trace.py:289-329) walks it -- with
 * each master tile read from HBM once for all of its mirrors.  Source i
 * (h_src_k/h_src_v[i], n_src <= 16) is one master cache (L, source_rows, H,
 * D); the plan's arena rows are virtual: row i*source_rows + r is row r of
 * source i (units and jobs' seg_row0 use them).  Job j (of n_jobs) is one
 * mirror whose rows go to d_dst_rows (pool slots) rotated by its table row(s)
 * exactly as tdkv_collect, except where its diff stores the (layer l, block
 * b): d_overlay[j].map_k[l*nb + b] >= 0 names the payload block of
 * d_overlay[j].pay_k holding those K rows (rows of block_size tokens: the
 * encoder's slab), and likewise map_v / pay_v for V (a NULL map = no diff of
 * that plane; the encoder's diffs share one map).  Payload-sourced planes are skipped by K1 and written by a second
 * kernel in the same call (payload -> rotate -> pool): the overlay precedes
 * rotation (restore.py:5-8).  max_rows must divide block_size (a tile never
 * straddles a diff block); masters, payloads and the pool 16-byte aligned
 * with 16-byte rows.  Stream-ordered and capturable. */
typedef struct {
    const void* pay_k;
    const void* pay_v;
    const int32_t* map_k;    /* (L * nb) payload block or -1 */
    const int32_t* map_v;
} tdkv_collect_overlay;

int32_t tdkv_restore_family(const void* const* h_src_k, const void* const* h_src_v,
                            int32_t n_src, int64_t source_rows,
                            const tdkv_collect_unit* d_units, int32_t n_units, int32_t max_rows,
                            const tdkv_collect_job* d_jobs, int32_t n_jobs,
                            const int64_t* d_dst_rows, const tdkv_collect_overlay* d_overlay,
                            int32_t nb, int32_t block_size,
                            const void* d_table, int32_t rotate, void* d_dst_k, void* d_dst_v,
                            int64_t dst_layer_stride, int32_t num_layers, int32_t num_heads,
                            int32_t head_dim, int32_t dtype, int32_t grid_limit, void* stream);

/* ------------------------------------------------------------------------
 * K2  block-diff encoder.  Replaces diffstore.encode_diff
 * (diffstore.py:119-182) for a batch of (master, mirror) pairs of identical
 * geometry (L, T, H, D), dense planes with layer stride T*H*D.
 *
 * tdkv_diff_compare: for every pair p, layer l, block b
 *     changed[(p*L + l)*nb + b] = any(mirror != master) over K and V rows
 * with float '!=' semantics (np.array_equal, diffstore.py:151-153).  A
 * changed block whose d_hinted[p*nb + b] is 0 is a soundness violation:
 * d_violation[p] receives the smallest l*nb + b (layer-major order, the
 * reference's first raise) and d_viol_maxabs[(p*L+l)*nb + b] the block's
 * max |mirror - master| over both planes (diffstore.py:157-160).
 *
 * tdkv_diff_compact: per (p, l), stream-compacts the changed blocks in
 * ascending order: indices[l*cap + s] = b, counts[p*L + l] = n, payload
 * block (l*cap + s) = mirror rows of block b zero-padded to block_size
 * (_pad_rows, diffstore.py:110-116), and blkmap[l*nb + b] = l*cap + s for
 * changed blocks, -1 otherwise.  cap must be >= the number of changed blocks
 * of any layer (the hinted-block count is a bound when there is no
 * violation).
 * ---------------------------------------------------------------------- */
typedef struct {
    const void* master_k;
    const void* master_v;
    const void* mirror_k;
    const void* mirror_v;
} tdkv_diff_pair;

typedef struct {
    void* payload_k;     /* (L*cap, block_size, H, D) */
    void* payload_v;
    int32_t* indices;    /* (L*cap) */
    int32_t* blkmap;     /* (L*nb) */
    int32_t cap;
    int32_t pad_;
} tdkv_diff_out;

int32_t tdkv_diff_compare(const tdkv_diff_pair* d_pairs, int32_t n_pairs,
                          const uint8_t* d_hinted,
                          uint8_t* d_changed, int32_t* d_violation,
                          float* d_viol_maxabs,
                          int32_t num_layers, int32_t num_tokens,
                          int32_t num_heads, int32_t head_dim,
                          int32_t block_size, int32_t dtype, void* stream);

int32_t tdkv_diff_compact(const tdkv_diff_pair* d_pairs,
                          const tdkv_diff_out* d_outs, int32_t n_pairs,
                          const uint8_t* d_changed, int32_t* d_counts,
                          int32_t num_layers, int32_t num_tokens,
                          int32_t num_heads, int32_t head_dim,
                          int32_t block_size, int32_t dtype, void* stream);

/* Single-pass form of the two calls above (what the encoder uses): compare,
 * stream compaction and payload copy in one launch.  Tiles (pair, layer,
 * block) are handed out by an atomic ticket (d_ticket, 1 int32 scratch); a
 * block publishes its status in d_flags (n_pairs*L*nb int32 scratch) and a
 * changed, hinted block finds its payload slot by looking back over the
 * flags of the earlier blocks of its layer.  Same outputs and violation
 * reporting as tdkv_diff_compare + tdkv_diff_compact. */
int32_t tdkv_diff_encode(const tdkv_diff_pair* d_pairs, const tdkv_diff_out* d_outs,
                         int32_t n_pairs, const uint8_t* d_hinted, int32_t* d_flags,
                         int32_t* d_ticket, int32_t* d_counts, int32_t* d_violation,
                         float* d_viol_maxabs, int32_t num_layers, int32_t num_tokens,
                         int32_t num_heads, int32_t head_dim, int32_t block_size,
                         int32_t dtype, void* stream);

/* ------------------------------------------------------------------------
 * K3  row mover: gather -> (diff overlay) -> rotate -> scatter.
 * Replaces restore.fused_restore (restore.py:50-104, with _apply_layer_diff
 * :39-47 and rope_recover toymodel.py:86-96), diff_decode_dense
 * (diffstore.py:185-203), dense_restore (restore.py:107-139), rope_apply /
 * rope_recover, and PagedPool.write_rows / read_rows (paged_pool.py:150-164).
 *
 * For job j, layer l, token t (block b = t / block_size):
 *   if map_k && map_k[l*nb + b] >= 0: K source = pay_k row
 *        (map_k[l*nb+b] * block_size + t - b*block_size)
 *   else K source = src_k[l*src_layer_stride + srow(t)*H*D],
 *        srow(t) = src_rows ? src_rows[t] : t
 *   (V likewise with map_v / pay_v; the diff overlays BEFORE rotation,
 *   restore.py:5-8)
 *   K is rotated with cos/sin row tbl_row + t*tbl_stride when rotate != 0,
 *   then K and V are written to dst row drow(t) = dst_rows ? dst_rows[t] : t.
 *   dst_v == NULL makes a K-only job (rope_apply).
 * ---------------------------------------------------------------------- */
typedef struct {
    const void* src_k;
    const void* src_v;
    int64_t src_layer_stride;    /* elements */
    const int64_t* src_rows;     /* NULL = identity */
    const void* pay_k;
    const void* pay_v;
    const int32_t* map_k;        /* NULL = no diff */
    const int32_t* map_v;
    void* dst_k;
    void* dst_v;
    int64_t dst_layer_stride;    /* elements */
    const int64_t* dst_rows;     /* NULL = identity */
    int32_t num_tokens;
    int32_t tbl_row;
    int32_t tbl_stride;
    int32_t rotate;
} tdkv_rows_job;

/* flags: TDKV_ROWS_CONTIGUOUS promises that every job has src_rows == NULL
 * and 16-byte aligned planes, payloads and strides; rows that are whole
 * 16-byte units then take the TMA-staged path (tiles of tile_rows rows,
 * 0 = block_size, double-buffered in shared memory by cp.async.bulk). */
#define TDKV_ROWS_CONTIGUOUS 1
/* TDKV_ROWS_JOB_MINOR orders the work items (layer, block, tile, job): the
 * jobs of one family (mirrors of one master, trace.py:289-329) then read each
 * master tile back to back, so DRAM serves it once and L2 the rest. */
#define TDKV_ROWS_JOB_MINOR 2

int32_t tdkv_rows(const tdkv_rows_job* d_jobs, int32_t n_jobs,
                  int32_t max_tokens, const void* d_table,
                  int32_t num_layers, int32_t num_heads, int32_t head_dim,
                  int32_t block_size, int32_t dtype, int32_t flags,
                  int32_t tile_rows, int32_t grid_limit, void* stream);

/* ------------------------------------------------------------------------
 * K4  check-layer selection.  Replaces the batched
 * difference pass of pic.probe_and_select (pic.py:268-281).
 *
 * tdkv_keydiff: mags[r] = sqrt(sum_e (fresh[r,e] - cached[row(r),e])^2)
 * over one token's H*D elements (key_diff, pic.py:166-171); fresh is dense
 * (n_rows, H*D), cached rows are d_cached_rows[r] (NULL = r), e.g. the pool's
 * check-layer plane addressed by slots.  float32 difference and product as
 * numpy, float64 accumulation, float32 result.
 *
 * tdkv_select_important: member m owns mags[member_off[m] .. member_off[m+1]);
 * writes its top min(budget[m], #nonzero) positions by (-mag, index), in
 * ascending order, to out_idx[out_off[m] ...] (out_off NULL: member_off;
 * an exclusive prefix of the budgets packs the results densely) (select_important,
 * pic.py:180-189), their number to out_count[m], and the float32 sum of its
 * magnitudes to deviation[m] (pic.py:280).  One CTA per member runs a
 * radix select over the magnitudes' bit patterns; at most 49152 positions
 * per member.
 * ---------------------------------------------------------------------- */
int32_t tdkv_keydiff(const void* d_fresh, const void* d_cached,
                     const int64_t* d_cached_rows, int64_t n_rows, int32_t row_elems,
                     int32_t dtype, float* d_mags, void* stream);

int32_t tdkv_select_important(const float* d_mags, const int64_t* d_member_off,
                              const int32_t* d_budget, const int64_t* d_out_off,
                              int32_t n_members,
                              int32_t max_count, int32_t* d_out_idx,
                              int32_t* d_out_count, float* d_deviation, void* stream);

/* ------------------------------------------------------------------------
 * K5 building block: C[m, n] (+)= A[m, :k] . B[n, :k] on the
 * tcgen05 tensor cores, accumulator in TMEM.  A (lda) and B (ldb) row-major
 * (K-major), C (ldc) float32 row-major; accumulate != 0 adds into C.  For
 * TDKV_F32 operands the product runs as 3xTF32 (hi/lo split) to stay within
 * float32 tolerance; TDKV_BF16 runs kind::f16 with bf16 operands.  Used for
 * the Q/K/V/mix projections of the selective recompute
 * (toymodel._selective_forward, toymodel.py:99-151).
 * ---------------------------------------------------------------------- */
int32_t tdkv_gemm(const void* d_a, int32_t lda, const void* d_b, int32_t ldb,
                  float* d_c, int32_t ldc, int32_t m, int32_t n, int32_t k,
                  int32_t dtype, int32_t accumulate, void* stream);

/* 3xTF32 with the split done once, outside the GEMM: tdkv_tf32_split writes
 * the tf32 hi (cvt.rna of x) and lo (cvt.rna of x - hi) planes of n floats
 * (n % 4 == 0, 16-byte aligned); tdkv_gemm_tf32x3 is tdkv_gemm for TDKV_F32
 * with A and B given as such planes (same lda / ldb) -- a pure TMA ->
 * tcgen05 pipeline (A_hi B_hi + A_hi B_lo + A_lo B_hi per k-step) with no
 * in-kernel split; the selective recompute splits its weights once and its
 * activations per GEMM. */
int32_t tdkv_tf32_split(const float* d_src, int64_t n, float* d_hi, float* d_lo, void* stream);
int32_t tdkv_gemm_tf32x3(const float* d_a_hi, const float* d_a_lo, int32_t lda,
                         const float* d_b_hi, const float* d_b_lo, int32_t ldb,
                         float* d_c, int32_t ldc, int32_t m, int32_t n, int32_t k,
                         int32_t accumulate, void* stream);

/* K5 non-GEMM stages of one layer of the selective forward (float32 toy
 * model, toymodel.py:111-150):
 *   tdkv_qkv_rope: qkv (n_rows, 3*H*D) -> q, k rotated by the row's cos/sin
 *     (double2 table rows, one per fixed row), v copied; (n_rows, H*D) each.
 *   tdkv_attention: mix[f, h, :] = softmax_t(q[f,h].key_t * scale) . value_t
 *     over t <= fix_idx[f]; key/value rows come from the fresh rows where
 *     fresh_of[t] >= 0, else from the context planes (num_tokens, H*D). */
int32_t tdkv_qkv_rope(const float* d_qkv, const void* d_table, int32_t n_rows,
                      int32_t num_heads, int32_t head_dim, float* d_q, float* d_k,
                      float* d_v, void* stream);
int32_t tdkv_attention(const float* d_q, const float* d_k_fresh, const float* d_v_fresh,
                       const float* d_ctx_k, const float* d_ctx_v,
                       const int32_t* d_fresh_of, const int64_t* d_fix_idx,
                       int32_t n_fix, int32_t num_tokens, int32_t num_heads,
                       int32_t head_dim, float scale, float* d_mix, void* stream);

/* tdkv_attention over several members' fixed rows in one launch (grouped
 * recovery batches the members' forwards, collective.py:152-187): the rows
 * of q / fresh K,V / mix are the members' rows concatenated; member m owns
 * rows [row0, row0 + n_rows), attends over its own context (layer ``layer``
 * of planes with ctx_layer_stride elements per layer), and its fresh_of
 * indexes its own slice of the fresh rows.  d_members sorted by row0.
 * n_tiles > 0 selects a query-tiled kernel: member m's rows form
 * ceil(n_rows / rows_per_tile) tiles starting at tile index tile0 (n_tiles in
 * total), each CTA serving one tile of one member with every staged
 * key/value tile.  rows_per_tile 8 (head_dim <= 128): two-pass softmax over a
 * stored score row; rows_per_tile 16 (head_dim <= 128): online softmax
 * (running max / sum, float64 accumulators rescaled per 32-token tile);
 * rows_per_tile 64 (head_dim 8, 16, 32, 64 or 128): register-blocked, 256
 * threads per CTA, 64-token key/value tiles double-buffered by 16-byte async
 * copies, 4x4 score blocks, float32 P.V sums per tile folded into float64;
 * rows_per_tile 128 (head_dim 32 or 64): tensor cores, 256 threads per CTA,
 * the tile's rows in TMEM lanes, S = Q K^T and O = P V per 64-key tile as
 * tcgen05.mma kind::tf32 in 3xTF32 (hi/lo split operands), online softmax in
 * float32 with the running max shared by the two threads of a row.
 * The 64- and 128-row tiles move 16-byte vectors: every row plane (q, fresh
 * K/V, mix and each member's context planes) 16-byte aligned, H*D % 4 == 0
 * (TDKV_EINVAL otherwise, for the planes passed here).
 * n_tiles == 0 runs one CTA per row. */
typedef struct {
    const float* ctx_k;          /* (L, num_tokens, H*D) context planes */
    const float* ctx_v;
    const int32_t* fresh_of;     /* (num_tokens,) member-local fresh row or -1 */
    const int64_t* fix_idx;      /* (n_rows,) token index of each fixed row */
    int64_t ctx_layer_stride;
    int32_t row0;
    int32_t n_rows;
    int32_t num_tokens;
    int32_t tile0;               /* first query tile (n_tiles > 0) */
} tdkv_attn_member;

int32_t tdkv_attention_many(const float* d_q, const float* d_k_fresh, const float* d_v_fresh,
                            const tdkv_attn_member* d_members, int32_t n_members, int32_t layer,
                            int32_t total_rows, int32_t n_tiles, int32_t rows_per_tile,
                            int32_t max_tokens, int32_t num_heads, int32_t head_dim, float scale,
                            float* d_mix, void* stream);

/* ------------------------------------------------------------------------
 * Host slot allocator of the paged pool, policy of
 * PagedPool.allocate (paged_pool.py:106-135): whole free blocks ascending
 * first (a prefix of the last), then the lowest free slots.  Host memory
 * only; thread-safe.  take() writes n slots to out_slots or returns
 * TDKV_ENOSLOTS; release() rejects slots that are not allocated. */
void* tdkv_alloc_create(int64_t capacity, int32_t block_size);
void tdkv_alloc_destroy(void* handle);
int64_t tdkv_alloc_free_count(void* handle);
int32_t tdkv_alloc_take(void* handle, int64_t n, int64_t* out_slots);
int32_t tdkv_alloc_release(void* handle, const int64_t* slots, int64_t n);

/* Fill rows of every layer with a value (NaN poisoning of freed slots,
 * paged_pool.py:144-147).  value_bits is the element bit pattern. */
int32_t tdkv_fill_rows(void* d_plane, int64_t layer_stride, int32_t num_layers,
                       const int64_t* d_rows, int64_t n_rows, int32_t row_elems,
                       int32_t dtype, uint32_t value_bits, void* stream);

/* ------------------------------------------------------------------------
 * Wire format (TDDF) on the GPU.  Replaces the byte assembly of
 * serialize_diff (diffstore.py:210-239) and the payload extraction of
 * deserialize_diff (diffstore.py:242-306); the host keeps the structural
 * parse and the validation (magic, version, flags, ascending indices,
 * truncation, trailing bytes, valid_len), which are O(layers).
 *
 * An image is described by byte segments.  tdkv_wire_pack writes, for each
 * segment, ``nbytes`` bytes at byte ``offset`` of d_out taken from ``ptr``:
 * kind TDKV_WIRE_RAW copies bytes; TDKV_WIRE_BF16_TO_F32 reads nbytes/4
 * bf16 values and writes their float32 encodings (exact).  Segments must not
 * overlap; d_out must be 4-byte aligned.  tdkv_wire_unpack reads, for each
 * segment, nbytes (a multiple of 4) of d_in starting at byte ``offset`` and
 * writes them to ``ptr`` (TDKV_WIRE_RAW: 32-bit words, e.g. block indices)
 * or converts float32 -> bf16 (TDKV_WIRE_F32_TO_BF16, round to nearest
 * even); d_in must be 4-byte aligned with >= 4 readable bytes past the last
 * segment.  max_seg_bytes = the largest segment (sizes the grid).
 * ---------------------------------------------------------------------- */
#define TDKV_WIRE_RAW 0
#define TDKV_WIRE_BF16_TO_F32 1
#define TDKV_WIRE_F32_TO_BF16 2

typedef struct {
    uint64_t offset;       /* byte offset in the wire image */
    uint64_t nbytes;       /* bytes of the wire image covered */
    const void* ptr;       /* pack: source; unpack: destination (device) */
    int32_t kind;
    int32_t pad;
} tdkv_wire_seg;           /* 32 bytes */

int32_t tdkv_wire_pack(const tdkv_wire_seg* d_segs, int32_t n_segs, int64_t max_seg_bytes,
                       void* d_out, void* stream);
int32_t tdkv_wire_unpack(const tdkv_wire_seg* d_segs, int32_t n_segs, int64_t max_seg_bytes,
                         const void* d_in, void* stream);

/* ------------------------------------------------------------------------
 * Host segment index.  Replaces segment_index.SegmentIndex
 * (segment_index.py:86-183): content-digest (16-byte token_digest) keyed
 * entries, the most recent entry per digest wins a lookup, byte-budget LRU
 * eviction that skips pinned entries.  Pins are queried at eviction time
 * through ``pinned(ctx, entry_id)`` (nonzero = pinned; may be NULL).  The
 * index keeps ids and sizes; evicted ids are returned LRU-first so the
 * owner can release its objects (the reference's on_evict order).
 * ---------------------------------------------------------------------- */
typedef int32_t (*tdkv_pinned_fn)(void* ctx, int64_t entry_id);

void* tdkv_segidx_create(int64_t budget_bytes);
void tdkv_segidx_destroy(void* handle);
int64_t tdkv_segidx_count(void* handle);
int64_t tdkv_segidx_total(void* handle);
/* Insert, then evict LRU-first down to the budget (ids into evicted[cap]). */
int32_t tdkv_segidx_insert(void* handle, const uint8_t* digest16, int64_t entry_id,
                           int64_t nbytes, tdkv_pinned_fn pinned, void* ctx, int64_t* evicted,
                           int32_t cap, int32_t* n_evicted);
/* n digests (16 bytes each) -> most recent entry id or -1; refresh != 0
 * moves each hit to most-recently-used (SegmentIndex.lookup), 0 does not
 * (SegmentIndex.__contains__). */
int32_t tdkv_segidx_lookup(void* handle, const uint8_t* digests16, int32_t n, int32_t refresh,
                           int64_t* out_ids);
/* Remove an entry; for an id that is not present the reference still
 * subtracts the entry's size (segment_index.py:172-181), so nbytes is
 * subtracted then too. */
int32_t tdkv_segidx_remove(void* handle, int64_t entry_id, int64_t nbytes);
int32_t tdkv_segidx_evict(void* handle, int64_t budget_bytes, tdkv_pinned_fn pinned, void* ctx,
                          int64_t* evicted, int32_t cap, int32_t* n_evicted);
/* Live entry ids, least recently used first. */
int32_t tdkv_segidx_entries(void* handle, int64_t* out_ids, int64_t cap, int64_t* n_out);

/* ------------------------------------------------------------------------
 * Request preparation for a round (host; replaces pic.prepare_request,
 * pic.py:110-163, with core.flatten_prompt core.py:130-140 and
 * PromptLayout.segment_starts core.py:120-127).
 *
 * The round's prompts index a table of distinct segments: segment s has kind
 * seg_kind[s] (TDKV_SEG_*), tokens seg_tokens[seg_tok_off[s] ..
 * seg_tok_off[s+1]) and a 16-byte digest.  Prompt p is the segment ids
 * prompt_seg[prompt_seg_off[p] .. prompt_seg_off[p+1]) (private history
 * first, exactly once).  Every SHARED segment is looked up in the segment
 * index, in prompt order then segment order, refreshing recency like
 * SegmentIndex.lookup.  Outputs (caller-allocated; flat token count and the
 * structural capacity follow from the inputs, see paper_2604_03143_b200/
 * prepare.py): per prompt its flat tokens (one separator between
 * consecutive segments), label_entry / label_offset (entry id and offset in
 * the segment for hit positions, -1 elsewhere; entry id = nid_entry[native
 * id]), its ascending structural positions (separators, misses, task
 * segments), its private length, and one hit record (prompt segment index,
 * entry id, target start, length) + native entry id per hit.
 * threads <= 0 = all hardware threads (capped at 32).
 * Errors: TDKV_EINVAL with the reference's message for a separator inside a
 * segment, an empty segment, a negative token, a misplaced private segment.
 * ---------------------------------------------------------------------- */
#define TDKV_SEG_PRIVATE 0
#define TDKV_SEG_SHARED 1
#define TDKV_SEG_TASK 2

int32_t tdkv_prepare_batch(void* segidx, int32_t n_prompts, const int32_t* prompt_seg_off,
                           const int32_t* prompt_seg, int32_t n_segs, const int32_t* seg_kind,
                           const int64_t* seg_tok_off, const int64_t* seg_tokens,
                           const uint8_t* seg_digest16, int64_t separator,
                           const int64_t* nid_entry, int64_t n_nid, int64_t* out_tok_off,
                           int64_t* out_tokens, int64_t* out_label_entry,
                           int64_t* out_label_offset, int64_t* out_struct_off,
                           int64_t* out_structural, int64_t* out_private_len,
                           int64_t* out_hits, int64_t* out_hit_off, int64_t* out_hit_nid,
                           int32_t threads);

/* ---- Round planning (host only) -------------------------------------------
 * The collector plan of a round whose job j writes rows[dst_off[j] + i] of a
 * device-resident row table and rotates by job_delta[j]: jobs sorted by
 * segment (stable), (tile, job-chunk) units over the segments read, enough
 * (layer, unit) items for target_items.  Replaces the numpy planning of
 * KVCollector.plan_offsets (the batched form of align_cached's per-agent walk
 * over its hits, pic.py:208-235).  out_jobs / out_deltas: n_jobs entries;
 * out_units: unit_cap entries; out_info = [n_units, rotate, rows_written,
 * master_rows].  TDKV_EINVAL (out_info[0] = units needed) when unit_cap is
 * too small. */
int32_t tdkv_plan_offsets(int32_t n_seg, const int64_t* seg_row0, const int64_t* seg_len,
                          int32_t n_jobs, const int64_t* segments, const int64_t* dst_off,
                          const int64_t* job_delta, int32_t num_layers, int32_t tile_rows,
                          int64_t target_items, tdkv_collect_job* out_jobs, int64_t* out_deltas,
                          tdkv_collect_unit* out_units, int64_t unit_cap, int64_t* out_info);


#ifdef __cplusplus
}
#endif
#endif /* TDKV_H */
