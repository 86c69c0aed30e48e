// Host-side round planning in C++ (no device code): the collector plan of a
// round whose jobs write contiguous runs of a device-resident row table
// (collector.plan_host_offsets, the numpy form it replaces on the product
// path).  The reference has no plan -- every agent's align_cached walks its
// own hits (pic.py:208-235) -- so this is the metadata step of the batched
// collector: jobs sorted by segment (stable), (tile, job-chunk) units over
// the segments the round reads, one delta per job.
//
// Bit-identical to plan_host_offsets (tests/test_plan.py): the same stable
// order, the same chunking rule (nchunk = min(max jobs per segment,
// max(1, ceil(target_items / (L * tiles))))), the same unit order.

#include <algorithm>
#include <cstdint>
#include <vector>

#include "tdkv_common.cuh"

using namespace tdkv;

extern "C" int32_t tdkv_plan_offsets(int32_t n_seg, const int64_t* seg_row0, const int64_t* seg_len,
                                     int32_t n_jobs, const int64_t* segments, const int64_t* dst_off,
                                     const int64_t* job_delta, int32_t num_layers, int32_t tile_rows,
                                     int64_t target_items, tdkv_collect_job* out_jobs,
                                     int64_t* out_deltas, tdkv_collect_unit* out_units,
                                     int64_t unit_cap, int64_t* out_info) {
    // out_info: [n_units, rotate, rows_written, master_rows]
    if (n_seg < 0 || n_jobs < 0 || num_layers <= 0 || tile_rows <= 0 || !out_info ||
        (n_seg && (!seg_row0 || !seg_len)) ||
        (n_jobs && (!segments || !dst_off || !job_delta || !out_jobs || !out_deltas)))
        return set_error(TDKV_EINVAL, "tdkv_plan_offsets: bad arguments");
    out_info[0] = out_info[1] = out_info[2] = out_info[3] = 0;
    if (n_jobs == 0) return TDKV_OK;
    // stable counting sort of the jobs by segment
    std::vector<int32_t> count((size_t)n_seg + 1, 0);
    for (int32_t j = 0; j < n_jobs; ++j) {
        const int64_t s = segments[j];
        if (s < 0 || s >= n_seg)
            return set_error(TDKV_EINVAL, "tdkv_plan_offsets: job %d names segment %lld of %d", j,
                             (long long)s, n_seg);
        if (seg_len[s] < 0 || seg_row0[s] < 0 || seg_row0[s] + seg_len[s] > INT32_MAX)
            return set_error(TDKV_EINVAL, "tdkv_plan_offsets: segment %lld out of range",
                             (long long)s);
        ++count[(size_t)s + 1];
    }
    std::vector<int32_t> first(count.size() - 1);
    for (int32_t s = 0; s < n_seg; ++s) {
        first[(size_t)s] = count[(size_t)s];
        count[(size_t)s + 1] += count[(size_t)s];
    }
    std::vector<int32_t> pos(first);
    int64_t rows_written = 0;
    bool rotate = false;
    for (int32_t j = 0; j < n_jobs; ++j) {
        const int64_t s = segments[j];
        const int32_t o = pos[(size_t)s]++;
        tdkv_collect_job& job = out_jobs[o];
        job.dst_off = dst_off[j];
        job.seg_row0 = (int32_t)seg_row0[s];
        job.tbl_row = o;
        job.tbl_stride = 0;
        job.pad_ = 0;
        out_deltas[o] = job_delta[j];
        rotate |= job_delta[j] != 0;
        rows_written += seg_len[s];
    }
    // the segments the round reads, ascending (np.unique order)
    int64_t tiles = 0, master_rows = 0, max_jobs = 0;
    for (int32_t s = 0; s < n_seg; ++s) {
        const int64_t nj = count[(size_t)s + 1] - count[(size_t)s];
        if (!nj) continue;
        tiles += (seg_len[s] + tile_rows - 1) / tile_rows;
        master_rows += seg_len[s];
        max_jobs = std::max(max_jobs, nj);
    }
    const int64_t base_items = std::max<int64_t>(1, (int64_t)num_layers * tiles);
    const int64_t want = std::max<int64_t>(1, (target_items + base_items - 1) / base_items);
    const int64_t nchunk = std::min(max_jobs, want);
    int64_t n_units = 0;
    for (int32_t s = 0; s < n_seg; ++s) {
        const int64_t nj = count[(size_t)s + 1] - count[(size_t)s];
        if (!nj) continue;
        const int64_t per = std::max<int64_t>(1, (nj + nchunk - 1) / nchunk);
        const int64_t nc = (nj + per - 1) / per;
        const int64_t nt = (seg_len[s] + tile_rows - 1) / tile_rows;
        for (int64_t t = 0; t < nt; ++t) {
            for (int64_t c = 0; c < nc; ++c, ++n_units) {
                if (n_units >= unit_cap) continue;         // count only: the caller grows
                tdkv_collect_unit& u = out_units[n_units];
                u.row0 = (int32_t)(seg_row0[s] + t * tile_rows);
                u.nrows = (int32_t)std::min<int64_t>(tile_rows, seg_len[s] - t * tile_rows);
                const int64_t jb = first[(size_t)s] + c * per;
                u.job_begin = (int32_t)jb;
                u.job_end = (int32_t)std::min<int64_t>(jb + per, first[(size_t)s] + nj);
            }
        }
    }
    out_info[0] = n_units;
    out_info[1] = rotate;
    out_info[2] = rows_written;
    out_info[3] = master_rows;
    if (n_units > unit_cap)
        return set_error(TDKV_EINVAL, "tdkv_plan_offsets: %lld units exceed the capacity %lld",
                         (long long)n_units, (long long)unit_cap);
    return TDKV_OK;
}
