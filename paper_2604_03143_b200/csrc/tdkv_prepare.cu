// Host-side request preparation for a whole round (
// reference pic.prepare_request, pic.py:110-163, with core.flatten_prompt,
// core.py:130-140, and PromptLayout.segment_starts, core.py:120-127).
//
// A round's prompts reference a table of DISTINCT segments (every agent's
// prompt holds the same shared outputs; only the private history differs), so
// the caller converts each distinct segment's tokens once and each prompt is
// a list of segment ids.  Per prompt the reference flattens the segments with
// one separator between consecutive segments, resolves SHARED_OUTPUT
// segments against the segment index (a miss -- and every ROUND_TASK
// segment -- becomes structural-fresh), labels each hit position with the
// entry id and its offset inside the segment, and adds the separator before
// every segment after the first to the structural set.
//
// Lookups run first, sequentially in prompt order and segment order (the
// reference's recency effects, pic.py:137), through one tdkv_segidx_lookup
// call; the per-prompt fill (tokens, labels, structural lists) then runs on
// host threads, each prompt writing only its own output ranges.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "tdkv_common.cuh"

using namespace tdkv;

extern "C" int32_t tdkv_segidx_lookup(void* h, const uint8_t* digests, int32_t n, int32_t refresh,
                                      int64_t* out_ids);

namespace {

constexpr int32_t kPrivate = TDKV_SEG_PRIVATE;
constexpr int32_t kShared = TDKV_SEG_SHARED;

struct PromptWork {
    int64_t tok0;          // first flat token of the prompt in the outputs
    int64_t struct0;       // first structural slot
    int64_t hit0;          // first hit record
};

}  // namespace

extern "C" int32_t tdkv_prepare_batch(void* segidx, int32_t n_prompts, const int32_t* prompt_seg_off,
                                      const int32_t* prompt_seg, int32_t n_segs,
                                      const int32_t* seg_kind, const int64_t* seg_tok_off,
                                      const int64_t* seg_tokens, const uint8_t* seg_digest16,
                                      int64_t separator, const int64_t* nid_entry, int64_t n_nid,
                                      int64_t* out_tok_off, int64_t* out_tokens,
                                      int64_t* out_label_entry, int64_t* out_label_offset,
                                      int64_t* out_struct_off, int64_t* out_structural,
                                      int64_t* out_private_len, int64_t* out_hits,
                                      int64_t* out_hit_off, int64_t* out_hit_nid, int32_t threads) {
    if (n_prompts < 0 || n_segs < 0 || !prompt_seg_off || (n_prompts > 0 && !prompt_seg) ||
        (n_segs > 0 && (!seg_kind || !seg_tok_off || !seg_tokens || !seg_digest16)))
        return set_error(TDKV_EINVAL, "tdkv_prepare_batch: bad arguments");
    // validation (PromptLayout / Segment invariants, core.py:70-108)
    for (int32_t s = 0; s < n_segs; ++s) {
        const int64_t n = seg_tok_off[s + 1] - seg_tok_off[s];
        if (n <= 0) return set_error(TDKV_EINVAL, "segment %d: segment must contain at least one token", s);
        const int64_t* t = seg_tokens + seg_tok_off[s];
        for (int64_t i = 0; i < n; ++i) {
            if (t[i] < 0) return set_error(TDKV_EINVAL, "segment %d: token ids must be non-negative", s);
            if (t[i] == separator)   // flatten_prompt, core.py:132-134
                return set_error(TDKV_EINVAL, "separator id must not occur inside a segment");
        }
    }
    std::vector<PromptWork> work((size_t)n_prompts);
    int64_t tok = 0, st = 0, nshared = 0;
    for (int32_t p = 0; p < n_prompts; ++p) {
        const int32_t a = prompt_seg_off[p], b = prompt_seg_off[p + 1];
        if (b <= a) return set_error(TDKV_EINVAL, "prompt %d: prompt needs at least one segment", p);
        for (int32_t i = a; i < b; ++i) {
            const int32_t s = prompt_seg[i];
            if (s < 0 || s >= n_segs) return set_error(TDKV_EINVAL, "prompt %d: bad segment id %d", p, s);
            if ((seg_kind[s] == kPrivate) != (i == a))
                return set_error(TDKV_EINVAL,
                                 "prompt %d: exactly one private-history segment, and it must be first", p);
            if (seg_kind[s] == kShared) ++nshared;
        }
        work[p].tok0 = tok;
        work[p].struct0 = st;
        out_tok_off[p] = tok;
        out_struct_off[p] = st;
        for (int32_t i = a; i < b; ++i) {
            const int32_t s = prompt_seg[i];
            const int64_t n = seg_tok_off[s + 1] - seg_tok_off[s];
            tok += n + (i > a ? 1 : 0);
            // upper bound: every non-private segment and every separator
            if (seg_kind[s] != kPrivate) st += n;
            if (i > a) st += 1;
        }
    }
    out_tok_off[n_prompts] = tok;
    out_struct_off[n_prompts] = st;   // capacity; exact counts are compacted below
    // lookups: every SHARED_OUTPUT segment in prompt order, one native call
    std::vector<uint8_t> keys((size_t)nshared * 16);
    std::vector<int64_t> nids((size_t)nshared, -1);
    {
        int64_t k = 0;
        for (int32_t p = 0; p < n_prompts; ++p)
            for (int32_t i = prompt_seg_off[p]; i < prompt_seg_off[p + 1]; ++i) {
                const int32_t s = prompt_seg[i];
                if (seg_kind[s] == kShared) memcpy(&keys[16 * (size_t)k++], seg_digest16 + 16 * (size_t)s, 16);
            }
        if (nshared > 0) {
            if (!segidx) return set_error(TDKV_EINVAL, "tdkv_prepare_batch: null segment index");
            const int32_t rc = tdkv_segidx_lookup(segidx, keys.data(), (int32_t)nshared, 1, nids.data());
            if (rc) return rc;
        }
    }
    // hit records in prompt order
    int64_t nh = 0;
    {
        int64_t k = 0;
        for (int32_t p = 0; p < n_prompts; ++p) {
            work[p].hit0 = nh;
            out_hit_off[p] = nh;
            for (int32_t i = prompt_seg_off[p]; i < prompt_seg_off[p + 1]; ++i)
                if (seg_kind[prompt_seg[i]] == kShared && nids[(size_t)k++] >= 0) ++nh;
        }
        out_hit_off[n_prompts] = nh;
    }
    for (int64_t i = 0; i < nshared; ++i)
        if (nids[(size_t)i] >= n_nid) return set_error(TDKV_EINVAL, "tdkv_prepare_batch: entry table too small");
    // shared-lookup cursor of each prompt
    std::vector<int64_t> look0((size_t)n_prompts + 1, 0);
    for (int32_t p = 0; p < n_prompts; ++p) {
        int64_t c = 0;
        for (int32_t i = prompt_seg_off[p]; i < prompt_seg_off[p + 1]; ++i) c += seg_kind[prompt_seg[i]] == kShared;
        look0[p + 1] = look0[p] + c;
    }
    std::vector<int64_t> struct_n((size_t)n_prompts, 0);

    auto fill = [&](int32_t p) {
        const int32_t a = prompt_seg_off[p], b = prompt_seg_off[p + 1];
        int64_t pos = 0;
        int64_t* tk = out_tokens + work[p].tok0;
        int64_t* le = out_label_entry + work[p].tok0;
        int64_t* lo = out_label_offset + work[p].tok0;
        int64_t* sp = out_structural + work[p].struct0;
        int64_t ns = 0, h = work[p].hit0, look = look0[p];
        for (int32_t i = a; i < b; ++i) {
            const int32_t s = prompt_seg[i];
            const int64_t n = seg_tok_off[s + 1] - seg_tok_off[s];
            if (i > a) {                       // separator before every later segment
                tk[pos] = separator;
                le[pos] = -1;
                lo[pos] = -1;
                sp[ns++] = pos;
                ++pos;
            }
            memcpy(tk + pos, seg_tokens + seg_tok_off[s], (size_t)n * sizeof(int64_t));
            int64_t nid = -1;
            if (seg_kind[s] == kShared) nid = nids[(size_t)look++];
            if (seg_kind[s] == kPrivate) {
                out_private_len[p] = n;
                for (int64_t j = 0; j < n; ++j) { le[pos + j] = -1; lo[pos + j] = -1; }
            } else if (nid >= 0) {
                const int64_t eid = nid_entry ? nid_entry[nid] : nid;
                for (int64_t j = 0; j < n; ++j) { le[pos + j] = eid; lo[pos + j] = j; }
                int64_t* rec = out_hits + 4 * h;
                rec[0] = i - a;                  // segment index inside the prompt
                rec[1] = eid;
                rec[2] = pos;                    // target start (prompt index)
                rec[3] = n;
                out_hit_nid[h] = nid;
                ++h;
            } else {                             // miss or task segment: structural-fresh
                for (int64_t j = 0; j < n; ++j) { le[pos + j] = -1; lo[pos + j] = -1; sp[ns++] = pos + j; }
            }
            pos += n;
        }
        struct_n[(size_t)p] = ns;
    };

    int nt = threads > 0 ? threads : (int)std::thread::hardware_concurrency();
    nt = std::max(1, std::min(nt, 32));
    if (n_prompts < 4 * nt) nt = std::max(1, n_prompts / 4);
    if (nt <= 1) {
        for (int32_t p = 0; p < n_prompts; ++p) fill(p);
    } else {
        std::vector<std::thread> pool;
        for (int t = 0; t < nt; ++t)
            pool.emplace_back([&, t] {
                for (int32_t p = t; p < n_prompts; p += nt) fill(p);
            });
        for (auto& th : pool) th.join();
    }
    // compact the structural lists (each prompt's list is already ascending:
    // segments and separators are emitted in stream order)
    int64_t w = 0;
    for (int32_t p = 0; p < n_prompts; ++p) {
        const int64_t r = work[p].struct0, n = struct_n[(size_t)p];
        if (w != r) memmove(out_structural + w, out_structural + r, (size_t)n * sizeof(int64_t));
        out_struct_off[p] = w;
        w += n;
    }
    out_struct_off[n_prompts] = w;
    return TDKV_OK;
}
