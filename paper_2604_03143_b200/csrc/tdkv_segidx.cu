// Host-side content-addressed segment index (reference
// segment_index.SegmentIndex, segment_index.py:86-183).
//
// Entries are keyed by a 16-byte content digest (core.token_digest,
// blake2b-128); several entries may share a digest and a lookup returns the
// most recently inserted one.  Recency is a doubly linked list (least
// recently used first); lookups move the hit to the back.  Eviction walks
// the list from the front, skipping entries the owner reports pinned (a
// callback, consulted at eviction time exactly like the reference's
// is_pinned), until the byte total fits the budget.  The index stores ids
// and sizes only; the Python wrapper owns the entry objects.  One mutex per
// index; lookups of a whole round go through one call (tdkv_segidx_lookup).
#include <cstdint>
#include <cstring>
#include <list>
#include <mutex>
#include <new>
#include <unordered_map>
#include <vector>

#include "tdkv_common.cuh"

namespace {

struct Digest {
    uint64_t lo, hi;
    bool operator==(const Digest& o) const { return lo == o.lo && hi == o.hi; }
};
struct DigestHash {
    size_t operator()(const Digest& d) const { return (size_t)(d.lo ^ (d.hi * 0x9E3779B97F4A7C15ull)); }
};

struct Entry {
    Digest digest;
    int64_t nbytes;
    std::list<int64_t>::iterator pos;     // place in the recency list
};

struct Index {
    int64_t budget;
    int64_t total = 0;
    std::unordered_map<int64_t, Entry> entries;
    std::unordered_map<Digest, std::vector<int64_t>, DigestHash> by_digest;   // oldest first
    std::list<int64_t> lru;                                                 // LRU first
    std::mutex mu;

    explicit Index(int64_t b) : budget(b) {}

    void remove(int64_t id) {
        auto it = entries.find(id);
        if (it == entries.end()) return;
        auto& stack = by_digest[it->second.digest];
        for (size_t i = 0; i < stack.size(); ++i)
            if (stack[i] == id) {
                stack.erase(stack.begin() + (long)i);
                break;
            }
        if (stack.empty()) by_digest.erase(it->second.digest);
        lru.erase(it->second.pos);
        total -= it->second.nbytes;
        entries.erase(it);
    }

    // LRU-first eviction to ``target`` bytes, skipping pinned entries
    int32_t evict(int64_t target, tdkv_pinned_fn pinned, void* ctx, int64_t* out, int32_t cap,
                  int32_t* n_out) {
        int32_t n = 0;
        for (auto it = lru.begin(); it != lru.end() && total > target;) {
            const int64_t id = *it++;
            if (pinned && pinned(ctx, id)) continue;
            if (n >= cap) return tdkv::set_error(TDKV_EINVAL, "tdkv_segidx: eviction list too small");
            remove(id);
            out[n++] = id;
        }
        *n_out = n;
        return TDKV_OK;
    }
};

Digest load_digest(const uint8_t* p) {
    Digest d;
    memcpy(&d.lo, p, 8);
    memcpy(&d.hi, p + 8, 8);
    return d;
}

}  // namespace

using namespace tdkv;

extern "C" void* tdkv_segidx_create(int64_t budget_bytes) {
    if (budget_bytes < 0) {
        set_error(TDKV_EINVAL, "tdkv_segidx_create: negative budget");
        return nullptr;
    }
    return new (std::nothrow) Index(budget_bytes);
}

extern "C" void tdkv_segidx_destroy(void* h) { delete static_cast<Index*>(h); }

extern "C" int64_t tdkv_segidx_count(void* h) {
    Index* ix = static_cast<Index*>(h);
    std::lock_guard<std::mutex> g(ix->mu);
    return (int64_t)ix->entries.size();
}

extern "C" int64_t tdkv_segidx_total(void* h) {
    Index* ix = static_cast<Index*>(h);
    std::lock_guard<std::mutex> g(ix->mu);
    return ix->total;
}

extern "C" int32_t tdkv_segidx_insert(void* h, const uint8_t* digest, int64_t entry_id,
                                      int64_t nbytes, tdkv_pinned_fn pinned, void* ctx,
                                      int64_t* evicted, int32_t cap, int32_t* n_evicted) {
    if (!h || !digest || !n_evicted || (cap > 0 && !evicted))
        return set_error(TDKV_EINVAL, "tdkv_segidx_insert: null pointer");
    if (nbytes <= 0) return set_error(TDKV_EINVAL, "tdkv_segidx_insert: entry size must be positive");
    Index* ix = static_cast<Index*>(h);
    std::lock_guard<std::mutex> g(ix->mu);
    if (ix->entries.count(entry_id))
        return set_error(TDKV_EINVAL, "tdkv_segidx_insert: entry %lld already present",
                         (long long)entry_id);
    const Digest d = load_digest(digest);
    ix->lru.push_back(entry_id);
    ix->entries.emplace(entry_id, Entry{d, nbytes, std::prev(ix->lru.end())});
    ix->by_digest[d].push_back(entry_id);
    ix->total += nbytes;
    *n_evicted = 0;
    return ix->evict(ix->budget, pinned, ctx, evicted, cap, n_evicted);
}

extern "C" int32_t tdkv_segidx_lookup(void* h, const uint8_t* digests, int32_t n, int32_t refresh,
                                      int64_t* out_ids) {
    if (!h || n < 0 || (n > 0 && (!digests || !out_ids)))
        return set_error(TDKV_EINVAL, "tdkv_segidx_lookup: bad arguments");
    Index* ix = static_cast<Index*>(h);
    std::lock_guard<std::mutex> g(ix->mu);
    for (int32_t i = 0; i < n; ++i) {
        auto it = ix->by_digest.find(load_digest(digests + 16 * (size_t)i));
        if (it == ix->by_digest.end() || it->second.empty()) {
            out_ids[i] = -1;
            continue;
        }
        const int64_t id = it->second.back();
        out_ids[i] = id;
        if (refresh) {
            Entry& e = ix->entries.at(id);
            ix->lru.splice(ix->lru.end(), ix->lru, e.pos);   // most recently used
        }
    }
    return TDKV_OK;
}

extern "C" int32_t tdkv_segidx_remove(void* h, int64_t entry_id, int64_t nbytes) {
    if (!h) return set_error(TDKV_EINVAL, "tdkv_segidx_remove: null handle");
    Index* ix = static_cast<Index*>(h);
    std::lock_guard<std::mutex> g(ix->mu);
    if (ix->entries.count(entry_id))
        ix->remove(entry_id);
    else
        ix->total -= nbytes;     // the reference's accounting for an absent entry
    return TDKV_OK;
}

extern "C" int32_t tdkv_segidx_evict(void* h, int64_t budget_bytes, tdkv_pinned_fn pinned,
                                     void* ctx, int64_t* evicted, int32_t cap,
                                     int32_t* n_evicted) {
    if (!h || !n_evicted || (cap > 0 && !evicted))
        return set_error(TDKV_EINVAL, "tdkv_segidx_evict: null pointer");
    Index* ix = static_cast<Index*>(h);
    std::lock_guard<std::mutex> g(ix->mu);
    *n_evicted = 0;
    return ix->evict(budget_bytes, pinned, ctx, evicted, cap, n_evicted);
}

extern "C" int32_t tdkv_segidx_entries(void* h, int64_t* out_ids, int64_t cap, int64_t* n_out) {
    if (!h || !n_out || (cap > 0 && !out_ids))
        return set_error(TDKV_EINVAL, "tdkv_segidx_entries: null pointer");
    Index* ix = static_cast<Index*>(h);
    std::lock_guard<std::mutex> g(ix->mu);
    if ((int64_t)ix->lru.size() > cap)
        return set_error(TDKV_EINVAL, "tdkv_segidx_entries: output too small");
    int64_t n = 0;
    for (int64_t id : ix->lru) out_ids[n++] = id;
    *n_out = n;
    return TDKV_OK;
}
