// Host-side slot allocator of the paged pool.
//
// Keeps the reference policy bit-for-bit (paged_pool.PagedPool.allocate,
// paged_pool.py:106-135): take every block whose slots are all free, in
// ascending block order (a prefix of the last one when less is needed), then
// top up with the lowest remaining free slots.  The reference walks every
// block with Python set lookups per call (O(capacity)); here a per-slot free
// bitmap, a "block wholly free" bitmap and per-block free counts make a call
// O(blocks taken + words scanned).  Thread-safe (one mutex per allocator).
#include <cstdint>
#include <mutex>
#include <new>
#include <vector>

#include "tdkv_common.cuh"

namespace {

struct Allocator {
    int64_t capacity;
    int32_t block_size;
    int64_t nblocks;
    int64_t nfree;
    std::vector<uint64_t> slot_free;     // 1 = free
    std::vector<uint64_t> block_whole;   // 1 = every slot of the block free
    std::vector<int32_t> block_free;     // free slots per block
    std::mutex mu;

    Allocator(int64_t cap, int32_t bs)
        : capacity(cap), block_size(bs), nblocks((cap + bs - 1) / bs), nfree(cap),
          slot_free((cap + 63) / 64, ~0ull), block_whole((nblocks + 63) / 64, ~0ull),
          block_free(nblocks) {
        if (cap % 64) slot_free.back() = (1ull << (cap % 64)) - 1;
        if (nblocks % 64) block_whole.back() = (1ull << (nblocks % 64)) - 1;
        for (int64_t b = 0; b < nblocks; ++b) block_free[b] = (int32_t)block_len(b);
    }

    int64_t block_len(int64_t b) const {
        const int64_t lo = b * block_size;
        return (lo + block_size <= capacity ? block_size : capacity - lo);
    }
    bool is_free(int64_t s) const { return (slot_free[s >> 6] >> (s & 63)) & 1ull; }

    void take_slot(int64_t s) {
        slot_free[s >> 6] &= ~(1ull << (s & 63));
        const int64_t b = s / block_size;
        if (block_free[b]-- == block_len(b)) block_whole[b >> 6] &= ~(1ull << (b & 63));
        --nfree;
    }
    void give_slot(int64_t s) {
        slot_free[s >> 6] |= 1ull << (s & 63);
        const int64_t b = s / block_size;
        if (++block_free[b] == block_len(b)) block_whole[b >> 6] |= 1ull << (b & 63);
        ++nfree;
    }
};

}  // namespace

using namespace tdkv;

extern "C" void* tdkv_alloc_create(int64_t capacity, int32_t block_size) {
    if (capacity < 1 || block_size < 1) {
        set_error(TDKV_EINVAL, "tdkv_alloc_create: capacity and block_size must be positive");
        return nullptr;
    }
    return new (std::nothrow) Allocator(capacity, block_size);
}

extern "C" void tdkv_alloc_destroy(void* handle) { delete static_cast<Allocator*>(handle); }

extern "C" int64_t tdkv_alloc_free_count(void* handle) {
    Allocator* a = static_cast<Allocator*>(handle);
    std::lock_guard<std::mutex> g(a->mu);
    return a->nfree;
}

extern "C" int32_t tdkv_alloc_take(void* handle, int64_t n, int64_t* out_slots) {
    Allocator* a = static_cast<Allocator*>(handle);
    if (!a || !out_slots) return set_error(TDKV_EINVAL, "tdkv_alloc_take: null pointer");
    if (n < 1) return set_error(TDKV_EINVAL, "allocation must cover at least one token");
    std::lock_guard<std::mutex> g(a->mu);
    if (n > a->nfree)
        return set_error(TDKV_ENOSLOTS, "requested %lld slots, %lld free", (long long)n,
                         (long long)a->nfree);
    int64_t got = 0;
    // 1) wholly free blocks, ascending (state before this call: blocks are
    //    disjoint, so taking one never changes another's status)
    for (size_t w = 0; w < a->block_whole.size() && got < n; ++w) {
        uint64_t bits = a->block_whole[w];
        while (bits && got < n) {
            const int64_t b = (int64_t)w * 64 + __builtin_ctzll(bits);
            bits &= bits - 1;
            const int64_t lo = b * a->block_size;
            const int64_t take = std::min<int64_t>(n - got, a->block_len(b));
            for (int64_t s = lo; s < lo + take; ++s) {
                a->take_slot(s);
                out_slots[got++] = s;
            }
        }
    }
    // 2) the lowest remaining free slots
    for (size_t w = 0; w < a->slot_free.size() && got < n; ++w) {
        uint64_t bits = a->slot_free[w];
        while (bits && got < n) {
            const int64_t s = (int64_t)w * 64 + __builtin_ctzll(bits);
            bits &= bits - 1;
            a->take_slot(s);
            out_slots[got++] = s;
        }
    }
    return TDKV_OK;
}

extern "C" int32_t tdkv_alloc_release(void* handle, const int64_t* slots, int64_t n) {
    Allocator* a = static_cast<Allocator*>(handle);
    if (!a || (n > 0 && !slots)) return set_error(TDKV_EINVAL, "tdkv_alloc_release: null pointer");
    std::lock_guard<std::mutex> g(a->mu);
    for (int64_t i = 0; i < n; ++i) {
        const int64_t s = slots[i];
        if (s < 0 || s >= a->capacity || a->is_free(s)) {
            // undo this call's releases so the allocator state stays consistent
            for (int64_t j = 0; j < i; ++j) a->take_slot(slots[j]);
            return set_error(TDKV_EINVAL, "tdkv_alloc_release: slot %lld is not allocated",
                             (long long)s);
        }
        a->give_slot(s);
    }
    return TDKV_OK;
}
