// Host-side segment heaps (native replacement of allocators.py:36-190).
//
// Deterministic state machines: the same call sequence yields the same offsets
// on every rank, which is what makes "remote address = same offset" work
// (global_memory.py:3-9).  Offsets, rounding and reuse order are bit-for-bit
// those of the reference:
//   linear   bump from 0, alignment rounding, exact-size LIFO reuse
//   buddy    2^ceil(log2(max(size,256))) blocks, lowest-address free block,
//            optional reserved tail never handed out nor merged over
//   reverse  bump downward from the top, exact-size LIFO reuse
// DIOMP_FAULT_INJECT=alloc_overlap reproduces the reference's mutation seam
// (allocators.py:193-197) for linear and buddy heaps.
#pragma once

#include <cstdlib>
#include <cstring>
#include <list>
#include <map>
#include <set>
#include <unordered_map>
#include <vector>

#include "../../include/diomp_b200.h"

namespace diomp {

static inline int ceil_log2_u64(uint64_t n) {
    if (n <= 1) return 0;
    return 64 - __builtin_clzll(n - 1);
}

static inline uint64_t align_up_u64(uint64_t v, uint64_t a) { return (v + a - 1) & ~(a - 1); }

static inline bool fault_inject_overlap() {
    const char *v = std::getenv("DIOMP_FAULT_INJECT");
    return v && std::strcmp(v, "alloc_overlap") == 0;
}

// Insertion-ordered offset -> size map (the reference's `live` dict).
struct LiveMap {
    std::list<std::pair<uint64_t, uint64_t>> order;
    std::unordered_map<uint64_t, std::list<std::pair<uint64_t, uint64_t>>::iterator> index;

    bool contains(uint64_t off) const { return index.count(off) != 0; }
    bool empty() const { return order.empty(); }
    uint64_t last_key() const { return order.back().first; }
    void set(uint64_t off, uint64_t size) {  // dict assignment: keeps position of an existing key
        auto it = index.find(off);
        if (it != index.end()) {
            it->second->second = size;
            return;
        }
        order.emplace_back(off, size);
        index[off] = std::prev(order.end());
    }
    uint64_t pop(uint64_t off) {
        auto it = index.find(off);
        uint64_t size = it->second->second;
        order.erase(it->second);
        index.erase(it);
        return size;
    }
};

struct Heap {
    int kind;
    uint64_t capacity = 0, alignment = 64, floor_ = 0;
    // linear / reverse
    uint64_t cursor = 0;
    std::unordered_map<uint64_t, std::vector<uint64_t>> free_lists;
    // buddy
    int min_order = 8, max_order = 0;
    std::vector<std::set<uint64_t>> free_sets;
    std::unordered_map<uint64_t, int> live_order;
    LiveMap live;

    uint64_t block_size(uint64_t size) const {
        if (kind == DIOMP_HEAP_BUDDY) {
            int o = ceil_log2_u64(size ? size : 1);
            return 1ull << (o > min_order ? o : min_order);
        }
        return align_up_u64(size ? size : 1, alignment);
    }

    uint64_t maybe_inject(uint64_t off) const {
        if (kind != DIOMP_HEAP_REVERSE && !live.empty() && fault_inject_overlap())
            return live.last_key();
        return off;
    }

    int alloc(uint64_t size, uint64_t *out) {
        if (kind == DIOMP_HEAP_BUDDY) {
            if (size > capacity) return DIOMP_OUT_OF_SEGMENT;
            int o = ceil_log2_u64(size ? size : 1);
            int order = o > min_order ? o : min_order;
            int src = order;
            while (src <= max_order && free_sets[src].empty()) ++src;
            if (src > max_order) return DIOMP_OUT_OF_SEGMENT;
            uint64_t off = *free_sets[src].begin();
            free_sets[src].erase(free_sets[src].begin());
            while (src > order) {
                --src;
                free_sets[src].insert(off + (1ull << src));
            }
            off = maybe_inject(off);
            live.set(off, 1ull << order);
            live_order[off] = order;
            *out = off;
            return DIOMP_OK;
        }
        uint64_t rounded = block_size(size);
        auto fl = free_lists.find(rounded);
        uint64_t off;
        if (fl != free_lists.end() && !fl->second.empty()) {
            off = fl->second.back();
            fl->second.pop_back();
        } else if (kind == DIOMP_HEAP_LINEAR) {
            if (cursor + rounded > capacity) return DIOMP_OUT_OF_SEGMENT;
            off = cursor;
            cursor = off + rounded;
        } else {
            if (rounded > cursor) return DIOMP_OUT_OF_SEGMENT;
            off = (cursor - rounded) & ~(alignment - 1);
            if (off < floor_) return DIOMP_OUT_OF_SEGMENT;
            cursor = off;
        }
        off = maybe_inject(off);
        live.set(off, rounded);
        *out = off;
        return DIOMP_OK;
    }

    int free_block(uint64_t offset, uint64_t *size_out) {
        if (!live.contains(offset)) return DIOMP_DOUBLE_FREE;
        uint64_t size = live.pop(offset);
        if (size_out) *size_out = size;
        if (kind != DIOMP_HEAP_BUDDY) {
            free_lists[size].push_back(offset);
            return DIOMP_OK;
        }
        int order = live_order[offset];
        live_order.erase(offset);
        uint64_t off = offset;
        while (order < max_order) {
            uint64_t buddy = off ^ (1ull << order);
            auto it = free_sets[order].find(buddy);
            if (it == free_sets[order].end()) break;
            free_sets[order].erase(it);
            off = off < buddy ? off : buddy;
            ++order;
        }
        free_sets[order].insert(off);
        return DIOMP_OK;
    }
};

}  // namespace diomp

extern "C" {

int diomp_heap_create(int kind, uint64_t capacity, uint64_t arg, uint64_t alignment,
                      void **heap_out) {
    using namespace diomp;
    if (alignment == 0 || (alignment & (alignment - 1))) return DIOMP_BAD_REQUEST;
    Heap *h = new Heap();
    h->kind = kind;
    h->alignment = alignment;
    if (kind == DIOMP_HEAP_LINEAR) {
        h->capacity = capacity;
        h->cursor = 0;
    } else if (kind == DIOMP_HEAP_REVERSE) {
        h->capacity = capacity;
        h->floor_ = arg;
        h->cursor = capacity;
    } else if (kind == DIOMP_HEAP_BUDDY) {
        if (capacity == 0 || (capacity & (capacity - 1))) {
            delete h;
            return DIOMP_BAD_REQUEST;
        }
        h->capacity = capacity;
        h->min_order = ceil_log2_u64(256);
        h->max_order = ceil_log2_u64(capacity);
        h->free_sets.assign(h->max_order + 1, std::set<uint64_t>());
        if (arg == UINT64_MAX) {
            h->free_sets[h->max_order].insert(0);
        } else {
            // Seed with the buddy decomposition of [0, reserve_from).
            uint64_t off = 0, rest = arg;
            int order = h->max_order;
            while (rest > 0) {
                uint64_t blk = 1ull << order;
                if (blk <= rest && off % blk == 0) {
                    h->free_sets[order].insert(off);
                    off += blk;
                    rest -= blk;
                } else if (--order < h->min_order) {
                    delete h;
                    return DIOMP_BAD_REQUEST;
                }
            }
        }
    } else {
        delete h;
        return DIOMP_BAD_REQUEST;
    }
    *heap_out = h;
    return DIOMP_OK;
}

int diomp_heap_destroy(void *heap) {
    delete (diomp::Heap *)heap;
    return DIOMP_OK;
}

int diomp_heap_alloc(void *heap, uint64_t size, uint64_t *offset_out) {
    return ((diomp::Heap *)heap)->alloc(size, offset_out);
}

int diomp_heap_free(void *heap, uint64_t offset, uint64_t *size_out) {
    return ((diomp::Heap *)heap)->free_block(offset, size_out);
}

int diomp_heap_block_size(void *heap, uint64_t size, uint64_t *block_out) {
    *block_out = ((diomp::Heap *)heap)->block_size(size);
    return DIOMP_OK;
}

int diomp_heap_live(void *heap, uint64_t *offsets, uint64_t *sizes, uint64_t *n_inout) {
    auto *h = (diomp::Heap *)heap;
    uint64_t cap = *n_inout, i = 0;
    for (auto &kv : h->live.order) {
        if (i < cap) {
            if (offsets) offsets[i] = kv.first;
            if (sizes) sizes[i] = kv.second;
        }
        ++i;
    }
    *n_inout = i;
    return DIOMP_OK;
}

}  // extern "C"
