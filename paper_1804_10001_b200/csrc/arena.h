// H1 data structures shared by the arena C ABI (arena.cpp) and the torch
// CUDAPluggableAllocator hooks (torch_alloc.cpp).
#pragma once

#include <algorithm>
#include <set>
#include <unordered_map>
#include <utility>
#include <vector>

#include "common.h"

using mp::set_error;

// --------------------------------------------------------------------------
// fallback pool
// --------------------------------------------------------------------------
struct mp_pool {
    int64_t capacity = -1;  // < 0: unbounded
    std::set<std::pair<int64_t, int64_t>> freel;  // (size, addr)
    std::unordered_map<int64_t, std::pair<int64_t, int64_t>> live;  // ref -> (addr, size)
    int64_t next_ref = 1, cursor = 0, reserved = 0, peak = 0, live_bytes = 0;

    int alloc(int64_t size, int64_t *addr_out) {
        if (size < 1) {
            set_error("pool allocation size must be >= 1, got " + std::to_string(size));
            return MP_ERR_INVALID;
        }
        const int64_t ref = next_ref++;
        auto it = freel.lower_bound({size, INT64_MIN});
        if (it != freel.end()) {
            const int64_t bsize = it->first, addr = it->second;
            freel.erase(it);
            live[ref] = {addr, bsize};
            live_bytes += bsize;
            *addr_out = addr;
            return MP_OK;
        }
        if (capacity >= 0 && reserved + size > capacity) {
            for (auto &b : freel) reserved -= b.first;  // flush
            freel.clear();
            if (reserved + size > capacity) {
                set_error("request of " + std::to_string(size) + " bytes over capacity " +
                          std::to_string(capacity) + " with " + std::to_string(reserved) +
                          " bytes live");
                return MP_ERR_OUT_OF_MEMORY;
            }
        }
        const int64_t addr = cursor;
        cursor += size;
        reserved += size;
        if (reserved > peak) peak = reserved;
        live[ref] = {addr, size};
        live_bytes += size;
        *addr_out = addr;
        return MP_OK;
    }

    int free_ref(int64_t ref) {
        auto it = live.find(ref);
        if (it == live.end()) {
            if (ref >= 1 && ref < next_ref) {
                set_error("pool allocation " + std::to_string(ref) + " freed twice");
                return MP_ERR_DOUBLE_FREE;
            }
            set_error("unknown pool allocation " + std::to_string(ref));
            return MP_ERR_UNKNOWN_ID;
        }
        const int64_t addr = it->second.first, size = it->second.second;
        live.erase(it);
        live_bytes -= size;
        freel.insert({size, addr});
        return MP_OK;
    }
    int64_t last_ref() const { return next_ref - 1; }
};

// --------------------------------------------------------------------------
// replay arena
// --------------------------------------------------------------------------
enum : uint8_t { K_MANAGED = 0, K_POOL = 1, K_ZERO = 2 };

struct mp_arena {
    uint64_t base = 0;
    bool strict = false, closed = false;
    int64_t alignment = 1;
    int device = 0;
    // per block id (index bid; slot 0 unused)
    std::vector<int64_t> dsize, dalloc, dfree;  // block definitions
    std::vector<int64_t> expected, observed, offsets;
    std::vector<uint64_t> live_addr;
    std::vector<int64_t> live_size;
    std::vector<uint8_t> live_on;
    int64_t n_live = 0;
    int64_t plan_peak = 0;
    int64_t lam = 1;
    std::vector<std::pair<uint8_t, int64_t>> seq;  // this epoch's allocations
    std::vector<uint8_t> freed;                   // per ref (1-based)
    int64_t depth = 0;
    int64_t reopt_count = 0, forced_closes = 0, plan_version = 0;
    mp_pool pool;

    int64_t nblocks() const { return (int64_t)dsize.size() - 1; }

    void resize_blocks(int64_t n) {
        dsize.resize(n + 1); dalloc.resize(n + 1); dfree.resize(n + 1);
        expected.resize(n + 1); observed.resize(n + 1, 0); offsets.resize(n + 1);
        live_addr.resize(n + 1); live_size.resize(n + 1); live_on.resize(n + 1, 0);
    }

    void append_block(int64_t size) {  // arena.py:293-301
        int64_t t_lo = 0, t_hi = 1;
        const int64_t n = nblocks();
        if (n > 0) {
            t_lo = dalloc[1];
            t_hi = dfree[1];
            for (int64_t b = 2; b <= n; b++) {
                t_lo = std::min(t_lo, dalloc[b]);
                t_hi = std::max(t_hi, dfree[b]);
            }
        }
        resize_blocks(n + 1);
        dsize[n + 1] = size;
        dalloc[n + 1] = t_lo;
        dfree[n + 1] = t_hi;
        expected[n + 1] = 0;  // forces the reoptimisation below
        offsets[n + 1] = 0;
    }

    int reoptimize() {  // arena.py:303-322
        const int64_t n = nblocks();
        std::vector<int64_t> s(n), a(n), f(n), off(n);
        for (int64_t b = 1; b <= n; b++) {
            int64_t sz = std::max(dsize[b], observed[b]);
            sz = ((sz + alignment - 1) / alignment) * alignment;  // build_instance round-up
            s[b - 1] = sz;
            a[b - 1] = dalloc[b];
            f[b - 1] = dfree[b];
        }
        int64_t peak = 0;
        int rc = mp_plan_bestfit(a.data(), f.data(), s.data(), n, off.data(), &peak, 0, device,
                                 nullptr);
        if (rc != MP_OK) return rc;
        for (int64_t b = 1; b <= n; b++) {
            dsize[b] = s[b - 1];
            expected[b] = s[b - 1];
            offsets[b] = off[b - 1];
        }
        plan_peak = peak;
        for (int64_t b = 1; b <= n; b++)
            if (live_on[b]) live_addr[b] = base + (uint64_t)offsets[b];
        reopt_count++;
        plan_version++;
        return MP_OK;
    }

    int alloc(int64_t size, uint64_t *addr_out) {  // arena.py:227-254
        if (closed) {
            set_error("arena is closed");
            return MP_ERR_ALLOC_AFTER_CLOSE;
        }
        if (size < 0) {
            set_error("negative allocation size " + std::to_string(size));
            return MP_ERR_NEGATIVE_SIZE;
        }
        if (size == 0) {
            seq.emplace_back(K_ZERO, 0);
            *addr_out = base;
            return MP_OK;
        }
        if (depth > 0) {
            int64_t addr = 0;
            int rc = pool.alloc(size, &addr);
            if (rc != MP_OK) return rc;
            seq.emplace_back(K_POOL, pool.last_ref());
            *addr_out = (uint64_t)addr;
            return MP_OK;
        }
        const int64_t bid = lam;
        if (bid > nblocks()) {
            if (strict) {
                set_error("allocation " + std::to_string(bid) + " beyond the " +
                          std::to_string(nblocks()) + "-block plan");
                return MP_ERR_EXTRA_REQUEST;
            }
            append_block(size);
        }
        if (size > observed[bid]) observed[bid] = size;
        if (size > expected[bid]) {
            int rc = reoptimize();
            if (rc != MP_OK) return rc;
        }
        const uint64_t addr = base + (uint64_t)offsets[bid];
        if (!live_on[bid]) {
            live_on[bid] = 1;
            n_live++;
        }
        live_addr[bid] = addr;
        live_size[bid] = size;
        seq.emplace_back(K_MANAGED, bid);
        lam++;
        *addr_out = addr;
        return MP_OK;
    }

    int free_ref(int64_t ref) {  // arena.py:256-271
        if (ref < 1 || ref > (int64_t)seq.size()) {
            set_error("free of allocation " + std::to_string(ref) + ", but only " +
                      std::to_string(seq.size()) + " allocations this epoch");
            return MP_ERR_UNKNOWN_ID;
        }
        if ((int64_t)freed.size() < ref + 1) freed.resize(std::max<size_t>(ref + 1, 2 * freed.size()), 0);
        if (freed[ref]) {
            set_error("allocation " + std::to_string(ref) + " freed twice");
            return MP_ERR_DOUBLE_FREE;
        }
        freed[ref] = 1;
        const auto &e = seq[ref - 1];
        if (e.first == K_MANAGED) {
            if (live_on[e.second]) {
                live_on[e.second] = 0;
                n_live--;
            }
        } else if (e.first == K_POOL) {
            return pool.free_ref(e.second);
        }
        return MP_OK;
    }

    int reset() {  // arena.py:273-291
        if (n_live) {
            if (strict) {
                set_error(std::to_string(n_live) + " monitored blocks live at reset");
                return MP_ERR_LIVE_AT_RESET;
            }
            forced_closes += n_live;
            std::fill(live_on.begin(), live_on.end(), 0);
            n_live = 0;
        }
        lam = 1;
        const size_t used = seq.size() + 1;
        seq.clear();
        std::fill(freed.begin(), freed.begin() + std::min(used, freed.size()), 0);
        depth = 0;
        return MP_OK;
    }
};

