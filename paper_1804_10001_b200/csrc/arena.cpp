// H1 — replay arena and fallback pool (the torch CUDAPluggableAllocator hooks
// that drive an arena over real device memory are in torch_alloc.cpp).
//
// Arena replaces memplan.arena.Arena (arena.py:146-322) with identical
// observable semantics: the lambda-th monitored allocation of an epoch gets
// base + offset[lambda]; zero-size requests get base and consume no slot;
// requests inside interrupt regions go to the fallback pool; a request larger
// than planned triggers reoptimisation (re-plan on the GPU with observed
// running maxima, alignment kept — arena.py:303-322); lenient mode appends a
// block conflicting with everything for extra requests (arena.py:293-301),
// strict mode raises.  The hot alloc path is a handful of array operations.
//
// Pool replaces PoolAllocator (arena.py:59-129): smallest sufficient free
// block reused whole (ties: lowest address), else bump allocation; finite
// capacity flushes the pool before failing.
#include <chrono>

#include <cuda_runtime.h>

#include "arena.h"

extern "C" {

// ---- pool -----------------------------------------------------------------
int mp_pool_create(int64_t capacity, mp_pool **out) {
    *out = new mp_pool();
    (*out)->capacity = capacity;
    return MP_OK;
}
void mp_pool_destroy(mp_pool *p) { delete p; }
int mp_pool_alloc(mp_pool *p, int64_t size, int64_t *addr_out, int64_t *ref_out) {
    int rc = p->alloc(size, addr_out);
    if (ref_out) *ref_out = p->last_ref();
    return rc;
}
int mp_pool_free(mp_pool *p, int64_t ref) { return p->free_ref(ref); }
int mp_pool_stats(mp_pool *p, int64_t *peak, int64_t *cursor, int64_t *live_bytes,
                  int64_t *last_ref) {
    if (peak) *peak = p->peak;
    if (cursor) *cursor = p->cursor;
    if (live_bytes) *live_bytes = p->live_bytes;
    if (last_ref) *last_ref = p->last_ref();
    return MP_OK;
}

// simulate_pool (arena.py:343-364): every allocation served dynamically.
int mp_simulate_pool(const int32_t *kinds, const int64_t *values, int64_t n_events,
                     int64_t capacity, int64_t *peak_out) {
    mp_pool pool;
    pool.capacity = capacity;
    std::vector<int64_t> refs;
    refs.reserve((size_t)n_events);
    for (int64_t i = 0; i < n_events; i++) {
        if (kinds[i] == 0) {
            if (values[i] == 0) {
                refs.push_back(0);
            } else {
                int64_t addr = 0;
                int rc = pool.alloc(values[i], &addr);
                if (rc != MP_OK) return rc;
                refs.push_back(pool.last_ref());
            }
        } else if (kinds[i] == 1) {
            const int64_t r = values[i];
            if (r < 1 || r > (int64_t)refs.size()) {
                set_error("free of unknown allocation " + std::to_string(r));
                return MP_ERR_UNKNOWN_ID;
            }
            if (refs[r - 1]) {
                int rc = pool.free_ref(refs[r - 1]);
                if (rc != MP_OK) return rc;
            }
        }
    }
    *peak_out = pool.peak;
    return MP_OK;
}

// ---- arena ----------------------------------------------------------------
int mp_arena_open(const int64_t *size, const int64_t *alloc, const int64_t *free_,
                  const int64_t *offsets, int64_t n, int64_t peak, uint64_t base,
                  int64_t alignment, int strict, int device, mp_arena **out) {
    if (n < 0 || alignment < 1) {
        set_error("invalid arena arguments");
        return MP_ERR_INVALID;
    }
    mp_arena *a = new mp_arena();
    a->base = base;
    a->strict = strict != 0;
    a->alignment = alignment;
    a->device = device;
    a->resize_blocks(n);
    for (int64_t b = 1; b <= n; b++) {
        a->dsize[b] = size[b - 1];
        a->dalloc[b] = alloc[b - 1];
        a->dfree[b] = free_[b - 1];
        a->expected[b] = size[b - 1];
        a->offsets[b] = offsets[b - 1];
    }
    a->plan_peak = peak;
    a->seq.reserve(1024);
    a->freed.assign(1024, 0);
    *out = a;
    return MP_OK;
}

void mp_arena_close_handle(mp_arena *a) { delete a; }
int mp_arena_alloc(mp_arena *a, int64_t size, uint64_t *addr_out) { return a->alloc(size, addr_out); }
int mp_arena_free(mp_arena *a, int64_t ref) { return a->free_ref(ref); }
int mp_arena_reset(mp_arena *a) { return a->reset(); }
int mp_arena_interrupt(mp_arena *a) {
    a->depth++;
    return MP_OK;
}
int mp_arena_resume(mp_arena *a) {
    if (a->depth == 0) {
        set_error("resume without matching interrupt");
        return MP_ERR_UNBALANCED_RESUME;
    }
    a->depth--;
    return MP_OK;
}
int mp_arena_close(mp_arena *a) {
    a->closed = true;
    return MP_OK;
}
int mp_arena_reoptimize(mp_arena *a) { return a->reoptimize(); }
mp_pool *mp_arena_pool(mp_arena *a) { return &a->pool; }

int mp_arena_get_state(mp_arena *a, mp_arena_state *o) {
    o->lam = a->lam;
    o->reopt_count = a->reopt_count;
    o->forced_closes = a->forced_closes;
    o->plan_peak = a->plan_peak;
    o->pool_peak = a->pool.peak;
    o->n_blocks = a->nblocks();
    o->n_live = a->n_live;
    o->depth = a->depth;
    o->plan_version = a->plan_version;
    o->pool_last_ref = a->pool.last_ref();
    return MP_OK;
}

int mp_arena_get_plan(mp_arena *a, int64_t *offsets, int64_t *sizes, int64_t *allocs,
                      int64_t *frees) {
    const int64_t n = a->nblocks();
    for (int64_t b = 1; b <= n; b++) {
        if (offsets) offsets[b - 1] = a->offsets[b];
        if (sizes) sizes[b - 1] = a->dsize[b];
        if (allocs) allocs[b - 1] = a->dalloc[b];
        if (frees) frees[b - 1] = a->dfree[b];
    }
    return MP_OK;
}

int mp_arena_get_live(mp_arena *a, int64_t *ids, uint64_t *addrs, int64_t *sizes) {
    int64_t k = 0;
    for (int64_t b = 1; b <= a->nblocks(); b++) {
        if (!a->live_on[b]) continue;
        if (ids) ids[k] = b;
        if (addrs) addrs[k] = a->live_addr[b];
        if (sizes) sizes[k] = a->live_size[b];
        k++;
    }
    return MP_OK;
}

int mp_arena_get_observed(mp_arena *a, int64_t *observed) {
    for (int64_t b = 1; b <= a->nblocks(); b++) observed[b - 1] = a->observed[b];
    return MP_OK;
}

int mp_arena_replay(mp_arena *a, const int32_t *kinds, const int64_t *values, int64_t n_events,
                    uint64_t *addrs_out, int64_t *n_addrs_out) {
    int64_t k = 0;
    for (int64_t i = 0; i < n_events; i++) {
        int rc = MP_OK;
        switch (kinds[i]) {
            case 0: {
                uint64_t addr = 0;
                rc = a->alloc(values[i], &addr);
                if (rc == MP_OK && addrs_out) addrs_out[k] = addr;
                k++;
                break;
            }
            case 1: rc = a->free_ref(values[i]); break;
            case 2: a->depth++; break;
            case 3: rc = mp_arena_resume(a); break;
            default:
                set_error("unknown event kind " + std::to_string(kinds[i]));
                rc = MP_ERR_INVALID;
        }
        if (rc != MP_OK) {
            if (n_addrs_out) *n_addrs_out = k;
            return rc;
        }
    }
    if (n_addrs_out) *n_addrs_out = k;
    return MP_OK;
}

int mp_arena_bench(mp_arena *a, const int32_t *kinds, const int64_t *values, int64_t n_events,
                   int64_t reps, double *ns_per_alloc) {
    int64_t n_alloc = 0;
    for (int64_t i = 0; i < n_events; i++) n_alloc += kinds[i] == 0;
    // warm-up epoch (may reoptimise once)
    int rc = mp_arena_replay(a, kinds, values, n_events, nullptr, nullptr);
    if (rc != MP_OK) return rc;
    MP_TRY(a->reset());
    double best = 1e300;
    for (int64_t r = 0; r < reps; r++) {
        auto t0 = std::chrono::steady_clock::now();
        for (int64_t i = 0; i < n_events; i++) {
            if (kinds[i] == 0) {
                uint64_t addr;
                rc = a->alloc(values[i], &addr);
            } else if (kinds[i] == 1) {
                rc = a->free_ref(values[i]);
            } else if (kinds[i] == 2) {
                a->depth++;
            } else {
                a->depth--;
            }
            if (rc != MP_OK) return rc;
        }
        auto t1 = std::chrono::steady_clock::now();
        MP_TRY(a->reset());
        const double ns = std::chrono::duration<double, std::nano>(t1 - t0).count();
        best = std::min(best, ns);
    }
    *ns_per_alloc = n_alloc ? best / (double)n_alloc : 0.0;
    return MP_OK;
}

}  // extern "C"

