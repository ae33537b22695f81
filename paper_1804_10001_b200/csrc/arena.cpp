// H1 — replay arena, fallback pool, and the torch CUDAPluggableAllocator hooks.
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
#include <algorithm>
#include <chrono>
#include <mutex>
#include <set>
#include <unordered_map>
#include <utility>
#include <vector>

#include <cuda_runtime.h>

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
namespace {
enum : uint8_t { K_MANAGED = 0, K_POOL = 1, K_ZERO = 2 };
}

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

// --------------------------------------------------------------------------
// torch.cuda.memory.CUDAPluggableAllocator hooks
// --------------------------------------------------------------------------
namespace {

struct TorchState {
    std::mutex mu;
    int mode = 0;  // 0 passthrough, 1 record, 2 replay
    mp_arena *arena = nullptr;
    // record mode: trace of (kind, value) with kind 0 alloc(size), 1 free(ref)
    std::vector<int32_t> kinds;
    std::vector<int64_t> values;
    std::unordered_map<uintptr_t, int64_t> ptr_ref;  // live pointer -> alloc ref
    // replay mode: pointers served outside the plan (growth/extra/interrupt)
    std::unordered_map<uintptr_t, int64_t> side;     // ptr -> ref
    int64_t n_allocs = 0;
    void *region = nullptr;  // the one cudaMalloc'd replay region (mp_torch_replay_begin)
    int device = 0;          // device of the replay arena
    // live planned blocks by address: slot (addr - base) >> gshift -> ref
    std::vector<int64_t> slot_ref;
    uint64_t span = 0, gran = 1;
    int gshift = 0;
    int64_t n_planned = 0, n_side = 0;  // replay-mode counters since the mode switch
    int64_t n_diverged = 0;             // epochs that left the plan (see mp_torch_alloc)
    // replay guard: the profile clock of profiler.py (y starts at 1, +1 after
    // every non-zero allocation and every free of one); a planned block is
    // only placed when its allocation happens at its planned tick, and a
    // free off its planned tick ends planned placement for the epoch
    int64_t clock = 1;
    bool diverged = false;
    // zero-size requests: no block id, no tick (profiler.py), but torch
    // needs distinct pointers: hand out bytes of a small dummy region
    char *zbase = nullptr;
    int64_t zcap = 0, zcount = 0;
};

TorchState &ts() {
    static TorchState s;
    return s;
}

}  // namespace

extern "C" {

int mp_torch_replay_begin(mp_arena *arena, int device, uint64_t *base_out) {
    TorchState &s = ts();
    if (!arena) {
        set_error("null arena");
        return MP_ERR_INVALID;
    }
    {
        std::lock_guard<std::mutex> g(s.mu);
        if (s.region) {
            set_error("a replay region is already active");
            return MP_ERR_INVALID;
        }
    }
    MP_TRY(mp::use_device(device));
    void *p = nullptr;
    const size_t bytes = arena->plan_peak > 0 ? (size_t)arena->plan_peak : 1;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e != cudaSuccess) return mp::cuda_fail(e, "cudaMalloc(replay region)");
    arena->base = (uint64_t)(uintptr_t)p;
    void *z = nullptr;
    e = cudaMalloc(&z, 1 << 20);
    if (e != cudaSuccess) {
        cudaFree(p);
        return mp::cuda_fail(e, "cudaMalloc(zero-size region)");
    }
    MP_TRY(mp_torch_set_mode(2, arena));
    std::lock_guard<std::mutex> g(s.mu);
    s.region = p;
    s.zbase = static_cast<char *>(z);
    s.zcap = 1 << 20;
    s.zcount = 0;
    if (base_out) *base_out = arena->base;
    return MP_OK;
}

int mp_torch_replay_end(void) {
    TorchState &s = ts();
    MP_TRY(mp_torch_set_mode(0, nullptr));
    std::lock_guard<std::mutex> g(s.mu);
    if (s.region) {
        cudaFree(s.region);
        s.region = nullptr;
    }
    if (s.zbase) {
        cudaFree(s.zbase);
        s.zbase = nullptr;
        s.zcap = 0;
    }
    return MP_OK;
}

int mp_torch_set_mode(int mode, mp_arena *arena) {
    TorchState &s = ts();
    std::lock_guard<std::mutex> g(s.mu);
    if (mode < 0 || mode > 2 || (mode == 2 && !arena)) {
        set_error("invalid torch allocator mode");
        return MP_ERR_INVALID;
    }
    s.mode = mode;
    s.arena = arena;
    s.kinds.clear();
    s.values.clear();
    s.ptr_ref.clear();
    s.slot_ref.clear();
    s.n_allocs = 0;
    s.n_planned = 0;
    s.n_side = 0;
    s.n_diverged = 0;
    s.clock = 1;
    s.diverged = false;
    if (mode == 2) {
        // planned addresses are base + (multiples of the alignment): index the
        // live blocks directly when the table stays small
        uint64_t g = 1;
        int sh = 0;
        while ((int64_t)(g << 1) <= arena->alignment && (arena->alignment % (int64_t)(g << 1)) == 0) {
            g <<= 1;
            sh++;
        }
        const uint64_t span = arena->plan_peak > 0 ? (uint64_t)arena->plan_peak : 0;
        if (span / g <= (uint64_t(1) << 24)) {
            s.gran = g;
            s.gshift = sh;
            s.span = span;
            s.slot_ref.assign((size_t)(span / g) + 1, 0);
        }
        cudaGetDevice(&s.device);
    }
    return MP_OK;
}

int mp_torch_get_trace(int32_t *kinds, int64_t *values, int64_t cap, int64_t *n_out) {
    TorchState &s = ts();
    std::lock_guard<std::mutex> g(s.mu);
    const int64_t n = (int64_t)s.kinds.size();
    for (int64_t i = 0; i < n && i < cap; i++) {
        kinds[i] = s.kinds[i];
        values[i] = s.values[i];
    }
    *n_out = n;
    return MP_OK;
}

int mp_torch_epoch_reset(void) {
    TorchState &s = ts();
    std::lock_guard<std::mutex> g(s.mu);
    s.n_allocs = 0;
    s.ptr_ref.clear();
    std::fill(s.slot_ref.begin(), s.slot_ref.end(), 0);
    if (s.diverged) s.n_diverged++;
    s.clock = 1;
    s.diverged = false;
    if (s.mode == 2 && s.arena) return s.arena->reset();
    return MP_OK;
}

void *mp_torch_alloc(size_t size, int device, mp_stream_t stream) {
    (void)stream;
    TorchState &s = ts();
    std::lock_guard<std::mutex> g(s.mu);
    if (s.mode == 2 && s.arena) {
        mp_arena *a = s.arena;
        if (size == 0 && s.zbase) return s.zbase + (s.zcount++ % s.zcap);
        const int64_t bid = a->lam;
        const int64_t sz = (int64_t)size;
        const bool on_plan = !s.diverged && device == s.device && a->depth == 0 && !a->closed &&
                             bid <= a->nblocks() && a->dalloc[bid] == s.clock;
        if (!on_plan && sz > 0) s.diverged = true;
        s.clock += sz > 0 ? 1 : 0;
        if (on_plan && sz <= a->expected[bid] && sz > 0) {
            // hot path: base + offset[lambda] and one table store for the free
            uint64_t addr = 0;
            if (a->alloc(sz, &addr) == MP_OK) {
                s.n_allocs++;
                s.n_planned++;
                const int64_t ref = (int64_t)a->seq.size();
                const uint64_t rel = addr - a->base;
                if (!s.slot_ref.empty() && rel < s.span && (rel & (s.gran - 1)) == 0)
                    s.slot_ref[rel >> s.gshift] = ref;
                else
                    s.ptr_ref[(uintptr_t)addr] = ref;
                return (void *)addr;
            }
        }
        // outside the plan (growth, extra request, or the run left the
        // profiled order): live tensors cannot move, so serve from a side
        // allocation and remember the observed size for the next re-plan
        if (a->depth == 0 && bid <= a->nblocks() && sz > a->observed[bid]) a->observed[bid] = sz;
        int cur = -1;
        cudaGetDevice(&cur);
        if (cur != device) cudaSetDevice(device);
        void *p = nullptr;
        if (cudaMalloc(&p, size ? size : 1) != cudaSuccess) return nullptr;
        s.side[(uintptr_t)p] = sz;
        s.n_allocs++;
        s.n_side++;
        if (a->depth == 0 && sz > 0) a->lam++;
        return p;
    }
    int cur = -1;
    cudaGetDevice(&cur);
    if (cur != device) cudaSetDevice(device);
    void *p = nullptr;
    if (cudaMalloc(&p, size ? size : 1) != cudaSuccess) return nullptr;
    if (s.mode == 1) {
        s.kinds.push_back(0);
        s.values.push_back((int64_t)size);
        s.ptr_ref[(uintptr_t)p] = ++s.n_allocs;
    }
    return p;
}

void mp_torch_free(void *ptr, size_t size, int device, mp_stream_t stream) {
    (void)size;
    (void)device;
    (void)stream;
    TorchState &s = ts();
    std::lock_guard<std::mutex> g(s.mu);
    if (s.mode == 2 && s.arena) {
        mp_arena *a = s.arena;
        const uint64_t rel = (uint64_t)(uintptr_t)ptr - a->base;
        if (s.zbase && (char *)ptr >= s.zbase && (char *)ptr < s.zbase + s.zcap) return;
        int64_t ref = 0;
        if (!s.slot_ref.empty() && rel < s.span && (rel & (s.gran - 1)) == 0) {
            int64_t &r = s.slot_ref[rel >> s.gshift];
            ref = r;
            r = 0;
        }
        if (ref <= 0) {
            auto jt = s.ptr_ref.find((uintptr_t)ptr);
            if (jt != s.ptr_ref.end()) {
                ref = jt->second;
                s.ptr_ref.erase(jt);
            }
        }
        if (ref > 0) {  // hot path: a planned block (memory stays in the region)
            const auto &e = a->seq[ref - 1];
            if (!s.diverged && e.first == K_MANAGED && a->dfree[e.second] != s.clock)
                s.diverged = true;
            s.clock++;
            a->free_ref(ref);
            return;
        }
        auto it = s.side.find((uintptr_t)ptr);
        if (it != s.side.end()) {
            if (it->second > 0) s.clock++;
            s.side.erase(it);
        }
        cudaFree(ptr);  // a side allocation, or a passthrough one made before replay
        return;
    }
    if (s.mode == 1) {
        auto it = s.ptr_ref.find((uintptr_t)ptr);
        if (it != s.ptr_ref.end()) {
            s.kinds.push_back(1);
            s.values.push_back(it->second);
            s.ptr_ref.erase(it);
        }
    }
    cudaFree(ptr);
}

int mp_torch_stats(int64_t *n_planned, int64_t *n_side, int64_t *n_diverged) {
    TorchState &s = ts();
    std::lock_guard<std::mutex> g(s.mu);
    if (n_planned) *n_planned = s.n_planned;
    if (n_side) *n_side = s.n_side;
    if (n_diverged) *n_diverged = s.n_diverged + (s.diverged ? 1 : 0);
    return MP_OK;
}

int mp_torch_bench(const int32_t *kinds, const int64_t *values, int64_t n_events, int64_t reps,
                   double *ns_per_alloc) {
    TorchState &s = ts();
    if (s.mode != 2 || !s.arena) {
        set_error("mp_torch_bench needs replay mode (mp_torch_replay_begin)");
        return MP_ERR_INVALID;
    }
    int64_t n_alloc = 0;
    for (int64_t i = 0; i < n_events; i++) n_alloc += kinds[i] == 0;
    std::vector<void *> ptrs((size_t)n_alloc + 1, nullptr);
    double best = 1e300;
    for (int64_t r = 0; r < reps; r++) {
        MP_TRY(mp_torch_epoch_reset());
        int64_t k = 0;
        auto t0 = std::chrono::steady_clock::now();
        for (int64_t i = 0; i < n_events; i++) {
            if (kinds[i] == 0) {
                ptrs[k++] = mp_torch_alloc((size_t)values[i], s.device, nullptr);
            } else if (kinds[i] == 1) {
                mp_torch_free(ptrs[values[i] - 1], 0, s.device, nullptr);
                ptrs[values[i] - 1] = nullptr;
            }
        }
        auto t1 = std::chrono::steady_clock::now();
        for (int64_t j = 0; j < k; j++)
            if (ptrs[j]) mp_torch_free(ptrs[j], 0, s.device, nullptr), ptrs[j] = nullptr;
        best = std::min(best, std::chrono::duration<double, std::nano>(t1 - t0).count());
    }
    *ns_per_alloc = n_alloc ? best / (double)n_alloc : 0.0;
    return MP_OK;
}

}  // extern "C"
