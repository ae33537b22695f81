// H1 over real device memory: the torch.cuda.memory.CUDAPluggableAllocator
// hooks (paper §4.2-4.3; the reference package stops at the
// address arithmetic of memplan.arena.Arena, arena.py:146-322).
//
// Modes: 0 passthrough (cudaMalloc/cudaFree), 1 record (passthrough + the
// allocation trace of profiler.py's A/F events), 2 replay: the lambda-th
// allocation of an epoch is served at region + offset[lambda] out of ONE
// cudaMalloc'd region of plan.peak bytes.
//
// Real memory adds constraints the address-only reference Arena does not
// have, and the replay keeps them all:
//  * live tensors cannot move, so requests the plan does not cover — growth,
//    extra requests, requests on another stream, requests after the run left
//    the profiled order — are served by stream-ordered side allocations
//    (cudaMallocAsync on the request's stream);
//  * a planned block is placed only when it is requested at its planned tick
//    of the profile clock (profiler.py: +1 after every non-zero allocation and
//    every free of one) and the first free off its planned tick — planned or
//    side-served-because-grown — ends planned placement for the epoch, so a
//    run that leaves the profiled order never aliases live memory;
//  * planned blocks still live at an epoch boundary (a loss held across
//    steps) are CARRIED: their range stays reserved, and a planned request of
//    the next epoch that would overlap it is served from a side allocation;
//  * growth observed during an epoch is re-planned at the next epoch
//    boundary (Arena.reoptimize, arena.py:303-322, on the GPU planner K1,
//    observed running maxima, alignment kept); a plan that outgrows the
//    region gets a new region and the old one is retired until its carried
//    blocks are freed.  A pointer inside a region is never cudaFree'd.
//  * planned placement is bound to one stream (the first replay request's);
//    stream-ordered reuse inside the region is then as safe as the caching
//    allocator's same-stream reuse.  Requests on other streams go to side
//    allocations on their own stream.
//
// The hooks run under a spinlock (one atomic exchange + one release store),
// not a std::mutex: autograd runs backward on its own thread, so the state
// cannot be thread-confined, but the lock is uncontended in practice.
#include <atomic>
#include <chrono>
#include <mutex>
#include <sched.h>

#include <cuda_runtime.h>

#include "arena.h"

namespace {

struct SpinLock {
    std::atomic<bool> f{false};
    void lock() {
        for (int i = 0;; i++) {
            if (!f.exchange(true, std::memory_order_acquire)) return;
            while (f.load(std::memory_order_relaxed)) {
                if (++i > 256) sched_yield();
#if defined(__x86_64__)
                else __builtin_ia32_pause();
#endif
            }
        }
    }
    void unlock() { f.store(false, std::memory_order_release); }
};

struct Region {
    char *ptr = nullptr;
    uint64_t bytes = 0;
    int64_t carried_live = 0;
};

// a planned block still live at an epoch boundary: [lo, hi) stays reserved
struct Carried {
    uint64_t lo, hi;
    int region;
};

struct Side {
    int64_t size;
    int64_t bid;  // > 0: a planned block id (its free is tick-checked); 0: extra
    cudaStream_t stream;
};

struct TorchState {
    SpinLock lk;
    int mode = 0;  // 0 passthrough, 1 record, 2 replay
    mp_arena *arena = nullptr;
    // record mode: trace of (kind, value) with kind 0 alloc(size), 1 free(ref)
    std::vector<int32_t> kinds;
    std::vector<int64_t> values;
    std::unordered_map<uintptr_t, int64_t> ptr_ref;  // live pointer -> ref
    int64_t n_allocs = 0;
    // replay mode
    int device = 0;
    std::vector<Region> regions;  // regions[cur] serves the plan; others retired
    int cur = -1;
    std::vector<Carried> carried;
    // live planned blocks of the current region: slot (addr - base) >> gshift
    // -> ref (> 0), or -1 for a carried block
    std::vector<int64_t> slot_ref;
    uint64_t span = 0, gran = 1;
    int gshift = 0;
    std::unordered_map<uintptr_t, Side> side;
    cudaStream_t stream = nullptr;
    bool stream_bound = false;
    int64_t clock = 1;
    bool diverged = false, grew = false;
    int64_t n_planned = 0, n_side = 0, n_diverged = 0, n_replans = 0, n_unknown = 0;
    // zero-size requests: no block id, no tick (profiler.py), but torch needs
    // distinct pointers: bytes of a small dummy region (kept for the process)
    char *zbase = nullptr;
    int64_t zcap = 0, zcount = 0;
};

TorchState &ts() {
    static TorchState s;
    return s;
}

using Guard = std::lock_guard<SpinLock>;

inline bool in_region(const Region &r, uint64_t p) {
    return r.ptr && p >= (uint64_t)(uintptr_t)r.ptr && p < (uint64_t)(uintptr_t)r.ptr + r.bytes;
}

// index the current region's live planned blocks directly when the table
// stays small (planned addresses are base + multiples of the alignment)
void build_slot_table(TorchState &s) {
    mp_arena *a = s.arena;
    s.slot_ref.clear();
    s.span = 0;
    uint64_t g = 1;
    int sh = 0;
    while ((int64_t)(g << 1) <= a->alignment && (a->alignment % (int64_t)(g << 1)) == 0) {
        g <<= 1;
        sh++;
    }
    const uint64_t span = s.regions[s.cur].bytes;
    if (span / g <= (uint64_t(1) << 24)) {
        s.gran = g;
        s.gshift = sh;
        s.span = span;
        s.slot_ref.assign((size_t)(span / g) + 1, 0);
        for (const Carried &c : s.carried)
            if (c.region == s.cur) {
                const uint64_t rel = c.lo - (uint64_t)(uintptr_t)s.regions[s.cur].ptr;
                if ((rel & (g - 1)) == 0) s.slot_ref[rel >> sh] = -1;
            }
    }
}

bool hits_carried(const TorchState &s, uint64_t lo, uint64_t hi) {
    for (const Carried &c : s.carried)
        if (c.region == s.cur && lo < c.hi && c.lo < hi) return true;
    return false;
}

void release_region_if_idle(TorchState &s, int r) {
    Region &R = s.regions[r];
    if (r != s.cur && R.ptr && R.carried_live == 0) {
        cudaFree(R.ptr);  // synchronises: no kernel still reads the retired region
        R.ptr = nullptr;
        R.bytes = 0;
    }
}

// the live planned blocks of this epoch stay where they are
void carry_live_blocks(TorchState &s) {
    mp_arena *a = s.arena;
    if (!a || s.cur < 0 || a->n_live == 0) return;
    const uint64_t rbase = (uint64_t)(uintptr_t)s.regions[s.cur].ptr;
    for (int64_t b = 1; b <= a->nblocks(); b++) {
        if (!a->live_on[b]) continue;
        const uint64_t lo = a->live_addr[b];
        const uint64_t hi = lo + (uint64_t)std::max<int64_t>(a->dsize[b], 1);
        s.carried.push_back({lo, hi, s.cur});
        s.regions[s.cur].carried_live++;
        const uint64_t rel = lo - rbase;
        if (!s.slot_ref.empty() && rel < s.span && (rel & (s.gran - 1)) == 0)
            s.slot_ref[rel >> s.gshift] = -1;
        else
            s.ptr_ref.erase((uintptr_t)lo);
    }
}

// free of a carried block: the range is released, the region too when it is
// retired and this was its last carried block
bool free_carried(TorchState &s, uint64_t p) {
    for (size_t i = 0; i < s.carried.size(); i++) {
        if (s.carried[i].lo != p) continue;
        const int r = s.carried[i].region;
        s.carried[i] = s.carried.back();
        s.carried.pop_back();
        s.regions[r].carried_live--;
        release_region_if_idle(s, r);
        return true;
    }
    return false;
}

void *side_alloc(TorchState &s, size_t size, int device, cudaStream_t stream, int64_t bid) {
    int cur = -1;
    cudaGetDevice(&cur);
    if (cur != device) cudaSetDevice(device);
    void *p = nullptr;
    if (cudaMallocAsync(&p, size ? size : 1, stream) != cudaSuccess) return nullptr;
    s.side[(uintptr_t)p] = Side{(int64_t)size, bid, stream};
    s.n_side++;
    return p;
}

void *replay_alloc(TorchState &s, size_t size, int device, cudaStream_t stream) {
    mp_arena *a = s.arena;
    if (size == 0 && s.zbase) return s.zbase + (s.zcount++ % s.zcap);
    const int64_t sz = (int64_t)size;
    const int64_t bid = a->lam;
    const bool planned_id = a->depth == 0 && !a->closed && bid <= a->nblocks();
    if (!s.stream_bound) {
        s.stream = stream;
        s.stream_bound = true;
    }
    const bool on_tick =
        planned_id && !s.diverged && device == s.device && a->dalloc[bid] == s.clock;
    if (planned_id) {
        if (!on_tick) s.diverged = true;
        s.clock++;
    }
    s.n_allocs++;
    if (on_tick && sz <= a->expected[bid] && stream == s.stream &&
        (s.carried.empty() ||
         !hits_carried(s, a->base + (uint64_t)a->offsets[bid],
                       a->base + (uint64_t)a->offsets[bid] + (uint64_t)a->dsize[bid]))) {
        // hot path: base + offset[lambda] and one table store for the free
        uint64_t addr = 0;
        if (a->alloc(sz, &addr) == MP_OK) {
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
    // outside the plan: remember the observed size for the next re-plan
    if (planned_id && sz > a->observed[bid]) {
        a->observed[bid] = sz;
        if (sz > a->expected[bid]) s.grew = true;
    }
    if (a->depth == 0) a->lam++;
    return side_alloc(s, size, device, stream, planned_id ? bid : 0);
}

void replay_free(TorchState &s, void *ptr) {
    mp_arena *a = s.arena;
    const uint64_t p = (uint64_t)(uintptr_t)ptr;
    if (s.zbase && (char *)ptr >= s.zbase && (char *)ptr < s.zbase + s.zcap) return;
    if (s.cur >= 0 && in_region(s.regions[s.cur], p)) {
        const uint64_t rel = p - (uint64_t)(uintptr_t)s.regions[s.cur].ptr;
        int64_t ref = 0;
        if (!s.slot_ref.empty() && rel < s.span && (rel & (s.gran - 1)) == 0) {
            int64_t &r = s.slot_ref[rel >> s.gshift];
            ref = r;
            r = 0;
        }
        if (ref == 0) {
            auto jt = s.ptr_ref.find((uintptr_t)ptr);
            if (jt != s.ptr_ref.end()) {
                ref = jt->second;
                s.ptr_ref.erase(jt);
            }
        }
        if (ref > 0 && s.mode == 2 && a) {  // hot path: a planned block of this epoch
            const auto &e = a->seq[ref - 1];
            if (!s.diverged && e.first == K_MANAGED && a->dfree[e.second] != s.clock)
                s.diverged = true;
            s.clock++;
            a->free_ref(ref);
            return;
        }
        if (free_carried(s, p)) return;
        s.n_unknown++;  // never cudaFree a pointer inside the region
        return;
    }
    for (size_t r = 0; r < s.regions.size(); r++)
        if ((int)r != s.cur && in_region(s.regions[r], p)) {
            if (!free_carried(s, p)) s.n_unknown++;
            return;
        }
    auto it = s.side.find((uintptr_t)ptr);
    if (it != s.side.end()) {
        const Side sd = it->second;
        s.side.erase(it);
        if (s.mode == 2 && a && sd.bid > 0 && sd.bid <= a->nblocks()) {
            // a side-served planned block (growth, other stream): its free
            // must still happen at its planned tick
            if (!s.diverged && a->dfree[sd.bid] != s.clock) s.diverged = true;
            s.clock++;
        }
        cudaFreeAsync(ptr, sd.stream);
        return;
    }
    cudaFree(ptr);  // a passthrough allocation made before replay
}

}  // namespace

extern "C" {

int mp_torch_set_mode(int mode, mp_arena *arena) {
    TorchState &s = ts();
    Guard g(s.lk);
    if (mode < 0 || mode > 2 || (mode == 2 && !arena)) {
        set_error("invalid torch allocator mode");
        return MP_ERR_INVALID;
    }
    if (mode == 2 && s.cur < 0) {
        set_error("replay mode needs a region: use mp_torch_replay_begin");
        return MP_ERR_INVALID;
    }
    s.mode = mode;
    s.arena = mode == 2 ? arena : nullptr;
    s.kinds.clear();
    s.values.clear();
    s.ptr_ref.clear();
    s.n_allocs = 0;
    s.n_planned = s.n_side = s.n_diverged = s.n_replans = s.n_unknown = 0;
    s.clock = 1;
    s.diverged = s.grew = false;
    s.stream_bound = false;
    return MP_OK;
}

int mp_torch_replay_begin(mp_arena *arena, int device, uint64_t *base_out) {
    TorchState &s = ts();
    if (!arena) {
        set_error("null arena");
        return MP_ERR_INVALID;
    }
    MP_TRY(mp::use_device(device));
    {
        Guard g(s.lk);
        if (s.mode == 2) {
            set_error("a replay region is already active");
            return MP_ERR_INVALID;
        }
    }
    void *p = nullptr;
    const size_t bytes = arena->plan_peak > 0 ? (size_t)arena->plan_peak : 1;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e != cudaSuccess) return mp::cuda_fail(e, "cudaMalloc(replay region)");
    if (!s.zbase) {
        void *z = nullptr;
        e = cudaMalloc(&z, 1 << 20);
        if (e != cudaSuccess) {
            cudaFree(p);
            return mp::cuda_fail(e, "cudaMalloc(zero-size region)");
        }
        s.zbase = static_cast<char *>(z);
        s.zcap = 1 << 20;
    }
    // side allocations come from the device's default pool: keep its pages
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    arena->base = (uint64_t)(uintptr_t)p;
    Guard g(s.lk);
    Region r;
    r.ptr = static_cast<char *>(p);
    r.bytes = bytes;
    s.regions.push_back(r);
    s.cur = (int)s.regions.size() - 1;
    s.device = device;
    s.mode = 2;
    s.arena = arena;
    s.kinds.clear();
    s.values.clear();
    s.ptr_ref.clear();
    s.n_allocs = 0;
    s.n_planned = s.n_side = s.n_diverged = s.n_replans = s.n_unknown = 0;
    s.clock = 1;
    s.diverged = s.grew = false;
    s.stream_bound = false;
    s.zcount = 0;
    build_slot_table(s);
    if (base_out) *base_out = arena->base;
    return MP_OK;
}

int mp_torch_replay_end(void) {
    TorchState &s = ts();
    Guard g(s.lk);
    if (s.mode == 2) {
        carry_live_blocks(s);  // tensors made during replay may outlive it
        if (s.arena) s.arena->reset();
    }
    const int old = s.cur;
    s.cur = -1;
    if (old >= 0) release_region_if_idle(s, old);
    s.slot_ref.clear();
    s.span = 0;
    s.mode = 0;
    s.arena = nullptr;
    return MP_OK;
}

int mp_torch_get_trace(int32_t *kinds, int64_t *values, int64_t cap, int64_t *n_out) {
    TorchState &s = ts();
    Guard g(s.lk);
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
    Guard g(s.lk);
    s.n_allocs = 0;
    if (s.mode != 2 || !s.arena) {
        s.ptr_ref.clear();
        return MP_OK;
    }
    mp_arena *a = s.arena;
    if (a->n_live && a->strict) {
        set_error(std::to_string(a->n_live) + " monitored blocks live at reset");
        return MP_ERR_LIVE_AT_RESET;
    }
    carry_live_blocks(s);
    MP_TRY(a->reset());
    if (s.diverged) s.n_diverged++;
    s.clock = 1;
    s.diverged = false;
    if (s.grew) {
        // deferred Arena.reoptimize (arena.py:303-322) on the GPU planner:
        // observed running maxima, alignment kept
        s.grew = false;
        MP_TRY(a->reoptimize());
        s.n_replans++;
        if ((uint64_t)a->plan_peak > s.regions[s.cur].bytes) {
            void *p = nullptr;
            cudaError_t e = cudaMalloc(&p, (size_t)a->plan_peak);
            if (e != cudaSuccess) return mp::cuda_fail(e, "cudaMalloc(replay region)");
            Region r;
            r.ptr = static_cast<char *>(p);
            r.bytes = (uint64_t)a->plan_peak;
            const int old = s.cur;
            s.regions.push_back(r);
            s.cur = (int)s.regions.size() - 1;
            release_region_if_idle(s, old);
            build_slot_table(s);
        }
        a->base = (uint64_t)(uintptr_t)s.regions[s.cur].ptr;
    }
    return MP_OK;
}

void *mp_torch_alloc(size_t size, int device, mp_stream_t stream) {
    TorchState &s = ts();
    Guard g(s.lk);
    if (s.mode == 2 && s.arena) return replay_alloc(s, size, device, (cudaStream_t)stream);
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
    Guard g(s.lk);
    if (s.mode == 1) {
        auto it = s.ptr_ref.find((uintptr_t)ptr);
        if (it != s.ptr_ref.end()) {
            s.kinds.push_back(1);
            s.values.push_back(it->second);
            s.ptr_ref.erase(it);
        }
    }
    if (s.mode == 2 || !s.regions.empty() || !s.side.empty()) {
        replay_free(s, ptr);
        return;
    }
    cudaFree(ptr);
}

int mp_torch_stats(int64_t *n_planned, int64_t *n_side, int64_t *n_diverged) {
    TorchState &s = ts();
    Guard g(s.lk);
    if (n_planned) *n_planned = s.n_planned;
    if (n_side) *n_side = s.n_side;
    if (n_diverged) *n_diverged = s.n_diverged + (s.diverged ? 1 : 0);
    return MP_OK;
}

int mp_torch_stats_ex(mp_torch_stats_t *o) {
    TorchState &s = ts();
    Guard g(s.lk);
    o->n_planned = s.n_planned;
    o->n_side = s.n_side;
    o->n_diverged = s.n_diverged + (s.diverged ? 1 : 0);
    o->n_replans = s.n_replans;
    o->n_carried_live = (int64_t)s.carried.size();
    int64_t nr = 0;
    for (const Region &r : s.regions) nr += r.ptr != nullptr;
    o->n_regions = nr;
    o->n_unknown_free = s.n_unknown;
    o->n_side_live = (int64_t)s.side.size();
    o->region_base = s.cur >= 0 ? (uint64_t)(uintptr_t)s.regions[s.cur].ptr : 0;
    o->region_bytes = s.cur >= 0 ? (int64_t)s.regions[s.cur].bytes : 0;
    o->plan_peak = s.arena ? s.arena->plan_peak : 0;
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
    cudaStream_t st = s.stream_bound ? s.stream : nullptr;
    for (int64_t r = 0; r < reps; r++) {
        MP_TRY(mp_torch_epoch_reset());
        int64_t k = 0;
        auto t0 = std::chrono::steady_clock::now();
        for (int64_t i = 0; i < n_events; i++) {
            if (kinds[i] == 0) {
                ptrs[k++] = mp_torch_alloc((size_t)values[i], s.device, (mp_stream_t)st);
            } else if (kinds[i] == 1) {
                mp_torch_free(ptrs[values[i] - 1], 0, s.device, (mp_stream_t)st);
                ptrs[values[i] - 1] = nullptr;
            }
        }
        auto t1 = std::chrono::steady_clock::now();
        for (int64_t j = 0; j < k; j++)
            if (ptrs[j]) mp_torch_free(ptrs[j], 0, s.device, (mp_stream_t)st), ptrs[j] = nullptr;
        best = std::min(best, std::chrono::duration<double, std::nano>(t1 - t0).count());
    }
    *ns_per_alloc = n_alloc ? best / (double)n_alloc : 0.0;
    return MP_OK;
}

}  // extern "C"
