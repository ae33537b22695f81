/*
 * memplan_b200 — C ABI of the B200-native profile-guided memory planner.
 *
 * This is the drop-in boundary for the reference package `memplan`
 * (/root/reference/pkg/src/memplan, pure Python).  The reference has no FFI;
 * its boundary is the Python API, and each entry point below replaces one
 * reference call (cited).  The Python facade `paper_1804_10001_b200` binds
 * these with ctypes (see INTEGRATION.md for the binding a maintainer would
 * add to the reference itself).
 *
 * Conventions
 *  - Plain pointers and sizes only; int64 for times, sizes, offsets (the
 *    reference uses Python ints; the facade rejects values outside int64).
 *  - Arrays are indexed by block index k = id-1 (ids are 1..n in input
 *    order, core.py:106-111).
 *  - Every function returns an mp_status; on failure mp_last_error() gives
 *    a message (thread-local).  Status codes map 1:1 to the reference's
 *    exception classes (see paper_1804_10001_b200/_native.py).
 *  - Caller owns every buffer.  Only the arena copies and retains tables.
 *  - MP_DEVICE_PTRS in `flags` means the array arguments are device
 *    pointers (already resident in HBM); otherwise they are host pointers
 *    and the call includes the host<->device copies.
 *  - Calls that take a stream are stream-ordered on it; with MP_ASYNC they
 *    return without synchronising (device pointers only).
 *  - No CPU fallback: without a CUDA device the compute entry points return
 *    MP_ERR_NO_DEVICE.
 */
#ifndef MEMPLAN_B200_H
#define MEMPLAN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *mp_stream_t; /* == cudaStream_t */

typedef enum {
    MP_OK = 0,
    MP_ERR_INVALID = 1,           /* ValueError                                */
    MP_ERR_LOOP_BOUND = 2,        /* AssertionError, bestfit.py:297            */
    MP_ERR_ILLEGAL_LIFT = 3,      /* IllegalLift, bestfit.py:34-35,185-186     */
    MP_ERR_CUDA = 4,              /* CUDA runtime failure                      */
    MP_ERR_NO_DEVICE = 5,         /* no CUDA device: there is no CPU fallback  */
    MP_ERR_DOUBLE_FREE = 6,       /* DoubleFree, core.py:43-44                 */
    MP_ERR_UNKNOWN_ID = 7,        /* UnknownId, arena.py:51-52                 */
    MP_ERR_EXTRA_REQUEST = 8,     /* ExtraRequest, arena.py:39-40              */
    MP_ERR_ALLOC_AFTER_CLOSE = 9, /* AllocAfterClose, arena.py:43-44           */
    MP_ERR_LIVE_AT_RESET = 10,    /* LiveBlocksAtReset, arena.py:47-48         */
    MP_ERR_UNBALANCED_RESUME = 11,/* UnbalancedResume, core.py:47-48           */
    MP_ERR_INVALID_PLAN = 12,     /* InvalidPlan, arena.py:35-36               */
    MP_ERR_OUT_OF_MEMORY = 13,    /* OutOfMemory (pool), arena.py:55-56        */
    MP_ERR_NEGATIVE_SIZE = 14,    /* ValueError on negative request size       */
    MP_ERR_TRACE = 15             /* trace ingest error, see mp_ingest_info    */
} mp_status;

enum {
    MP_DEVICE_PTRS = 1 << 0, /* array args are device pointers             */
    MP_ASYNC = 1 << 1,       /* do not synchronise the stream (device ptrs) */
    MP_FORCE_GLOBAL = 1 << 2, /* debug: keep tables in global memory         */
    MP_STATS = 1 << 3         /* count reference window entries (sum_wlive)  */
};

/* Per-plan diagnostics of the last mp_plan_* call on this thread. */
typedef struct {
    int64_t steps;        /* best-fit loop iterations, bestfit.py:295-297   */
    int64_t lifts;        /* iterations that lifted a line, :300-302        */
    int64_t max_lines;    /* high-water mark of skyline line slots          */
    float prep_ms;        /* K0 (sort/rank/pack) device time                */
    float plan_ms;        /* K1/K2 planner device time incl. status check   */
    float kernel_ms;      /* first planner launch alone (CUDA events)       */
    int32_t engine;       /* which planner variant ran      */
    int32_t cluster;      /* CTAs per trace                                 */
    int64_t sum_wlive;    /* with MP_STATS: live window entries, all steps  */
    int64_t launches;     /* kernels launched by this call                  */
    int64_t diag[4];      /* with MP_STATS: choose scans, skeleton passes,
                             table segments read, edge rows read           */
    int64_t cycles[6];    /* with env MEMPLAN_TIMING: SM cycles spent in the
                             choose / query / update / retire phases, and in
                             lift / place steps                             */
} mp_plan_info;

/* ---- planning: replaces solve_bestfit(instance) -> Plan (bestfit.py:276) */
int mp_plan_bestfit(const int64_t *alloc, const int64_t *free_, const int64_t *size,
                    int64_t n, int64_t *offsets_out, int64_t *peak_out, int flags,
                    int device, mp_stream_t stream);

/* Batched: T independent traces in CSR form (trace t owns blocks
 * [trace_ptr[t], trace_ptr[t+1])).  Replaces T solve_bestfit calls
 * (SPEC.md:257 permits independent concurrent solves).  offsets_out is
 * CSR-aligned with the inputs; peaks_out has T entries. */
int mp_plan_bestfit_batched(const int64_t *trace_ptr, const int64_t *alloc,
                            const int64_t *free_, const int64_t *size, int64_t T,
                            int64_t *offsets_out, int64_t *peaks_out, int flags,
                            int device, mp_stream_t stream);

int mp_plan_last_info(mp_plan_info *out);

/* Pipelined batched planning from host arrays: a stream of batches (the
 * same calls as mp_plan_bestfit_batched, i.e. many independent
 * solve_bestfit calls, bestfit.py:276) where batch k's upload overlaps
 * batch k-1's planning and its download overlaps batch k+1's.  Results are
 * those of mp_plan_bestfit_batched; host arrays must stay untouched until
 * mp_pipe_wait(ticket) returns.  At most two batches are in flight (a third
 * submit waits for the first); a ticket's status stays available for 1024
 * further submits.  No reference counterpart (the reference
 * plans one profile per call); the facade's PlanPipe wraps it. */
typedef struct mp_plan_pipe mp_plan_pipe;
mp_plan_pipe *mp_pipe_create(int device);
int mp_pipe_submit(mp_plan_pipe *pipe, const int64_t *trace_ptr, const int64_t *alloc,
                   const int64_t *free_, const int64_t *size, int64_t T,
                   int64_t *offsets_out, int64_t *peaks_out, int flags, int64_t *ticket_out);
int mp_pipe_wait(mp_plan_pipe *pipe, int64_t ticket);
void mp_pipe_destroy(mp_plan_pipe *pipe);

/* ---- validation: replaces verify_plan(instance, plan) (verifier.py:44-81)
 * over colliding_pairs (core.py:227-249).  The report carries the exact
 * 128-bit sum of size*lifetime so the facade can compute utilisation
 * (verifier.py:67-73) with exact integer division. */
typedef struct {
    int64_t n_violations;
    int64_t peak_recomputed;
    int32_t offsets_ok;     /* every offset >= 0 */
    int32_t pad;
    uint64_t used_lo, used_hi;
} mp_verify_report;

typedef struct {
    int64_t i, j;           /* 1-based ids, i < j (Violation.pair) */
    int64_t overlap_bytes;
    int64_t overlap_ticks;
} mp_violation;

/* viol_out receives min(n_violations, viol_cap) violations sorted by (i, j). */
int mp_verify(const int64_t *alloc, const int64_t *free_, const int64_t *size,
              const int64_t *offsets, int64_t n, mp_verify_report *out,
              mp_violation *viol_out, int64_t viol_cap, int flags, int device,
              mp_stream_t stream);

/* ---- peak live bytes lower bound: replaces clique_lower_bound (core.py:252) */
int mp_clique_lower_bound(const int64_t *alloc, const int64_t *free_,
                          const int64_t *size, int64_t n, int64_t *lb_out,
                          int flags, int device, mp_stream_t stream);

/* ---- host ingest: replaces parse_trace + record + the block columns of
 * profile_to_instance (profiler.py:97-231, core.py:184-224) ----------------
 * One pass over ASCII trace text ("A size [label]", "F k", "I", "R", "#"
 * comments).  Outputs the planned blocks in id order: aligned size, alloc
 * and free clock ticks (cap = capacity of the three arrays).  On
 * MP_ERR_TRACE, err_kind says which reference exception applies (the facade
 * formats the reference's message): 1 "A needs a size", 2 bad size (token
 * at err_tok_off/len), 3 NegativeSize (err_value), 4 "F needs exactly one
 * block ref", 5 bad block ref (token), 6 ref < 1 (err_value), 7/8 "I"/"R"
 * take no arguments, 9 unknown directive (token), 10 UnknownBlockRef
 * (err_value, err_seen), 11 DoubleFree (err_value), 12 UnbalancedResume,
 * 13 outside the ASCII / int64 restatement: use the Python path.  Syntax
 * errors carry err_line and take precedence over recording errors, as in
 * the two-stage reference. */
typedef struct {
    int64_t n_blocks, unmanaged_count, horizon, n_events;
    int64_t err_line, err_tok_off, err_tok_len, err_value, err_seen;
    int32_t err_kind, pad;
} mp_ingest_info;

int mp_ingest_trace(const char *text, int64_t len, int64_t alignment, int64_t *size_out,
                    int64_t *alloc_out, int64_t *free_out, int64_t cap, mp_ingest_info *info);

/* ---- replay arena: replaces Arena (arena.py:146-322) ---------------------
 * Opens over a plan; copies the tables.  `alignment` is the instance
 * alignment used when reoptimisation rebuilds the instance (arena.py:312).
 * The arena does NOT re-verify (call mp_verify first, as Arena.__init__
 * does at arena.py:165).  Reoptimisation calls the GPU planner on `device`. */
typedef struct mp_arena mp_arena;

int mp_arena_open(const int64_t *size, const int64_t *alloc, const int64_t *free_,
                  const int64_t *offsets, int64_t n, int64_t peak, uint64_t base,
                  int64_t alignment, int strict, int device, mp_arena **out);
void mp_arena_close_handle(mp_arena *a);                  /* destroy         */
int mp_arena_alloc(mp_arena *a, int64_t size, uint64_t *addr_out); /* .alloc  */
int mp_arena_free(mp_arena *a, int64_t ref);              /* .free(ref)      */
int mp_arena_reset(mp_arena *a);                          /* .reset()        */
int mp_arena_interrupt(mp_arena *a);                      /* .interrupt()    */
int mp_arena_resume(mp_arena *a);                         /* .resume()       */
int mp_arena_close(mp_arena *a);                          /* .close()        */
int mp_arena_reoptimize(mp_arena *a);                     /* .reoptimize()   */

typedef struct {
    int64_t lam;            /* Arena.lam                */
    int64_t reopt_count;    /* Arena.reopt_count        */
    int64_t forced_closes;  /* Arena.forced_closes      */
    int64_t plan_peak;      /* Arena.plan.peak          */
    int64_t pool_peak;      /* Arena.fallback.peak      */
    int64_t n_blocks;       /* blocks in the current plan */
    int64_t n_live;         /* len(Arena.live_blocks()) */
    int64_t depth;          /* Arena.interrupted_depth  */
    int64_t plan_version;   /* bumps on every reoptimisation */
    int64_t pool_last_ref;  /* fallback.last_ref         */
} mp_arena_state;

/* The arena's fallback pool (Arena.fallback, arena.py:172), owned by the
 * arena: usable with every mp_pool_* call, never mp_pool_destroy'd. */
struct mp_pool;
struct mp_pool *mp_arena_pool(mp_arena *a);
int mp_arena_get_state(mp_arena *a, mp_arena_state *out);
/* Current plan tables (n_blocks entries each; any pointer may be NULL). */
int mp_arena_get_plan(mp_arena *a, int64_t *offsets, int64_t *sizes,
                      int64_t *allocs, int64_t *frees);
/* Live monitored blocks: ids, addresses, requested sizes (n_live entries). */
int mp_arena_get_live(mp_arena *a, int64_t *ids, uint64_t *addrs, int64_t *sizes);
/* Observed running maxima (arena.py:206-207): n_blocks entries, 0 = unseen. */
int mp_arena_get_observed(mp_arena *a, int64_t *observed);
/* Replay one epoch of (kind, value) events — kind 0 alloc(size), 1 free(ref),
 * 2 interrupt, 3 resume — replaces replay_events (arena.py:325-340).
 * addrs_out receives one address per alloc event. */
int mp_arena_replay(mp_arena *a, const int32_t *kinds, const int64_t *values,
                    int64_t n_events, uint64_t *addrs_out, int64_t *n_addrs_out);
/* Benchmark helper: replay the epoch `reps` times with a reset after each,
 * returns the mean host nanoseconds per alloc call. */
int mp_arena_bench(mp_arena *a, const int32_t *kinds, const int64_t *values,
                   int64_t n_events, int64_t reps, double *ns_per_alloc);

/* ---- torch.cuda.memory.CUDAPluggableAllocator hooks ----------------------
 * Signatures from torch/csrc/cuda/CUDAPluggableAllocator.h:21-22.  The
 * allocator serves base + offset[lambda] out of one cudaMalloc'd region of
 * plan.peak bytes (north_star); requests the plan does not cover (growth,
 * extra requests, interrupted regions) are served from a side pool so live
 * tensors never move (documented divergence). */
void *mp_torch_alloc(size_t size, int device, mp_stream_t stream);
void mp_torch_free(void *ptr, size_t size, int device, mp_stream_t stream);
/* Configure the torch hooks: mode 0 = passthrough (cudaMalloc/cudaFree),
 * 1 = record the allocation trace, 2 = replay through `arena`. */
int mp_torch_set_mode(int mode, mp_arena *arena);
/* Recorded trace since the last mode switch: kind 0 alloc(size), 1 free(ref). */
int mp_torch_get_trace(int32_t *kinds, int64_t *values, int64_t cap, int64_t *n_out);
int mp_torch_epoch_reset(void); /* start a new replay epoch (Arena.reset) */
/* Replay through torch over ONE cudaMalloc'd region of plan.peak bytes:
 * allocates the region (outside torch's allocator, so torch never sees its
 * base pointer as an allocation of its own), rebases `arena` onto it and
 * switches the hooks to replay mode.  _end switches back to passthrough and
 * frees the region. */
int mp_torch_replay_begin(mp_arena *arena, int device, uint64_t *base_out);
int mp_torch_replay_end(void);
/* Replay-mode counters since the last mode switch: requests served from the
 * plan, requests served by side allocations, epochs that left the profiled
 * order.  Replay places a block only when its allocation happens at its
 * planned tick of the profile clock (profiler.py: +1 after every non-zero
 * allocation and every free of one) and stops placing for the rest of the
 * epoch once a free happens off its planned tick, so a run that deviates
 * from the profile can never alias live memory. */
int mp_torch_stats(int64_t *n_planned, int64_t *n_side, int64_t *n_diverged);
/* Extended replay counters (same clock as mp_torch_stats) plus the region
 * state: deferred re-plans done at epoch boundaries (Arena.reoptimize,
 * arena.py:303-322, run on the GPU planner when an epoch saw growth),
 * planned blocks carried live across an epoch boundary (their range stays
 * reserved; an overlapping planned request of the next epoch is served from
 * a side allocation), regions still held (the current one plus retired ones
 * with carried blocks), frees of unknown pointers inside a region (never
 * passed to cudaFree), live side allocations. */
typedef struct {
    int64_t n_planned, n_side, n_diverged, n_replans;
    int64_t n_carried_live, n_regions, n_unknown_free, n_side_live;
    uint64_t region_base;
    int64_t region_bytes, plan_peak;
} mp_torch_stats_t;
int mp_torch_stats_ex(mp_torch_stats_t *out);
/* Benchmark helper: replay the epoch `reps` times through mp_torch_alloc /
 * mp_torch_free directly (replay mode), best mean host ns per alloc call. */
int mp_torch_bench(const int32_t *kinds, const int64_t *values, int64_t n_events, int64_t reps,
                   double *ns_per_alloc);

/* ---- fallback pool (arena.py:59-129 PoolAllocator / :343-364) ------------ */
typedef struct mp_pool mp_pool;
int mp_pool_create(int64_t capacity /* <0: unbounded */, mp_pool **out);
void mp_pool_destroy(mp_pool *p);
int mp_pool_alloc(mp_pool *p, int64_t size, int64_t *addr_out, int64_t *ref_out);
int mp_pool_free(mp_pool *p, int64_t ref);
int mp_pool_stats(mp_pool *p, int64_t *peak, int64_t *cursor, int64_t *live_bytes,
                  int64_t *last_ref);
/* simulate_pool over (kind, value) events; kind 0 alloc(size), 1 free(ref). */
int mp_simulate_pool(const int32_t *kinds, const int64_t *values, int64_t n_events,
                     int64_t capacity, int64_t *peak_out);

/* ---- misc ---------------------------------------------------------------- */
const char *mp_last_error(void);
int mp_device_count(void);
const char *mp_version(void);

#ifdef __cplusplus
}
#endif
#endif /* MEMPLAN_B200_H */
