// K0 interface (see prep.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "plan_types.cuh"

namespace mp {

struct PrepIn {
    const int64_t *trace_ptr;  // device, T+1
    const int64_t *alloc, *free_, *size;  // device, N each
    int64_t N, T;
};

struct PrepOut {
    uint2 *ent;   // device, N (alloc order per trace): (free rank, priority)
    // chunk-sorted table, 32 slots per chunk, chunk_base() indexing
    uint32_t *sf, *sp;
    uint4 *s0, *s1;        // chunk skeleton {K0,A,P,K15}, {K7,K23,P7,P15} per chunk
    uint2 *s2;             // chunk skeleton {P23, raw alloc origin} per chunk
    int64_t nchunks;       // total chunks of the batch (incl. per-trace gaps)
    uint4 *gs;             // group skeleton per group of 32 chunks
    int64_t ngroups;       // total groups of the batch (incl. per-trace gaps)
    uint32_t *cnt;         // live entries per chunk (planner stats)
    Rec *rec;     // device, N (priority order per trace)
    uint2 *raw2;       // device, N (priority order): raw alloc/free - tmin
    uint32_t *rawpos;  // device, N ((alloc,id) order): raw alloc - tmin
    int64_t *tmin;     // device, T: min alloc time
    int64_t *tspan;    // device, T: max free - tmin (INT64_MAX on overflow)
    uint32_t *U;  // device, T (time-rank count per trace)
    int64_t *unit;         // device, T: gcd of the trace's sizes
    uint64_t *total_units; // device, T: sum(size)/unit, saturating at 2^62
};

size_t prep_scratch_bytes(int64_t N, int64_t T);
// kernels (incl. CUB passes) launched by the last prep_run on this thread
int prep_launches();
int prep_run(const PrepIn &in, PrepOut &out, void *scratch, size_t scratch_bytes,
             cudaStream_t s);

}  // namespace mp
