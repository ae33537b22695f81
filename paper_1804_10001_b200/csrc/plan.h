// Planner host interface (see plan.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/memplan_b200.h"

namespace mp {

// Optional device-to-host copy of the results that plan_device enqueues
// before its one synchronisation (host-array callers: one round trip
// instead of two).  `done` is set when the copy was made.
struct HostCopy {
    void *dst[2];
    const void *src[2];
    size_t bytes[2];
    int n;
    bool done;
};

// All arrays device-resident; trace_ptr_h is the host copy of the CSR
// offsets (sizes the launch).  Synchronises `s` before returning.
int plan_device(const int64_t *trace_ptr_d, const int64_t *trace_ptr_h, int64_t T,
                const int64_t *alloc_d, const int64_t *free_d, const int64_t *size_d,
                int64_t *offsets_d, int64_t *peaks_d, int flags, int device, cudaStream_t s,
                HostCopy *hc = nullptr);

// Per-thread device workspace kept across plan calls (grown on demand):
// small plans then cost no allocation at all.
void *plan_workspace(size_t bytes, cudaStream_t s);

const mp_plan_info &last_plan_info();
// Replace this thread's plan info (chunked batches report their sum).
void set_plan_info(const mp_plan_info &info);

}  // namespace mp
