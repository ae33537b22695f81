// Planner host interface (see plan.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/memplan_b200.h"

namespace mp {

// All arrays device-resident; trace_ptr_h is the host copy of the CSR
// offsets (sizes the launch).  Synchronises `s` before returning.
int plan_device(const int64_t *trace_ptr_d, const int64_t *trace_ptr_h, int64_t T,
                const int64_t *alloc_d, const int64_t *free_d, const int64_t *size_d,
                int64_t *offsets_d, int64_t *peaks_d, int flags, int device, cudaStream_t s);

const mp_plan_info &last_plan_info();

}  // namespace mp
