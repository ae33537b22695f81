// Replay-benchmark helper (torch extension, measurement tooling only).
//
// Replays one epoch of (kind, value) allocation events — kind 0 alloc(size),
// kind 1 free(k-th allocation, 1-based), the reference trace semantics of
// profiler.py:3-11 — through whatever allocator torch's CUDA caching-allocator
// front end currently dispatches to: the native caching allocator, the
// cudaMallocAsync backend, or memplan's CUDAPluggableAllocator hooks
// (mp_torch_alloc / mp_torch_free).  Times the host cost per allocation with
// a steady clock, outside Python.
#include <torch/extension.h>
#include <c10/cuda/CUDACachingAllocator.h>

#include <chrono>
#include <cuda_runtime.h>
#include <vector>

// Returns (nanoseconds for the epoch, allocations outside [lo, lo + span)).
std::vector<double> replay_epoch(torch::Tensor kinds, torch::Tensor values, int64_t lo,
                                 int64_t span) {
    TORCH_CHECK(kinds.dtype() == torch::kInt32 && values.dtype() == torch::kInt64);
    const int32_t *k = kinds.data_ptr<int32_t>();
    const int64_t *v = values.data_ptr<int64_t>();
    const int64_t n = kinds.numel();
    std::vector<void *> ptrs;
    ptrs.reserve(n);
    auto t0 = std::chrono::steady_clock::now();
    for (int64_t i = 0; i < n; i++) {
        if (k[i] == 0) {
            ptrs.push_back(c10::cuda::CUDACachingAllocator::raw_alloc((size_t)v[i]));
        } else if (k[i] == 1) {
            void *&p = ptrs[v[i] - 1];
            if (p) c10::cuda::CUDACachingAllocator::raw_delete(p);
            p = nullptr;
        }
    }
    auto t1 = std::chrono::steady_clock::now();
    double outside = 0;
    for (void *p : ptrs) {
        if (!p) continue;
        const int64_t a = (int64_t)(uintptr_t)p;
        if (span > 0 && (a < lo || a >= lo + span)) outside += 1;
    }
    // never-freed blocks are released after the timed region
    for (void *p : ptrs)
        if (p) c10::cuda::CUDACachingAllocator::raw_delete(p);
    return {std::chrono::duration<double, std::nano>(t1 - t0).count(), outside};
}

// Addresses handed out for the epoch's allocations (for placement checks).
std::vector<int64_t> epoch_addresses(torch::Tensor kinds, torch::Tensor values) {
    const int32_t *k = kinds.data_ptr<int32_t>();
    const int64_t *v = values.data_ptr<int64_t>();
    const int64_t n = kinds.numel();
    std::vector<void *> ptrs;
    std::vector<int64_t> out;
    for (int64_t i = 0; i < n; i++) {
        if (k[i] == 0) {
            void *p = c10::cuda::CUDACachingAllocator::raw_alloc((size_t)v[i]);
            ptrs.push_back(p);
            out.push_back((int64_t)(uintptr_t)p);
        } else if (k[i] == 1) {
            void *&p = ptrs[v[i] - 1];
            if (p) c10::cuda::CUDACachingAllocator::raw_delete(p);
            p = nullptr;
        }
    }
    for (void *p : ptrs)
        if (p) c10::cuda::CUDACachingAllocator::raw_delete(p);
    return out;
}

// Front-end floor of torch's CUDAPluggableAllocator: hooks that do nothing
// but hand out distinct 512-byte-aligned addresses from a 64 MB ring (a
// live set of up to 131072 allocations; the replayed epochs never touch the
// memory).  Timing raw_alloc/raw_delete through these measures what torch's
// pluggable front end costs by itself, the floor under memplan's hooks.
extern "C" {
static char *g_floor_base = nullptr;
static uint64_t g_floor_next = 0;
static const uint64_t kFloorSlots = 131072;
void *floor_alloc(size_t size, int device, cudaStream_t stream) {
    (void)size; (void)device; (void)stream;
    if (!g_floor_base && cudaMalloc((void **)&g_floor_base, kFloorSlots * 512) != cudaSuccess)
        return nullptr;
    return g_floor_base + 512 * (g_floor_next++ % kFloorSlots);
}
void floor_free(void *ptr, size_t size, int device, cudaStream_t stream) {
    (void)ptr; (void)size; (void)device; (void)stream;
}
}

PYBIND11_MODULE(TORCH_EXTENSION_NAME, m) {
    m.def("replay_epoch", &replay_epoch);
    m.def("epoch_addresses", &epoch_addresses);
}
