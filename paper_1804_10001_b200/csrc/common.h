// Shared host-side helpers for libmemplan_b200: status/error plumbing and a
// per-device scratch allocator.  Included by every translation unit.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/memplan_b200.h"

namespace mp {

// Thread-local last error message (mp_last_error()).
void set_error(const std::string &msg);
const char *last_error();

// Convert a CUDA error into MP_ERR_CUDA / MP_ERR_NO_DEVICE with a message.
int cuda_fail(cudaError_t e, const char *what);

#define MP_CUDA(expr)                                                   \
    do {                                                                \
        cudaError_t _e = (expr);                                        \
        if (_e != cudaSuccess) return ::mp::cuda_fail(_e, #expr);       \
    } while (0)

#define MP_TRY(expr)                                                    \
    do {                                                                \
        int _rc = (expr);                                               \
        if (_rc != MP_OK) return _rc;                                   \
    } while (0)

// Select `device` for the current thread; fails with MP_ERR_NO_DEVICE when
// no CUDA device exists (there is no CPU fallback anywhere in the library).
int use_device(int device);

// Stream-ordered scratch buffer from the device's default memory pool
// (cudaMallocAsync with an unlimited release threshold, so repeated plans
// reuse the same pages without a cudaMalloc on the hot path).
struct Scratch {
    void *ptr = nullptr;
    size_t bytes = 0;
    cudaStream_t stream = nullptr;
    Scratch() = default;
    Scratch(const Scratch &) = delete;
    Scratch &operator=(const Scratch &) = delete;
    ~Scratch() { release(); }
    int alloc(size_t n, cudaStream_t s);
    void release();
    template <typename T> T *as() const { return static_cast<T *>(ptr); }
};

// Device buffer kept for a thread's lifetime and grown on demand (plain
// cudaMalloc, not stream-ordered: every user synchronises its stream before
// the buffer is reused, and the destructor does not depend on a stream the
// caller may already have destroyed).
struct KeptBuffer {
    void *ptr = nullptr;
    size_t bytes = 0;
    KeptBuffer() = default;
    KeptBuffer(const KeptBuffer &) = delete;
    KeptBuffer &operator=(const KeptBuffer &) = delete;
    ~KeptBuffer() {
        if (ptr) cudaFree(ptr);
    }
    // nullptr on failure (the CUDA error is left for the caller's check)
    void *get(size_t n) {
        if (n <= bytes && ptr) return ptr;
        const size_t want = n > bytes + bytes / 2 ? n : bytes + bytes / 2;
        if (ptr) {
            cudaDeviceSynchronize();  // no kernel of another stream still reads it
            cudaFree(ptr);
            ptr = nullptr;
            bytes = 0;
        }
        if (cudaMalloc(&ptr, want) != cudaSuccess) {
            ptr = nullptr;
            return nullptr;
        }
        bytes = want;
        return ptr;
    }
};

// Bump sub-allocator over one Scratch (keeps the number of pool calls at one
// per plan).  All carve-outs are 256-byte aligned.
struct Carver {
    char *base;
    size_t off = 0, cap;
    Carver(void *b, size_t c) : base(static_cast<char *>(b)), cap(c) {}
    template <typename T> T *take(size_t count) {
        size_t bytes = (count * sizeof(T) + 255) & ~size_t(255);
        T *p = reinterpret_cast<T *>(base + off);
        off += bytes;
        return p;
    }
    template <typename T> static size_t need(size_t count) {
        return (count * sizeof(T) + 255) & ~size_t(255);
    }
};

}  // namespace mp
