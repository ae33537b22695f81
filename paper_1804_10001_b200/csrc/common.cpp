// Error plumbing, device selection and scratch allocation.
#include "common.h"

#include <string>

namespace mp {

namespace {
thread_local std::string g_err;
}

void set_error(const std::string &msg) { g_err = msg; }
const char *last_error() { return g_err.c_str(); }

int cuda_fail(cudaError_t e, const char *what) {
    set_error(std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")");
    if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) return MP_ERR_NO_DEVICE;
    return MP_ERR_CUDA;
}

int use_device(int device) {
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0) {
        cudaGetLastError();
        set_error("no CUDA device available (memplan_b200 has no CPU fallback)");
        return MP_ERR_NO_DEVICE;
    }
    if (device < 0 || device >= count) {
        set_error("device index " + std::to_string(device) + " out of range");
        return MP_ERR_INVALID;
    }
    int cur = -1;
    cudaGetDevice(&cur);
    if (cur != device) MP_CUDA(cudaSetDevice(device));
    static thread_local bool pool_cfg[64] = {false};
    if (device < 64 && !pool_cfg[device]) {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
        cudaGetLastError();
        pool_cfg[device] = true;
    }
    return MP_OK;
}

int Scratch::alloc(size_t n, cudaStream_t s) {
    release();
    if (n == 0) n = 256;
    MP_CUDA(cudaMallocAsync(&ptr, n, s));
    bytes = n;
    stream = s;
    return MP_OK;
}

void Scratch::release() {
    if (ptr) cudaFreeAsync(ptr, stream);
    ptr = nullptr;
    bytes = 0;
}

}  // namespace mp
