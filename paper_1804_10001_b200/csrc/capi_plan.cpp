// extern "C" planning entry points (include/memplan_b200.h).
#include <stdlib.h>
#include <string.h>

#include <algorithm>

#include <vector>

#include "common.h"
#include "plan.h"

using namespace mp;

namespace {

// Pinned host staging for small host-array plans, one per thread and
// device, allocated on first use and kept (the per-network use case plans
// the same few-thousand-block traces over and over).
constexpr size_t kStageBytes = size_t(4) << 20;

int64_t *pinned_stage(int device) {
    static thread_local void *stage[64] = {nullptr};
    if (device < 0 || device >= 64) return nullptr;
    if (!stage[device] && cudaHostAlloc(&stage[device], kStageBytes, cudaHostAllocDefault) !=
                              cudaSuccess) {
        cudaGetLastError();
        stage[device] = nullptr;
    }
    return static_cast<int64_t *>(stage[device]);
}

int plan_entry(const int64_t *trace_ptr, bool trace_ptr_is_dev, const int64_t *alloc,
               const int64_t *free_, const int64_t *size, int64_t T, int64_t *offsets_out,
               int64_t *peaks_out, int flags, int device, cudaStream_t s);

// Largest batch one K0 pass plans: its ranks are 32-bit over the batch's 2N
// times (N < 2^30), and the device must hold the inputs, outputs and
// ~110 B/block of tables (MEMPLAN_MAX_BATCH_BLOCKS overrides, for tests).
int64_t batch_block_limit(bool host_inputs) {
    if (const char *env = getenv("MEMPLAN_MAX_BATCH_BLOCKS")) return std::max<int64_t>(1, atoll(env));
    size_t free_b = 0, total_b = 0;
    int64_t lim = int64_t(1) << 29;
    if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess)
        lim = std::min<int64_t>(lim, (int64_t)(free_b / (host_inputs ? 160 : 128)));
    cudaGetLastError();
    return std::max<int64_t>(lim, int64_t(1) << 20);
}

// A batch above the limit is planned as consecutive trace ranges, each one
// ordinary plan (traces are independent, so the results are the same); the
// plan info reports the sum.
int plan_chunked(const std::vector<int64_t> &tp_h, const int64_t *alloc, const int64_t *free_,
                 const int64_t *size, int64_t T, int64_t *offsets_out, int64_t *peaks_out,
                 int flags, int device, cudaStream_t s, int64_t lim) {
    mp_plan_info sum{};
    int64_t t0 = 0;
    while (t0 < T) {
        int64_t t1 = t0 + 1;
        while (t1 < T && tp_h[t1 + 1] - tp_h[t0] <= lim) t1++;
        const int64_t b0 = tp_h[t0];
        std::vector<int64_t> tp((size_t)(t1 - t0 + 1));
        for (int64_t i = 0; i <= t1 - t0; i++) tp[i] = tp_h[t0 + i] - b0;
        MP_TRY(plan_entry(tp.data(), false, alloc + b0, free_ + b0, size + b0, t1 - t0,
                          offsets_out + b0, peaks_out + t0, flags, device, s));
        const mp_plan_info &o = last_plan_info();
        sum.steps += o.steps;
        sum.lifts += o.lifts;
        sum.max_lines = std::max(sum.max_lines, o.max_lines);
        sum.prep_ms += o.prep_ms;
        sum.plan_ms += o.plan_ms;
        sum.kernel_ms += o.kernel_ms;
        sum.engine |= o.engine;
        sum.cluster = std::max(sum.cluster, o.cluster);
        sum.sum_wlive += o.sum_wlive;
        sum.launches += o.launches;
        for (int k = 0; k < 4; k++) sum.diag[k] += o.diag[k];
        for (int k = 0; k < 6; k++) sum.cycles[k] += o.cycles[k];
        t0 = t1;
    }
    set_plan_info(sum);
    return MP_OK;
}

int plan_entry(const int64_t *trace_ptr, bool trace_ptr_is_dev, const int64_t *alloc,
               const int64_t *free_, const int64_t *size, int64_t T, int64_t *offsets_out,
               int64_t *peaks_out, int flags, int device, cudaStream_t s) {
    MP_TRY(use_device(device));
    if (T < 0) {
        set_error("negative trace count");
        return MP_ERR_INVALID;
    }
    std::vector<int64_t> tp_h((size_t)T + 1);
    if (trace_ptr_is_dev) {
        MP_CUDA(cudaMemcpyAsync(tp_h.data(), trace_ptr, sizeof(int64_t) * (T + 1),
                                cudaMemcpyDeviceToHost, s));
        MP_CUDA(cudaStreamSynchronize(s));
    } else {
        memcpy(tp_h.data(), trace_ptr, sizeof(int64_t) * (T + 1));
    }
    for (int64_t t = 0; t < T; t++) {
        if (tp_h[t + 1] < tp_h[t]) {
            set_error("trace_ptr must be non-decreasing");
            return MP_ERR_INVALID;
        }
    }
    const int64_t N = T ? tp_h[T] : 0;
    if (T > 1 && (N > (int64_t(1) << 20) || getenv("MEMPLAN_MAX_BATCH_BLOCKS"))) {
        const int64_t lim = batch_block_limit(!(flags & MP_DEVICE_PTRS));
        if (N > lim)
            return plan_chunked(tp_h, alloc, free_, size, T, offsets_out, peaks_out, flags, device,
                                s, lim);
    }
    if (flags & MP_DEVICE_PTRS) {
        const int64_t *tp_d = trace_ptr;
        Scratch tps;
        if (!trace_ptr_is_dev) {
            MP_TRY(tps.alloc(sizeof(int64_t) * (T + 1), s));
            MP_CUDA(cudaMemcpyAsync(tps.ptr, tp_h.data(), sizeof(int64_t) * (T + 1),
                                    cudaMemcpyHostToDevice, s));
            tp_d = tps.as<int64_t>();
        }
        return plan_device(tp_d, tp_h.data(), T, alloc, free_, size, offsets_out, peaks_out,
                           flags, device, s);
    }
    // host pointers: stage through one device buffer laid out as
    // [trace_ptr | alloc | free | size] [offsets | peaks] so that each
    // direction is one copy
    const size_t nb = sizeof(int64_t) * (size_t)N;
    const size_t in_b = sizeof(int64_t) * (size_t)(T + 1) + 3 * nb;
    const size_t out_b = nb + sizeof(int64_t) * (size_t)T;
    // small plans reuse this thread's device workspace (no allocation); the
    // planner carves its own tables from a separate per-thread buffer
    int64_t *stage = (in_b <= kStageBytes && out_b <= kStageBytes) ? pinned_stage(device) : nullptr;
    Scratch buf;
    int64_t *tp_d;
    if (stage) {
        static thread_local KeptBuffer io[64];
        void *p = io[device].get(in_b + out_b + 256);
        if (!p) return cuda_fail(cudaGetLastError(), "cudaMalloc(plan staging)");
        tp_d = static_cast<int64_t *>(p);
    } else {
        MP_TRY(buf.alloc(in_b + out_b + 256, s));
        tp_d = buf.as<int64_t>();
    }
    int64_t *a_d = tp_d + (T + 1), *f_d = a_d + N, *s_d = f_d + N;
    int64_t *o_d = s_d + N, *p_d = o_d + N;
    // small plans whose caller arrays are already page-locked (torch
    // pin_memory, cudaHostAlloc) copy straight from and to them; otherwise
    // (per-network planning from numpy arrays) through a pinned staging
    // buffer: two copies instead of six pageable ones
    auto pinned = [](const void *p) {
        cudaPointerAttributes at;
        if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        return at.type == cudaMemoryTypeHost;
    };
    const bool direct = stage && N > 0 && T > 0 && pinned(alloc) && pinned(free_) &&
                        pinned(size) && pinned(offsets_out) && pinned(peaks_out);
    if (direct) {
        memcpy(stage, tp_h.data(), sizeof(int64_t) * (T + 1));
        MP_CUDA(cudaMemcpyAsync(tp_d, stage, sizeof(int64_t) * (T + 1), cudaMemcpyHostToDevice, s));
        MP_CUDA(cudaMemcpyAsync(a_d, alloc, nb, cudaMemcpyHostToDevice, s));
        MP_CUDA(cudaMemcpyAsync(f_d, free_, nb, cudaMemcpyHostToDevice, s));
        MP_CUDA(cudaMemcpyAsync(s_d, size, nb, cudaMemcpyHostToDevice, s));
    } else if (stage) {
        memcpy(stage, tp_h.data(), sizeof(int64_t) * (T + 1));
        if (N) {
            memcpy(stage + (T + 1), alloc, nb);
            memcpy(stage + (T + 1) + N, free_, nb);
            memcpy(stage + (T + 1) + 2 * N, size, nb);
        }
        MP_CUDA(cudaMemcpyAsync(tp_d, stage, in_b, cudaMemcpyHostToDevice, s));
    } else {
        MP_CUDA(cudaMemcpyAsync(tp_d, tp_h.data(), sizeof(int64_t) * (T + 1),
                                cudaMemcpyHostToDevice, s));
        if (N) {
            MP_CUDA(cudaMemcpyAsync(a_d, alloc, nb, cudaMemcpyHostToDevice, s));
            MP_CUDA(cudaMemcpyAsync(f_d, free_, nb, cudaMemcpyHostToDevice, s));
            MP_CUDA(cudaMemcpyAsync(s_d, size, nb, cudaMemcpyHostToDevice, s));
        }
    }
    // staged plans: the results' copy rides the planner's own synchronisation
    HostCopy hc{{stage, nullptr}, {o_d, nullptr}, {out_b, 0}, 1, false};
    if (direct) {
        hc.dst[0] = offsets_out;
        hc.src[0] = o_d;
        hc.bytes[0] = nb;
        hc.dst[1] = peaks_out;
        hc.src[1] = p_d;
        hc.bytes[1] = sizeof(int64_t) * (size_t)T;
        hc.n = 2;
    }
    {
        const int rc = plan_device(tp_d, tp_h.data(), T, a_d, f_d, s_d, o_d, p_d, flags, device, s,
                                   stage ? &hc : nullptr);
        if (rc != MP_OK) {
            // an early error return may leave the staged upload in flight:
            // the next call on this thread must not overwrite its source
            cudaStreamSynchronize(s);
            cudaGetLastError();
            return rc;
        }
    }
    if (direct) {
        if (!hc.done) {
            MP_CUDA(cudaMemcpyAsync(offsets_out, o_d, nb, cudaMemcpyDeviceToHost, s));
            MP_CUDA(cudaMemcpyAsync(peaks_out, p_d, sizeof(int64_t) * T, cudaMemcpyDeviceToHost, s));
            MP_CUDA(cudaStreamSynchronize(s));
        }
        return MP_OK;
    }
    if (stage) {
        // the staging buffer's input part was consumed by the upload above
        // (plan_device synchronised the stream)
        if (!hc.done) {
            MP_CUDA(cudaMemcpyAsync(stage, o_d, out_b, cudaMemcpyDeviceToHost, s));
            MP_CUDA(cudaStreamSynchronize(s));
        }
        if (N) memcpy(offsets_out, stage, nb);
        if (T) memcpy(peaks_out, stage + N, sizeof(int64_t) * T);
        return MP_OK;
    }
    if (N) MP_CUDA(cudaMemcpyAsync(offsets_out, o_d, nb, cudaMemcpyDeviceToHost, s));
    if (T) MP_CUDA(cudaMemcpyAsync(peaks_out, p_d, sizeof(int64_t) * T, cudaMemcpyDeviceToHost, s));
    MP_CUDA(cudaStreamSynchronize(s));
    return MP_OK;
}

}  // namespace

extern "C" {

int mp_plan_bestfit(const int64_t *alloc, const int64_t *free_, const int64_t *size, int64_t n,
                    int64_t *offsets_out, int64_t *peak_out, int flags, int device,
                    mp_stream_t stream) {
    if (n < 0) {
        set_error("negative block count");
        return MP_ERR_INVALID;
    }
    int64_t tp[2] = {0, n};
    if (flags & MP_DEVICE_PTRS) {
        // peak_out is a device pointer too
        return plan_entry(tp, false, alloc, free_, size, 1, offsets_out, peak_out, flags, device,
                          (cudaStream_t)stream);
    }
    return plan_entry(tp, false, alloc, free_, size, 1, offsets_out, peak_out, flags, device,
                      (cudaStream_t)stream);
}

int mp_plan_bestfit_batched(const int64_t *trace_ptr, const int64_t *alloc, const int64_t *free_,
                            const int64_t *size, int64_t T, int64_t *offsets_out,
                            int64_t *peaks_out, int flags, int device, mp_stream_t stream) {
    return plan_entry(trace_ptr, (flags & MP_DEVICE_PTRS) != 0, alloc, free_, size, T, offsets_out,
                      peaks_out, flags, device, (cudaStream_t)stream);
}

int mp_plan_last_info(mp_plan_info *out) {
    *out = last_plan_info();
    return MP_OK;
}

const char *mp_last_error(void) { return last_error(); }

int mp_device_count(void) {
    int c = 0;
    if (cudaGetDeviceCount(&c) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return c;
}

const char *mp_version(void) { return "memplan_b200 0.1 (sm_100a)"; }

}  // extern "C"
