// Pipelined batched planning from host arrays (mp_pipe_*).
//
// A caller planning a stream of batches (profiles arriving from many jobs,
// mini-batch sweeps) with mp_plan_bestfit_batched pays, per batch, the
// upload, K0 + the planner and the download back to back.  The planner
// holds every register of every SM (16 one-warp traces per SM at 128
// registers), so nothing else computes beside it — but the copy engines
// are idle.  A pipe keeps two device slots and three streams:
//
//   caller thread : H2D(k) on `in`            (overlaps plan(k-1))
//   worker thread : plan_device(k) on `comp`   (waits for H2D(k))
//                   D2H(k) on `out`            (overlaps plan(k+1))
//
// so in steady state a batch costs max(K0 + planner, copies) instead of
// their sum.  Same results as mp_plan_bestfit_batched (the same
// plan_device on the same inputs); the caller's host arrays must stay
// untouched until mp_pipe_wait(ticket) returns.  Batches beyond the
// device-memory limit of one K0 pass run synchronously (chunked) on the
// worker.
#include <condition_variable>
#include <deque>
#include <map>
#include <mutex>
#include <thread>
#include <vector>

#include "common.h"
#include "plan.h"

namespace {

using namespace mp;

struct Job {
    int64_t ticket;
    int slot;
    std::vector<int64_t> tp;  // host CSR offsets (sizes the launch)
    int64_t T, N;
    int64_t *offsets_out, *peaks_out;
    const int64_t *alloc, *free_, *size;  // host inputs (oversize batches only)
    int flags;
    bool direct;  // inputs uploaded into the slot
};

struct Slot {
    void *dev = nullptr;
    size_t cap = 0;
    cudaEvent_t in_done = nullptr, out_done = nullptr;
    int64_t ticket = -1;  // last job using the slot
};

}  // namespace

struct mp_plan_pipe {
    int device = 0;
    cudaStream_t in = nullptr, comp = nullptr, out = nullptr;
    Slot slot[2];
    std::mutex mu;
    std::condition_variable cv;
    std::deque<Job> queue;
    std::map<int64_t, int> result;  // ticket -> status, once its download is enqueued
    std::map<int64_t, bool> synced;
    std::map<int64_t, std::string> err;
    int64_t next = 0;
    int64_t limit = 0;  // blocks one slot / one K0 pass takes (pipe_block_limit)
    int64_t expired = 0;  // tickets below this were forgotten (kExpire behind `next`)
    bool stop = false;
    std::thread worker;
};

namespace {

// results of the last kExpire tickets are kept for mp_pipe_wait (older
// ones were synced when their slot was reused)
constexpr int64_t kExpire = 1024;

int64_t pipe_block_limit() {
    if (const char *env = getenv("MEMPLAN_MAX_BATCH_BLOCKS")) return std::max<int64_t>(1, atoll(env));
    size_t free_b = 0, total_b = 0;
    int64_t lim = int64_t(1) << 29;
    // two slots of 32 B/block plus the planner's ~110 B/block of tables
    if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess)
        lim = std::min<int64_t>(lim, (int64_t)(free_b / 200));
    cudaGetLastError();
    return std::max<int64_t>(lim, int64_t(1) << 20);
}

int run_job(mp_plan_pipe *p, Job &j) {
    if (!j.direct)  // oversize: the ordinary (chunked) host-array call
        return mp_plan_bestfit_batched(j.tp.data(), j.alloc, j.free_, j.size, j.T, j.offsets_out,
                                       j.peaks_out, j.flags & ~MP_DEVICE_PTRS, p->device,
                                       (mp_stream_t)p->comp);
    Slot &sl = p->slot[j.slot];
    int64_t *tp_d = static_cast<int64_t *>(sl.dev);
    int64_t *a_d = tp_d + (j.T + 1), *f_d = a_d + j.N, *s_d = f_d + j.N;
    int64_t *o_d = s_d + j.N, *p_d = o_d + j.N;
    MP_CUDA(cudaStreamWaitEvent(p->comp, sl.in_done, 0));
    MP_TRY(plan_device(tp_d, j.tp.data(), j.T, a_d, f_d, s_d, o_d, p_d, j.flags & ~MP_DEVICE_PTRS,
                       p->device, p->comp));
    // plan_device synchronised `comp`: the results are final
    if (j.N) MP_CUDA(cudaMemcpyAsync(j.offsets_out, o_d, sizeof(int64_t) * j.N,
                                     cudaMemcpyDeviceToHost, p->out));
    if (j.T) MP_CUDA(cudaMemcpyAsync(j.peaks_out, p_d, sizeof(int64_t) * j.T,
                                     cudaMemcpyDeviceToHost, p->out));
    MP_CUDA(cudaEventRecord(sl.out_done, p->out));
    return MP_OK;
}

void worker_main(mp_plan_pipe *p) {
    cudaSetDevice(p->device);
    for (;;) {
        Job j;
        {
            std::unique_lock<std::mutex> lk(p->mu);
            p->cv.wait(lk, [&] { return p->stop || !p->queue.empty(); });
            if (p->queue.empty()) return;
            j = std::move(p->queue.front());
            p->queue.pop_front();
        }
        const int rc = run_job(p, j);
        std::lock_guard<std::mutex> lk(p->mu);
        p->result[j.ticket] = rc;
        // a failed or synchronous job has nothing in flight
        p->synced[j.ticket] = rc != MP_OK || !j.direct;
        if (rc != MP_OK) p->err[j.ticket] = last_error();
        p->cv.notify_all();
    }
}

// Block until `ticket` is complete (download landed); caller holds `lk`.
int finish(mp_plan_pipe *p, std::unique_lock<std::mutex> &lk, int64_t ticket) {
    p->cv.wait(lk, [&] { return p->result.count(ticket) != 0; });
    if (!p->synced[ticket]) {
        const Slot &sl = p->slot[ticket & 1];
        // the slot's event still belongs to `ticket`: ticket + 2 cannot be
        // submitted before this ticket is synced
        const cudaError_t e = cudaEventSynchronize(sl.out_done);
        p->synced[ticket] = true;
        if (e != cudaSuccess) {
            p->result[ticket] = cuda_fail(e, "cudaEventSynchronize(pipe download)");
            p->err[ticket] = last_error();
        }
    }
    return p->result[ticket];
}

}  // namespace

extern "C" {

mp_plan_pipe *mp_pipe_create(int device) {
    if (use_device(device) != MP_OK) return nullptr;
    auto *p = new mp_plan_pipe();
    p->device = device;
    bool ok = cudaStreamCreateWithFlags(&p->in, cudaStreamNonBlocking) == cudaSuccess &&
              cudaStreamCreateWithFlags(&p->comp, cudaStreamNonBlocking) == cudaSuccess &&
              cudaStreamCreateWithFlags(&p->out, cudaStreamNonBlocking) == cudaSuccess;
    for (auto &s : p->slot)
        ok = ok && cudaEventCreateWithFlags(&s.in_done, cudaEventDisableTiming) == cudaSuccess &&
             cudaEventCreateWithFlags(&s.out_done, cudaEventDisableTiming) == cudaSuccess;
    if (!ok) {
        cuda_fail(cudaGetLastError(), "mp_pipe_create");
        mp_pipe_destroy(p);
        return nullptr;
    }
    p->worker = std::thread(worker_main, p);
    return p;
}

int mp_pipe_submit(mp_plan_pipe *p, const int64_t *trace_ptr, const int64_t *alloc,
                   const int64_t *free_, const int64_t *size, int64_t T, int64_t *offsets_out,
                   int64_t *peaks_out, int flags, int64_t *ticket_out) {
    if (!p) {
        set_error("null pipe");
        return MP_ERR_INVALID;
    }
    if (T < 0) {
        set_error("negative trace count");
        return MP_ERR_INVALID;
    }
    if (flags & MP_DEVICE_PTRS) {
        set_error("mp_pipe_submit takes host arrays");
        return MP_ERR_INVALID;
    }
    MP_TRY(use_device(p->device));
    Job j;
    j.tp.assign(trace_ptr, trace_ptr + T + 1);
    if (T && j.tp[0] != 0) {
        set_error("trace_ptr[0] must be 0");
        return MP_ERR_INVALID;
    }
    for (int64_t t = 0; t < T; t++)
        if (j.tp[t + 1] < j.tp[t]) {
            set_error("trace_ptr must be non-decreasing");
            return MP_ERR_INVALID;
        }
    j.T = T;
    j.N = T ? j.tp[T] : 0;
    j.offsets_out = offsets_out;
    j.peaks_out = peaks_out;
    j.alloc = alloc;
    j.free_ = free_;
    j.size = size;
    j.flags = flags;
    std::unique_lock<std::mutex> lk(p->mu);
    // cudaMemGetInfo costs far more than a small batch's upload: query it
    // only when a batch outgrows the last answer
    if (j.N > p->limit) p->limit = pipe_block_limit();
    j.direct = j.N <= p->limit;
    j.ticket = p->next++;
    j.slot = (int)(j.ticket & 1);
    while (!p->result.empty() && p->result.begin()->first < j.ticket - kExpire) {
        const int64_t old = p->result.begin()->first;
        p->result.erase(old);
        p->synced.erase(old);
        p->err.erase(old);
        p->expired = old + 1;
    }
    *ticket_out = j.ticket;
    Slot &sl = p->slot[j.slot];
    // the slot's previous batch must have landed on the host
    if (sl.ticket >= 0) finish(p, lk, sl.ticket);
    sl.ticket = j.ticket;
    auto upload = [&]() -> int {
        const size_t need = sizeof(int64_t) * ((size_t)T + 1 + 4 * (size_t)j.N + (size_t)T) + 256;
        if (need > sl.cap) {
            if (sl.dev) cudaFree(sl.dev);
            sl.dev = nullptr;
            sl.cap = 0;
            MP_CUDA(cudaMalloc(&sl.dev, need));
            sl.cap = need;
        }
        int64_t *tp_d = static_cast<int64_t *>(sl.dev);
        int64_t *a_d = tp_d + (T + 1), *f_d = a_d + j.N, *s_d = f_d + j.N;
        const size_t nb = sizeof(int64_t) * (size_t)j.N;
        // j.tp is pageable: the copy is staged before the call returns
        MP_CUDA(cudaMemcpyAsync(tp_d, j.tp.data(), sizeof(int64_t) * (T + 1),
                                cudaMemcpyHostToDevice, p->in));
        if (j.N) {
            MP_CUDA(cudaMemcpyAsync(a_d, alloc, nb, cudaMemcpyHostToDevice, p->in));
            MP_CUDA(cudaMemcpyAsync(f_d, free_, nb, cudaMemcpyHostToDevice, p->in));
            MP_CUDA(cudaMemcpyAsync(s_d, size, nb, cudaMemcpyHostToDevice, p->in));
        }
        MP_CUDA(cudaEventRecord(sl.in_done, p->in));
        return MP_OK;
    };
    const int rc = j.direct ? upload() : MP_OK;
    if (rc != MP_OK) {  // the ticket completes with the failure
        p->result[j.ticket] = rc;
        p->synced[j.ticket] = true;
        p->err[j.ticket] = last_error();
        return rc;
    }
    p->queue.push_back(std::move(j));
    p->cv.notify_all();
    return MP_OK;
}

int mp_pipe_wait(mp_plan_pipe *p, int64_t ticket) {
    if (!p) {
        set_error("null pipe");
        return MP_ERR_INVALID;
    }
    std::unique_lock<std::mutex> lk(p->mu);
    if (ticket < 0 || ticket >= p->next) {
        set_error("unknown pipe ticket");
        return MP_ERR_INVALID;
    }
    if (ticket < p->expired) {
        set_error("pipe ticket expired (more than 1024 submits ago)");
        return MP_ERR_INVALID;
    }
    const int rc = finish(p, lk, ticket);
    if (rc != MP_OK) set_error(p->err[ticket]);
    return rc;
}

void mp_pipe_destroy(mp_plan_pipe *p) {
    if (!p) return;
    if (p->worker.joinable()) {
        {
            std::lock_guard<std::mutex> lk(p->mu);
            p->stop = true;
            p->cv.notify_all();
        }
        p->worker.join();
    }
    cudaSetDevice(p->device);
    for (cudaStream_t s : {p->in, p->comp, p->out})
        if (s) cudaStreamSynchronize(s);
    for (auto &s : p->slot) {
        if (s.dev) cudaFree(s.dev);
        if (s.in_done) cudaEventDestroy(s.in_done);
        if (s.out_done) cudaEventDestroy(s.out_done);
    }
    for (cudaStream_t s : {p->in, p->comp, p->out})
        if (s) cudaStreamDestroy(s);
    cudaGetLastError();
    delete p;
}

}  // extern "C"
