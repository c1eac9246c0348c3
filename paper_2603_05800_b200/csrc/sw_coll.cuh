// sw_coll.cuh -- the cross-rank exchange step of the path.
//
// Every collective of libsw_plan.so goes through Coll: NCCL over NVLink/NVSwitch in
// production, or an in-process LOOPBACK group that emulates R ranks inside one process
// (one host thread and one stream per rank, any devices -- several ranks may share one
// GPU, which NCCL refuses).  The loopback exists so that the real device merge path
// (select_final_kernel over gathered winners, front_gather_pad_kernel + the cooperative
// Pareto merge over gathered fronts, the digest reduction) runs, and is checked against
// the oracle, on a one-GPU box.  It has NCCL's stream semantics: a collective is enqueued
// on the caller's stream, reads the peers' send buffers only after the work that wrote
// them, and the caller's later work on its send buffer waits until every peer has copied.
//
// Synchronisation with a multi-rank communicator polls ncclCommGetAsyncError while
// waiting and gives up after SW_NCCL_TIMEOUT_S seconds (default 600): a dead or
// diverged peer becomes SW_ENCCL instead of a hang.
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

#include <chrono>
#include <condition_variable>
#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <set>
#include <thread>
#include <vector>

#include "sw_plan.h"

namespace sw {

// ---------------------------------------------------------------- loopback group
struct LoopGroup {
    int n = 0;
    int alive = 0;  // ranks not yet destroyed
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t gen = 0;
    std::vector<const void*> send;
    std::vector<cudaEvent_t> ready, done;
    // generation barrier: returns when all n ranks have arrived
    void barrier() {
        std::unique_lock<std::mutex> lk(mu);
        const uint64_t g = gen;
        if (++arrived == n) {
            arrived = 0;
            gen++;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != g; });
        }
    }
};

struct LoopComm {
    uint64_t magic;
    LoopGroup* g;
    int rank;
};
constexpr uint64_t kLoopMagic = 0x53574c4f4f504241ull;  // "SWLOOPBA"

inline std::mutex& loop_registry_mu() {
    static std::mutex m;
    return m;
}
inline std::set<const void*>& loop_registry() {
    static std::set<const void*> s;
    return s;
}
// Is this communicator pointer a loopback rank created by sw_comm_loopback_create?
// NCCL communicators the library aborted after an asynchronous error or a timeout
// (sw_comm_destroy must not destroy them again)
inline std::set<const void*>& aborted_registry() {
    static std::set<const void*> s;
    return s;
}
inline void abort_comm(ncclComm_t c) {
    {
        std::lock_guard<std::mutex> lk(loop_registry_mu());
        aborted_registry().insert(c);
    }
    ncclCommAbort(c);
}
inline LoopComm* as_loop(const void* c) {
    if (!c) return nullptr;
    std::lock_guard<std::mutex> lk(loop_registry_mu());
    return loop_registry().count(c) ? (LoopComm*)c : nullptr;
}

// ---------------------------------------------------------------- Coll
struct Coll {
    ncclComm_t nccl = nullptr;
    LoopComm* loop = nullptr;
    cudaStream_t stream = nullptr;
    int rank = 0, nranks = 1;
};

// a = reduce over R rows of `count` u64 (op 0 sum, 1 max)
__global__ void coll_reduce_u64_kernel(const uint64_t* __restrict__ in, int R, uint32_t count, int op,
                                       uint64_t* __restrict__ out) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    uint64_t a = in[i];
    for (int r = 1; r < R; r++) {
        const uint64_t b = in[(uint64_t)r * count + i];
        a = op ? (b > a ? b : a) : a + b;
    }
    out[i] = a;
}

// recv[r * bytes, (r + 1) * bytes) = rank r's send[0, bytes)
inline cudaError_t loop_allgather(const Coll& c, const void* send, void* recv, size_t bytes) {
    LoopGroup* g = c.loop->g;
    const int r = c.loop->rank;
    cudaError_t e = cudaEventRecord(g->ready[r], c.stream);
    g->send[r] = send;
    g->barrier();  // every rank's send buffer and ready event published
    for (int q = 0; q < g->n && e == cudaSuccess; q++) {
        e = cudaStreamWaitEvent(c.stream, g->ready[q], 0);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync((char*)recv + (size_t)q * bytes, g->send[q], bytes, cudaMemcpyDefault, c.stream);
    }
    if (e == cudaSuccess) e = cudaEventRecord(g->done[r], c.stream);
    g->barrier();  // every rank's copies enqueued
    for (int q = 0; q < g->n && e == cudaSuccess; q++) e = cudaStreamWaitEvent(c.stream, g->done[q], 0);
    return e;
}

// The collectives used by the path; return SW_OK / SW_ENCCL / SW_ECUDA (message via *why).
inline sw_status coll_allgather(const Coll& c, const void* send, void* recv, size_t bytes, const char** why) {
    if (c.nranks == 1) {
        *why = "";
        return cudaMemcpyAsync(recv, send, bytes, cudaMemcpyDeviceToDevice, c.stream) == cudaSuccess ? SW_OK : SW_ECUDA;
    }
    if (c.loop) {
        cudaError_t e = loop_allgather(c, send, recv, bytes);
        *why = cudaGetErrorString(e);
        return e == cudaSuccess ? SW_OK : SW_ECUDA;
    }
    ncclResult_t r = ncclAllGather(send, recv, bytes, ncclUint8, c.nccl, c.stream);
    *why = ncclGetErrorString(r);
    return r == ncclSuccess ? SW_OK : SW_ENCCL;
}

// In place over count u64: op 0 = sum (mod 2^64), 1 = max.
inline sw_status coll_allreduce_u64(const Coll& c, uint64_t* buf, uint32_t count, int op, const char** why) {
    *why = "";
    if (c.nranks == 1) return SW_OK;
    if (c.loop) {
        uint64_t* tmp = nullptr;
        const size_t bytes = (size_t)count * 8;
        cudaError_t e = cudaMallocAsync((void**)&tmp, bytes * c.nranks, c.stream);
        if (e == cudaSuccess) e = loop_allgather(c, buf, tmp, bytes);
        if (e == cudaSuccess) {
            coll_reduce_u64_kernel<<<(count + 127) / 128, 128, 0, c.stream>>>(tmp, c.nranks, count, op, buf);
            e = cudaGetLastError();
        }
        if (tmp) cudaFreeAsync(tmp, c.stream);
        *why = cudaGetErrorString(e);
        return e == cudaSuccess ? SW_OK : SW_ECUDA;
    }
    ncclResult_t r = ncclAllReduce(buf, buf, count, ncclUint64, op ? ncclMax : ncclSum, c.nccl, c.stream);
    *why = ncclGetErrorString(r);
    return r == ncclSuccess ? SW_OK : SW_ENCCL;
}

// Wait for the stream.  With an NCCL communicator of > 1 rank: poll, checking the
// communicator's asynchronous error state, and abort the communicator after the timeout
// (SW_NCCL_TIMEOUT_S, default 600 s) so that a dead or diverged peer cannot hang the
// caller forever.  Returns SW_OK, SW_ECUDA or SW_ENCCL.
inline sw_status coll_sync(const Coll& c, const char** why) {
    *why = "";
    if (c.nranks == 1 || c.loop || !c.nccl) {
        cudaError_t e = cudaStreamSynchronize(c.stream);
        *why = cudaGetErrorString(e);
        return e == cudaSuccess ? SW_OK : SW_ECUDA;
    }
    static const double timeout_s = [] {
        const char* ev = getenv("SW_NCCL_TIMEOUT_S");
        return ev ? atof(ev) : 600.0;
    }();
    const auto t0 = std::chrono::steady_clock::now();
    for (uint32_t spin = 0;; spin++) {
        cudaError_t e = cudaStreamQuery(c.stream);
        if (e == cudaSuccess) return SW_OK;
        if (e != cudaErrorNotReady) {
            *why = cudaGetErrorString(e);
            return SW_ECUDA;
        }
        ncclResult_t ae = ncclSuccess;
        ncclResult_t q = ncclCommGetAsyncError(c.nccl, &ae);
        if (q != ncclSuccess || ae != ncclSuccess) {
            *why = ncclGetErrorString(q != ncclSuccess ? q : ae);
            abort_comm(c.nccl);
            return SW_ENCCL;
        }
        const double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (dt > timeout_s) {
            *why = "timeout waiting for a collective (a peer rank is dead or made a different call)";
            abort_comm(c.nccl);
            return SW_ENCCL;
        }
        if (spin > 64) std::this_thread::sleep_for(std::chrono::microseconds(20));
    }
}

}  // namespace sw
