// nccl_shim.cpp -- TEST INFRASTRUCTURE, not part of the product.
//
// A stand-in for libnccl.so.2 (built with that SONAME) that lets the
// engine's NCCL transport run with several ranks on ONE GPU: real NCCL
// refuses two ranks on one device ("duplicate GPU"), and this box has one.
// Ranks are engines of one process, each driven from its own host thread.
//
// Semantics kept from NCCL: ncclSend / ncclRecv are stream-ordered and
// matched per (sender, receiver) pair in posting order.  ncclSend snapshots
// the send buffer into a stream-ordered staging allocation on the sender's
// stream and never blocks; ncclRecv blocks the calling host thread until
// the matching send has been posted, then makes the receiver's stream wait
// for the snapshot and copies it.  Groups are no-ops: every group posts its
// sends before its receives, so no rank waits on a receive its peer has not
// reached.  Only ncclFloat64 payloads (what the engine sends).
#include <cuda_runtime.h>
#include <nccl.h>

#include <condition_variable>
#include <cstring>
#include <deque>
#include <map>
#include <memory>
#include <mutex>
#include <random>
#include <string>
#include <utility>

namespace {

struct Msg {
    void *stage;
    size_t bytes;
    cudaEvent_t ready;
};

struct Clique {
    std::mutex mu;
    std::condition_variable cv;
    std::map<std::pair<int, int>, std::deque<Msg>> q;  // (src, dst) -> FIFO
};

std::mutex g_mu;
std::map<std::string, std::shared_ptr<Clique>> g_cliques;

}  // namespace

struct ncclComm {
    std::shared_ptr<Clique> c;
    int rank, nranks;
};

extern "C" {

ncclResult_t ncclGetUniqueId(ncclUniqueId *id) {
    std::random_device rd;
    for (int i = 0; i < NCCL_UNIQUE_ID_BYTES; ++i) id->internal[i] = (char)(rd() & 0xff);
    return ncclSuccess;
}

ncclResult_t ncclCommInitRank(ncclComm_t *comm, int nranks, ncclUniqueId id, int rank) {
    if (rank < 0 || rank >= nranks) return ncclInvalidArgument;
    std::string key(id.internal, NCCL_UNIQUE_ID_BYTES);
    std::lock_guard<std::mutex> lk(g_mu);
    auto &c = g_cliques[key];
    if (!c) c = std::make_shared<Clique>();
    *comm = new ncclComm{c, rank, nranks};
    return ncclSuccess;
}

ncclResult_t ncclCommDestroy(ncclComm_t comm) {
    delete comm;
    return ncclSuccess;
}

ncclResult_t ncclGroupStart() { return ncclSuccess; }
ncclResult_t ncclGroupEnd() { return ncclSuccess; }

ncclResult_t ncclSend(const void *buf, size_t count, ncclDataType_t dt, int peer, ncclComm_t comm,
                      cudaStream_t st) {
    if (dt != ncclFloat64 || peer < 0 || peer >= comm->nranks) return ncclInvalidArgument;
    Msg m{nullptr, count * sizeof(double), nullptr};
    if (cudaMallocAsync(&m.stage, m.bytes ? m.bytes : 8, st) != cudaSuccess ||
        cudaMemcpyAsync(m.stage, buf, m.bytes, cudaMemcpyDeviceToDevice, st) != cudaSuccess ||
        cudaEventCreateWithFlags(&m.ready, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventRecord(m.ready, st) != cudaSuccess)
        return ncclUnhandledCudaError;
    Clique &c = *comm->c;
    {
        std::lock_guard<std::mutex> lk(c.mu);
        c.q[{comm->rank, peer}].push_back(m);
    }
    c.cv.notify_all();
    return ncclSuccess;
}

ncclResult_t ncclRecv(void *buf, size_t count, ncclDataType_t dt, int peer, ncclComm_t comm,
                      cudaStream_t st) {
    if (dt != ncclFloat64 || peer < 0 || peer >= comm->nranks) return ncclInvalidArgument;
    Clique &c = *comm->c;
    Msg m;
    {
        std::unique_lock<std::mutex> lk(c.mu);
        auto &fifo = c.q[{peer, comm->rank}];
        c.cv.wait(lk, [&] { return !fifo.empty(); });
        m = fifo.front();
        fifo.pop_front();
    }
    if (m.bytes != count * sizeof(double)) return ncclInvalidUsage;
    if (cudaStreamWaitEvent(st, m.ready, 0) != cudaSuccess ||
        cudaMemcpyAsync(buf, m.stage, m.bytes, cudaMemcpyDeviceToDevice, st) != cudaSuccess ||
        cudaFreeAsync(m.stage, st) != cudaSuccess || cudaEventDestroy(m.ready) != cudaSuccess)
        return ncclUnhandledCudaError;
    return ncclSuccess;
}

const char *ncclGetErrorString(ncclResult_t r) {
    return r == ncclSuccess ? "no error (nccl shim)" : "nccl shim error";
}

}  // extern "C"
