// comm.cu -- communicator backends of the row-partitioned path.
//
// The distributed solve needs exactly two stream-ordered exchange steps:
//   * a grouped point-to-point exchange: the halo of every distributed SpMV-class pass and the
//     allgatherv of the restricted residual at the gather level;
//   * an equal-size allgather: the batched partial dot products of the FCG recurrences, which every
//     rank then sums in rank order (so every rank holds bit-identical scalars, whatever algorithm
//     the collective uses).
// Backends:
//   * NcclComm -- one process per GPU; NCCL (grouped ncclSend/ncclRecv, ncclAllGather) over
//     NVLink 5 / NVSwitch.  libnccl.so.2 is opened at run time (dlopen), so single-GPU users need
//     no NCCL at all and the library uses whichever libnccl the process already loaded (torch's).
//   * ThreadComm -- P ranks as P host threads of one process on one device (test emulation of the
//     multi-GPU path on a single B200).  Every call: synchronise the caller's stream, meet at a host
//     barrier, copy peer buffers device-to-device, synchronise, meet again.  No kernel waits on
//     another rank's kernel.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <condition_variable>
#include <cstring>
#include <memory>
#include <mutex>

#include "../../include/amg.h"
#include "amg_internal.h"

namespace amg {

// ------------------------------------------------------------------ NCCL (dlopen)
struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

static NcclApi* nccl_api() {
    static NcclApi api;
    static bool tried = false, ok = false;
    static std::mutex mu;
    std::lock_guard<std::mutex> lk(mu);
    if (!tried) {
        tried = true;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (h) {
            api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
            api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
            api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
            api.Send = (decltype(api.Send))dlsym(h, "ncclSend");
            api.Recv = (decltype(api.Recv))dlsym(h, "ncclRecv");
            api.AllGather = (decltype(api.AllGather))dlsym(h, "ncclAllGather");
            api.GroupStart = (decltype(api.GroupStart))dlsym(h, "ncclGroupStart");
            api.GroupEnd = (decltype(api.GroupEnd))dlsym(h, "ncclGroupEnd");
            api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
            ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.Send && api.Recv && api.AllGather &&
                 api.GroupStart && api.GroupEnd && api.GetErrorString;
        }
    }
    if (!ok) throw Error(AMG_E_NCCL, "libnccl.so.2 could not be loaded (dlopen/dlsym)");
    return &api;
}

static void nccl_check(ncclResult_t r, const char* what) {
    if (r == ncclSuccess) return;
    std::string m = std::string(what) + " failed: " + nccl_api()->GetErrorString(r);
    throw Error(AMG_E_NCCL, m);
}

struct NcclComm final : Comm {
    ncclComm_t comm = nullptr;
    ~NcclComm() override {
        if (comm) nccl_api()->CommDestroy(comm);
    }
    void sendrecv(const std::vector<P2P>& sends, const std::vector<P2P>& recvs, cudaStream_t s) override {
        if (sends.empty() && recvs.empty()) return;
        NcclApi* A = nccl_api();
        nccl_check(A->GroupStart(), "ncclGroupStart");
        for (const P2P& p : sends) nccl_check(A->Send(p.ptr, p.bytes, ncclUint8, p.peer, comm, s), "ncclSend");
        for (const P2P& p : recvs) nccl_check(A->Recv(p.ptr, p.bytes, ncclUint8, p.peer, comm, s), "ncclRecv");
        nccl_check(A->GroupEnd(), "ncclGroupEnd");
    }
    void allgather(const void* in, void* out, size_t bytes, cudaStream_t s) override {
        nccl_check(nccl_api()->AllGather(in, out, bytes, ncclUint8, comm, s), "ncclAllGather");
    }
    bool capturable() const override { return true; }
    const char* kind() const override { return "nccl"; }
};

// ------------------------------------------------------------------ in-process threads
struct ThreadShared {
    int P = 0;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    long long gen = 0;
    bool aborted = false;
    std::vector<std::vector<P2P>> posted;  // per rank: its sends of the current exchange
    std::vector<const void*> agin;         // per rank: its allgather input
    int live = 0;                          // communicators not yet freed
};

struct ThreadComm final : Comm {
    std::shared_ptr<ThreadShared> sh;
    ~ThreadComm() override {}
    // host barrier of the P threads; a rank that fails mid-exchange aborts the group (no hang)
    void barrier() {
        std::unique_lock<std::mutex> lk(sh->mu);
        if (sh->aborted) throw Error(AMG_E_NCCL, "thread communicator aborted by another rank");
        const long long g = sh->gen;
        if (++sh->arrived == sh->P) {
            sh->arrived = 0;
            ++sh->gen;
            sh->cv.notify_all();
            return;
        }
        const bool ok = sh->cv.wait_for(lk, std::chrono::seconds(300), [&] { return sh->gen != g || sh->aborted; });
        if (sh->gen != g) return;  // the barrier completed (an abort after it concerns later exchanges)
        if (!ok || sh->aborted) {
            sh->aborted = true;
            sh->cv.notify_all();
            throw Error(AMG_E_NCCL, ok ? "thread communicator aborted by another rank" : "thread communicator timeout");
        }
    }
    void abort() override { abort_group(); }
    void abort_group() {
        std::lock_guard<std::mutex> lk(sh->mu);
        sh->aborted = true;
        sh->cv.notify_all();
    }
    void sendrecv(const std::vector<P2P>& sends, const std::vector<P2P>& recvs, cudaStream_t s) override {
        static const bool trace = getenv("AMG_COMM_TRACE") != nullptr;
        if (trace) {
            std::string m = "[comm] rank " + std::to_string(rank) + " sends";
            for (const P2P& p : sends) m += " " + std::to_string(p.peer) + ":" + std::to_string(p.bytes);
            m += " recvs";
            for (const P2P& p : recvs) m += " " + std::to_string(p.peer) + ":" + std::to_string(p.bytes);
            fprintf(stderr, "%s\n", m.c_str());
        }
        try {
            {
                std::lock_guard<std::mutex> lk(sh->mu);
                sh->posted[rank] = sends;
            }
            CK(cudaStreamSynchronize(s));
            barrier();
            std::vector<int> seen(size, 0);
            for (const P2P& r : recvs) {
                const std::vector<P2P>& ps = sh->posted[r.peer];
                int k = seen[r.peer]++, found = -1;
                for (size_t j = 0; j < ps.size(); ++j)
                    if (ps[j].peer == rank && k-- == 0) { found = (int)j; break; }
                if (found < 0 || ps[found].bytes != r.bytes)
                    throw Error(AMG_E_NCCL, "thread communicator: unmatched or mis-sized message (rank " +
                                                std::to_string(rank) + " <- " + std::to_string(r.peer) + ": expected " +
                                                std::to_string(r.bytes) + " bytes, posted " +
                                                (found < 0 ? std::string("none") : std::to_string(ps[found].bytes)) + ")");
                if (r.bytes) CK(cudaMemcpyAsync(r.ptr, ps[found].ptr, r.bytes, cudaMemcpyDeviceToDevice, s));
            }
            CK(cudaStreamSynchronize(s));
            barrier();
        } catch (...) {
            abort_group();
            throw;
        }
    }
    void allgather(const void* in, void* out, size_t bytes, cudaStream_t s) override {
        try {
            {
                std::lock_guard<std::mutex> lk(sh->mu);
                sh->agin[rank] = in;
            }
            CK(cudaStreamSynchronize(s));
            barrier();
            for (int r = 0; r < size; ++r)
                if (bytes)
                    CK(cudaMemcpyAsync(static_cast<char*>(out) + (size_t)r * bytes, sh->agin[r], bytes,
                                       cudaMemcpyDeviceToDevice, s));
            CK(cudaStreamSynchronize(s));
            barrier();
        } catch (...) {
            abort_group();
            throw;
        }
    }
    bool capturable() const override { return false; }
    const char* kind() const override { return "threads"; }
};

}  // namespace amg

using namespace amg;

extern "C" {

int amg_comm_unique_id(uint8_t* id) {
    if (!id) { set_last_error("amg_comm_unique_id: NULL"); return AMG_E_ARG; }
    try {
        ncclUniqueId u;
        nccl_check(nccl_api()->GetUniqueId(&u), "ncclGetUniqueId");
        memcpy(id, u.internal, AMG_COMM_ID_BYTES);
    } catch (const Error& e) {
        set_last_error(e.what());
        return e.code;
    }
    return AMG_OK;
}

int amg_comm_init_nccl(amg_comm* out, const uint8_t* id, int32_t nranks, int32_t rank) {
    if (!out || !id || nranks < 1 || rank < 0 || rank >= nranks) {
        set_last_error("amg_comm_init_nccl: bad arguments");
        return AMG_E_ARG;
    }
    *out = nullptr;
    NcclComm* c = new NcclComm();
    try {
        ncclUniqueId u;
        memcpy(u.internal, id, AMG_COMM_ID_BYTES);
        nccl_check(nccl_api()->CommInitRank(&c->comm, nranks, u, rank), "ncclCommInitRank");
        c->rank = rank;
        c->size = nranks;
    } catch (const Error& e) {
        set_last_error(e.what());
        delete c;
        return e.code;
    }
    amg_comm h = new amg_comm_s();
    h->c = c;
    *out = h;
    return AMG_OK;
}

int amg_comm_init_threads(amg_comm* out, int32_t nranks) {
    if (!out || nranks < 1) { set_last_error("amg_comm_init_threads: bad arguments"); return AMG_E_ARG; }
    auto sh = std::make_shared<ThreadShared>();
    sh->P = nranks;
    sh->posted.resize(nranks);
    sh->agin.resize(nranks, nullptr);
    sh->live = nranks;
    for (int r = 0; r < nranks; ++r) {
        ThreadComm* c = new ThreadComm();
        c->sh = sh;
        c->rank = r;
        c->size = nranks;
        out[r] = new amg_comm_s();
        out[r]->c = c;
    }
    return AMG_OK;
}

int amg_comm_rank(amg_comm c, int32_t* rank, int32_t* size) {
    if (!c || !c->c) { set_last_error("amg_comm_rank: NULL"); return AMG_E_ARG; }
    if (rank) *rank = c->c->rank;
    if (size) *size = c->c->size;
    return AMG_OK;
}

int amg_comm_free(amg_comm c) {
    if (!c) return AMG_OK;
    delete c->c;
    delete c;
    return AMG_OK;
}

}  // extern "C"
