// swe_transport.cu — row-strip collectives: NCCL (dlopen'ed, between GPUs) and
// the local group (contexts of one process on one device, for single-GPU tests).
#include <dlfcn.h>
#include <unistd.h>

#include <chrono>
#include <cstdio>
#include <condition_variable>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include <nccl.h>

#include "swe_runtime.h"

namespace swe_rt {
namespace {

// ---------------------------------------------------------------- NCCL (dlopen)
struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    bool load(std::string& err) {
        if (h) return true;
        const char* names[] = {"libnccl.so.2", "libnccl.so"};
        for (const char* n : names) {
            h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
            if (h) break;
        }
        if (!h) {
            err = "cannot dlopen libnccl.so.2";
            return false;
        }
#define SWE_SYM(f) f = reinterpret_cast<decltype(f)>(dlsym(h, "nccl" #f))
        SWE_SYM(GetUniqueId);
        SWE_SYM(CommInitRank);
        SWE_SYM(CommDestroy);
        SWE_SYM(AllReduce);
        SWE_SYM(Send);
        SWE_SYM(Recv);
        SWE_SYM(GroupStart);
        SWE_SYM(GroupEnd);
        SWE_SYM(GetErrorString);
#undef SWE_SYM
        if (!GetUniqueId || !CommInitRank || !AllReduce || !Send || !Recv || !GroupStart ||
            !GroupEnd) {
            err = "libnccl.so.2 lacks required symbols";
            return false;
        }
        return true;
    }
};
NcclApi g_nccl;

#define NCCL_TRY(x)                                                                              \
    do {                                                                                         \
        ncclResult_t r_ = (x);                                                                   \
        if (r_ != ncclSuccess)                                                                   \
            return set_status(st, SWE_ERR_RUNTIME, -1, -1, 0.0, "NCCL error %d at %s:%d",        \
                              static_cast<int>(r_), __FILE__, __LINE__);                         \
    } while (0)

// One communicator per (unique id, rank, size, device) and process: every
// Stepper of a rank built with the same id shares it (the bench and the CLI
// create several Steppers per run); destroyed with its last user.
struct CommEntry {
    ncclComm_t comm = nullptr;
    int refs = 0;
};
std::mutex g_comms_m;
std::map<std::string, CommEntry> g_comms;

struct NcclTransport final : Transport {
    ncclComm_t comm = nullptr;
    std::string key;
    std::vector<void*> ipc_opened;  // neighbour buffers mapped through CUDA IPC (closed with the transport)
    ~NcclTransport() override {
        for (void* q : ipc_opened) cudaIpcCloseMemHandle(q);
        std::lock_guard<std::mutex> lk(g_comms_m);
        auto it = g_comms.find(key);
        if (it != g_comms.end() && --it->second.refs == 0) {
            if (it->second.comm && g_nccl.CommDestroy) g_nccl.CommDestroy(it->second.comm);
            g_comms.erase(it);
        }
    }
    int allreduce_max(swe_ctx* c, cudaStream_t s, unsigned long long* d, int n, swe_status* st) override;
    int sendrecv(swe_ctx* c, cudaStream_t s, const void* su, void* ru, const void* sd, void* rd, size_t bytes,
                 swe_status* st) override;
    bool capturable() const override { return true; }
    int peer_buffers(swe_ctx* c, double* dn[2], double* up[2], int* nloc_dn, swe_status* st) override;
};


struct LocalGroup {
    std::mutex m;
    std::condition_variable cv;
    int n = 0, arrived = 0, refs = 0;
    unsigned long long gen = 0;
    bool broken = false;
    cudaEvent_t ready[kMaxLocalRanks] = {}, done[kMaxLocalRanks] = {};
    const void* su[kMaxLocalRanks] = {};
    const void* sd[kMaxLocalRanks] = {};
    const unsigned long long* red[kMaxLocalRanks] = {};
    double* buf[kMaxLocalRanks][2] = {};  // every rank's state buffers (fused halo push)
    int nloc[kMaxLocalRanks] = {};
    // all ranks arrive (or a 120 s timeout breaks the group, so a failing
    // test cannot hang the box)
    bool barrier() {
        std::unique_lock<std::mutex> lk(m);
        if (broken) return false;
        const unsigned long long g = gen;
        if (++arrived == n) {
            arrived = 0;
            ++gen;
            cv.notify_all();
            return true;
        }
        if (!cv.wait_for(lk, std::chrono::seconds(120), [&] { return gen != g || broken; })) broken = true;
        if (broken) {
            cv.notify_all();
            return false;
        }
        return true;
    }
};
std::mutex g_groups_m;
std::map<std::string, LocalGroup*> g_groups;

struct LocalTransport final : Transport {
    LocalGroup* grp = nullptr;
    std::string key;
    int rank = 0;
    ~LocalTransport() override {
        std::lock_guard<std::mutex> lk(g_groups_m);
        if (grp && --grp->refs == 0) {
            for (int r = 0; r < grp->n; ++r) {
                if (grp->ready[r]) cudaEventDestroy(grp->ready[r]);
                if (grp->done[r]) cudaEventDestroy(grp->done[r]);
            }
            g_groups.erase(key);
            delete grp;
        }
    }
    int allreduce_max(swe_ctx* c, cudaStream_t s, unsigned long long* d, int n, swe_status* st) override;
    int sendrecv(swe_ctx* c, cudaStream_t s, const void* su, void* ru, const void* sd, void* rd, size_t bytes,
                 swe_status* st) override;
    bool capturable() const override { return false; }
    int peer_buffers(swe_ctx* c, double* dn[2], double* up[2], int* nloc_dn, swe_status* st) override;
};

}  // namespace

int NcclTransport::allreduce_max(swe_ctx* c, cudaStream_t s, unsigned long long* d, int n, swe_status* st) {
    (void)c;
    NCCL_TRY(g_nccl.AllReduce(d, d, static_cast<size_t>(n), ncclUint64, ncclMax, comm, s));
    return SWE_OK;
}

int NcclTransport::sendrecv(swe_ctx* c, cudaStream_t s, const void* su, void* ru, const void* sd, void* rd,
                            size_t bytes, swe_status* st) {
    const int rk = c->ex.rank;
    NCCL_TRY(g_nccl.GroupStart());
    if (su) NCCL_TRY(g_nccl.Send(su, bytes, ncclUint8, rk + 1, comm, s));
    if (ru) NCCL_TRY(g_nccl.Recv(ru, bytes, ncclUint8, rk + 1, comm, s));
    if (sd) NCCL_TRY(g_nccl.Send(sd, bytes, ncclUint8, rk - 1, comm, s));
    if (rd) NCCL_TRY(g_nccl.Recv(rd, bytes, ncclUint8, rk - 1, comm, s));
    NCCL_TRY(g_nccl.GroupEnd());
    return SWE_OK;
}

#define GROUP_SYNC()                                                                                   \
    do {                                                                                               \
        if (!grp->barrier())                                                                           \
            return set_status(st, SWE_ERR_RUNTIME, -1, -1, 0.0, "local strip group: a rank timed out"); \
    } while (0)

// post -> barrier -> read the neighbours' posts -> barrier -> wait for the
// neighbours' reads before the posted rows may change again
int LocalTransport::sendrecv(swe_ctx* c, cudaStream_t s, const void* su, void* ru, const void* sd, void* rd,
                             size_t bytes, swe_status* st) {
    (void)c;
    const int r = rank, n = grp->n;
    grp->su[r] = su;
    grp->sd[r] = sd;
    CUDA_TRY(cudaEventRecord(grp->ready[r], s));
    GROUP_SYNC();
    if (ru && r + 1 < n) {
        CUDA_TRY(cudaStreamWaitEvent(s, grp->ready[r + 1], 0));
        CUDA_TRY(cudaMemcpyAsync(ru, grp->sd[r + 1], bytes, cudaMemcpyDeviceToDevice, s));
    }
    if (rd && r > 0) {
        CUDA_TRY(cudaStreamWaitEvent(s, grp->ready[r - 1], 0));
        CUDA_TRY(cudaMemcpyAsync(rd, grp->su[r - 1], bytes, cudaMemcpyDeviceToDevice, s));
    }
    CUDA_TRY(cudaEventRecord(grp->done[r], s));
    GROUP_SYNC();
    if (r + 1 < n) CUDA_TRY(cudaStreamWaitEvent(s, grp->done[r + 1], 0));
    if (r > 0) CUDA_TRY(cudaStreamWaitEvent(s, grp->done[r - 1], 0));
    return SWE_OK;
}

int LocalTransport::allreduce_max(swe_ctx* c, cudaStream_t s, unsigned long long* d, int n, swe_status* st) {
    const int r = rank, nr = grp->n;
    grp->red[r] = d;
    CUDA_TRY(cudaEventRecord(grp->ready[r], s));
    GROUP_SYNC();
    RedPtrs in{};
    for (int k = 0; k < nr; ++k) {
        CUDA_TRY(cudaStreamWaitEvent(s, grp->ready[k], 0));
        in.p[k] = grp->red[k];
    }
    max_reduce_kernel<<<1, 32, 0, s>>>(in, nr, n, c->d_xr);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaEventRecord(grp->done[r], s));
    GROUP_SYNC();
    for (int k = 0; k < nr; ++k) CUDA_TRY(cudaStreamWaitEvent(s, grp->done[k], 0));
    CUDA_TRY(cudaMemcpyAsync(d, c->d_xr, static_cast<size_t>(n) * sizeof(unsigned long long),
                             cudaMemcpyDeviceToDevice, s));
    return SWE_OK;
}
int LocalTransport::peer_buffers(swe_ctx* c, double* dn[2], double* up[2], int* nloc_dn, swe_status* st) {
    const int r = rank, n = grp->n;
    grp->buf[r][0] = c->d_buf[0];
    grp->buf[r][1] = c->d_buf[1];
    grp->nloc[r] = c->nloc;
    GROUP_SYNC();  // every rank has posted its buffers
    for (int k = 0; k < 2; ++k) {
        dn[k] = r > 0 ? grp->buf[r - 1][k] : nullptr;
        up[k] = r + 1 < n ? grp->buf[r + 1][k] : nullptr;
    }
    *nloc_dn = r > 0 ? grp->nloc[r - 1] : 0;
    GROUP_SYNC();
    return SWE_OK;
}
#undef GROUP_SYNC

// What a rank tells its strip neighbours about its state buffers.
struct PeerInfo {
    cudaIpcMemHandle_t h[2];
    double* ptr[2];
    int pid, device, nloc, ok;
};

int NcclTransport::peer_buffers(swe_ctx* c, double* dn[2], double* up[2], int* nloc_dn, swe_status* st) {
    dn[0] = dn[1] = up[0] = up[1] = nullptr;
    *nloc_dn = 0;
    PeerInfo mine{};
    mine.pid = static_cast<int>(getpid());
    mine.device = c->ex.device;
    mine.nloc = c->nloc;
    mine.ok = 1;
    for (int k = 0; k < 2; ++k) {
        mine.ptr[k] = c->d_buf[k];
        if (cudaIpcGetMemHandle(&mine.h[k], c->d_buf[k]) != cudaSuccess) mine.ok = 0;
    }
    cudaGetLastError();
    PeerInfo* d = nullptr;  // [mine, from up, from down]
    CUDA_TRY(cudaMalloc(&d, 3 * sizeof(PeerInfo)));
    CUDA_TRY(cudaMemcpyAsync(d, &mine, sizeof mine, cudaMemcpyHostToDevice, c->stream));
    const int rk = c->ex.rank, nr = c->ex.nranks;
    const bool has_up = rk + 1 < nr, has_dn = rk > 0;
    int rc = sendrecv(c, c->stream, has_up ? d : nullptr, has_up ? d + 1 : nullptr, has_dn ? d : nullptr,
                      has_dn ? d + 2 : nullptr, sizeof(PeerInfo), st);
    if (rc) {
        cudaFree(d);
        return rc;
    }
    PeerInfo got[2];
    CUDA_TRY(cudaMemcpyAsync(got, d + 1, 2 * sizeof(PeerInfo), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    cudaFree(d);
    auto map = [&](const PeerInfo& q, double* out[2]) {
        if (!q.ok) return false;
        if (q.pid == mine.pid) {  // strips of one process (the CLI's cuda:N): in-process peer access
            if (q.device != c->ex.device) {
                const cudaError_t e = cudaDeviceEnablePeerAccess(q.device, 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
                    cudaGetLastError();
                    return false;
                }
                cudaGetLastError();
            }
            out[0] = q.ptr[0];
            out[1] = q.ptr[1];
            return true;
        }
        for (int k = 0; k < 2; ++k) {  // another process: map its buffers over NVLink
            void* p = nullptr;
            if (cudaIpcOpenMemHandle(&p, q.h[k], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
                cudaGetLastError();
                return false;
            }
            ipc_opened.push_back(p);
            out[k] = static_cast<double*>(p);
        }
        return true;
    };
    bool ok = true;
    if (has_up) ok = map(got[0], up) && ok;
    if (has_dn) ok = map(got[1], dn) && ok;
    if (has_dn) *nloc_dn = got[1].nloc;
    if (!ok) {  // no peer path to a neighbour: the halo goes through NCCL send/recv
        dn[0] = dn[1] = up[0] = up[1] = nullptr;
        *nloc_dn = 0;
    }
    return SWE_OK;
}

int create_transport(swe_ctx* c, const swe_exec& ex, const void* nccl_id, swe_status* st) {
    if (ex.flags & SWE_EXEC_LOCAL_GROUP) {
        if (ex.nranks > kMaxLocalRanks)
            return set_status(st, SWE_ERR_CONFIG, -1, -1, 0, "exec: a local group holds at most %d ranks",
                              kMaxLocalRanks);
        auto* t = new LocalTransport();
        c->tr = t;
        t->key.assign(static_cast<const char*>(nccl_id), SWE_NCCL_ID_BYTES);
        t->rank = ex.rank;
        std::lock_guard<std::mutex> lk(g_groups_m);
        LocalGroup*& g = g_groups[t->key];
        if (!g) {
            g = new LocalGroup();
            g->n = ex.nranks;
        }
        if (g->n != ex.nranks)
            return set_status(st, SWE_ERR_CONFIG, -1, -1, 0, "exec: local group size mismatch");
        ++g->refs;
        t->grp = g;
        CUDA_TRY(cudaEventCreateWithFlags(&g->ready[ex.rank], cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&g->done[ex.rank], cudaEventDisableTiming));
    } else {
        std::string err;
        if (!g_nccl.load(err)) return set_status(st, SWE_ERR_RUNTIME, -1, -1, 0, "%s", err.c_str());
        auto* t = new NcclTransport();
        c->tr = t;
        t->key.assign(static_cast<const char*>(nccl_id), SWE_NCCL_ID_BYTES);
        t->key += ":" + std::to_string(ex.rank) + "/" + std::to_string(ex.nranks) + "@" + std::to_string(ex.device);
        std::lock_guard<std::mutex> lk(g_comms_m);
        CommEntry& e = g_comms[t->key];
        if (!e.comm) {
            ncclUniqueId id;
            std::memcpy(&id, nccl_id, sizeof id);
            const ncclResult_t r = g_nccl.CommInitRank(&e.comm, ex.nranks, id, ex.rank);
            if (r != ncclSuccess) {
                g_comms.erase(t->key);
                t->key.clear();
                return set_status(st, SWE_ERR_RUNTIME, -1, -1, 0.0, "NCCL error %d in ncclCommInitRank",
                                  static_cast<int>(r));
            }
            char bus[32] = "?";
            cudaDeviceGetPCIBusId(bus, sizeof bus, ex.device);
            std::fprintf(stderr, "swe-b200: NCCL communicator rank %d of %d on device %d (PCI %s) initialised\n",
                         ex.rank, ex.nranks, ex.device, bus);
        }
        ++e.refs;
        t->comm = e.comm;
    }
    return SWE_OK;
}

int nccl_unique_id(void* out, swe_status* st) {
    std::string err;
    if (!g_nccl.load(err)) return set_status(st, SWE_ERR_RUNTIME, -1, -1, 0, "%s", err.c_str());
    ncclUniqueId id;
    NCCL_TRY(g_nccl.GetUniqueId(&id));
    std::memcpy(out, &id, sizeof id);
    return ok_status(st);
}

}  // namespace swe_rt
