// Transports of the cross-GPU merge: NCCL (run-time loaded) and the in-process hub.
// See sinet_comm.h.
#include "sinet_comm.h"

#include <dlfcn.h>

#include <condition_variable>
#include <cstring>
#include <mutex>
#include <vector>

#include "sinet.h"

namespace sinet {

// ------------------------------------------------------------------ NCCL
namespace {

// Minimal declarations of the NCCL 2.x C API (values from nccl.h 2.28).
typedef struct ncclComm* ncclComm_t;
typedef struct { char internal[128]; } ncclUniqueId;
typedef int ncclResult_t;
constexpr int kNcclSum = 0;
constexpr int kNcclUint32 = 3;
constexpr int kNcclUint64 = 5;

struct NcclApi {
    bool loaded = false;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*ReduceScatter)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

std::mutex g_nccl_mu;

NcclApi* nccl_api(std::string* err) {
    static NcclApi api;
    std::lock_guard<std::mutex> lk(g_nccl_mu);
    if (api.loaded) return &api;
    // prefer the libnccl.so.2 already mapped into the process (torch's), else load by name
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) { *err = std::string("cannot load libnccl.so.2: ") + dlerror(); return nullptr; }
#define SINET_SYM(field, name) \
    api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, name)); \
    if (!api.field) { *err = std::string("libnccl.so.2 lacks ") + name; return nullptr; }
    SINET_SYM(GetUniqueId, "ncclGetUniqueId")
    SINET_SYM(CommInitRank, "ncclCommInitRank")
    SINET_SYM(CommDestroy, "ncclCommDestroy")
    SINET_SYM(ReduceScatter, "ncclReduceScatter")
    SINET_SYM(AllReduce, "ncclAllReduce")
    SINET_SYM(AllGather, "ncclAllGather")
    SINET_SYM(Send, "ncclSend")
    SINET_SYM(Recv, "ncclRecv")
    SINET_SYM(GroupStart, "ncclGroupStart")
    SINET_SYM(GroupEnd, "ncclGroupEnd")
    SINET_SYM(GetErrorString, "ncclGetErrorString")
#undef SINET_SYM
    api.loaded = true;
    return &api;
}

class NcclTransport final : public Transport {
public:
    NcclTransport(NcclApi* api, ncclComm_t comm) : api_(api), comm_(comm) {}
    ~NcclTransport() override { if (comm_) api_->CommDestroy(comm_); }
    const char* name() const override { return "nccl"; }
    int all_gather_u32(const uint32_t* send, uint32_t* recv, size_t count, cudaStream_t st, std::string* err) override {
        return ck(api_->AllGather(send, recv, count, kNcclUint32, comm_, st), "ncclAllGather", err);
    }
    int group_start(std::string* err) override { return ck(api_->GroupStart(), "ncclGroupStart", err); }
    int send_u64(const unsigned long long* buf, size_t count, int peer, cudaStream_t st, std::string* err) override {
        return ck(api_->Send(buf, count, kNcclUint64, peer, comm_, st), "ncclSend", err);
    }
    int recv_u64(unsigned long long* buf, size_t count, int peer, cudaStream_t st, std::string* err) override {
        return ck(api_->Recv(buf, count, kNcclUint64, peer, comm_, st), "ncclRecv", err);
    }
    int group_end(cudaStream_t, std::string* err) override { return ck(api_->GroupEnd(), "ncclGroupEnd", err); }
    int reduce_scatter_u64(const unsigned long long* send, unsigned long long* recv, size_t recvcount, cudaStream_t st,
                           std::string* err) override {
        return ck(api_->ReduceScatter(send, recv, recvcount, kNcclUint64, kNcclSum, comm_, st), "ncclReduceScatter", err);
    }
    int all_reduce_u64(const unsigned long long* send, unsigned long long* recv, size_t count, unsigned long long*,
                       cudaStream_t st, std::string* err) override {
        return ck(api_->AllReduce(send, recv, count, kNcclUint64, kNcclSum, comm_, st), "ncclAllReduce", err);
    }

private:
    int ck(ncclResult_t r, const char* what, std::string* err) {
        if (r == 0) return SINET_OK;
        *err = std::string(what) + ": " + api_->GetErrorString(r);
        return SINET_E_NCCL;
    }
    NcclApi* api_;
    ncclComm_t comm_;
};

}  // namespace

int nccl_unique_id(void* out128, std::string* err) {
    NcclApi* api = nccl_api(err);
    if (!api) return SINET_E_NCCL;
    ncclUniqueId id;
    if (api->GetUniqueId(&id) != 0) { *err = "ncclGetUniqueId failed"; return SINET_E_NCCL; }
    std::memcpy(out128, &id, sizeof id);
    return SINET_OK;
}

std::unique_ptr<Transport> make_nccl_transport(int world, int rank, const void* uid, std::string* err) {
    NcclApi* api = nccl_api(err);
    if (!api) return nullptr;
    ncclUniqueId id;
    std::memcpy(&id, uid, sizeof id);
    ncclComm_t comm = nullptr;
    ncclResult_t r = api->CommInitRank(&comm, world, id, rank);
    if (r != 0) { *err = std::string("ncclCommInitRank: ") + api->GetErrorString(r); return nullptr; }
    return std::unique_ptr<Transport>(new NcclTransport(api, comm));
}

}  // namespace sinet

// ------------------------------------------------------------------ in-process hub
// A rendezvous of `world` ranks that live in one process (one host thread per GPU).
// Host side: a generation barrier.  Device side: every collective posts this rank's buffer and
// a "ready" event (recorded on its stream), meets the others at barrier 1, makes its stream wait
// for the peers' ready events and moves / reduces the data, records "done", meets them at
// barrier 2 and makes its stream wait for every peer's "done" (so no peer is still reading its
// buffers when its stream moves on, as with NCCL).  Events alternate between two sets by
// collective parity: a peer may record the next collective's events before this rank has
// issued its waits on the previous ones, never two collectives ahead (barrier 1 of the next
// collective orders that).
struct sinet_hub {
    struct P2P { int peer; const unsigned long long* ptr; size_t count; };
    struct Slot {
        bool attached = false;
        int device = -1;
        const void* ptr = nullptr;
        size_t count = 0;
        cudaEvent_t ready[2] = {nullptr, nullptr};
        cudaEvent_t done[2] = {nullptr, nullptr};
        std::vector<P2P> sends;
    };
    explicit sinet_hub(int w) : world(w), slot((size_t)w) {}
    int world;
    int refs = 1;          // the creator's reference + one per attached rank (freed at zero)
    std::mutex mu;
    std::condition_variable cv;
    uint64_t generation = 0;
    int arrived = 0;
    std::vector<Slot> slot;

    void barrier() {
        std::unique_lock<std::mutex> lk(mu);
        const uint64_t g = generation;
        if (++arrived == world) {
            arrived = 0;
            ++generation;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return generation != g; });
        }
    }
};

namespace sinet {

int hub_world(const sinet_hub* hub) { return hub ? hub->world : 0; }

namespace {

class HubTransport final : public Transport {
public:
    HubTransport(sinet_hub* hub, int rank, int device) : hub_(hub), rank_(rank), device_(device) {}
    ~HubTransport() override {
        auto& s = hub_->slot[(size_t)rank_];
        for (int k = 0; k < 2; ++k) {
            if (s.ready[k]) cudaEventDestroy(s.ready[k]);
            if (s.done[k]) cudaEventDestroy(s.done[k]);
            s.ready[k] = s.done[k] = nullptr;
        }
        bool last;
        {
            std::lock_guard<std::mutex> lk(hub_->mu);
            s.attached = false;
            last = --hub_->refs == 0;
        }
        if (last) delete hub_;   // sinet_hub_destroy ran first: the last rank frees the hub
    }
    int init(std::string* err) {
        auto& s = hub_->slot[(size_t)rank_];
        for (int k = 0; k < 2; ++k) {
            if (cudaEventCreateWithFlags(&s.ready[k], cudaEventDisableTiming) != cudaSuccess ||
                cudaEventCreateWithFlags(&s.done[k], cudaEventDisableTiming) != cudaSuccess) {
                *err = "hub: cudaEventCreate failed";
                return SINET_E_CUDA;
            }
        }
        s.device = device_;
        return SINET_OK;
    }
    const char* name() const override { return "hub"; }

    int all_gather_u32(const uint32_t* send, uint32_t* recv, size_t count, cudaStream_t st, std::string* err) override {
        int rc = post(send, count, st, err);
        if (rc) return rc;
        for (int r = 0; r < hub_->world && !rc; ++r) {
            const auto& s = hub_->slot[(size_t)r];
            if (r != rank_) rc = cu(cudaStreamWaitEvent(st, s.ready[par_], 0), err);
            if (!rc) rc = cu(cudaMemcpyAsync(recv + (size_t)r * count, s.ptr, count * 4u, cudaMemcpyDefault, st), err);
        }
        return finish(rc, st, err);
    }
    int group_start(std::string*) override {
        in_group_ = true;
        recvs_.clear();
        hub_->slot[(size_t)rank_].sends.clear();
        return SINET_OK;
    }
    int send_u64(const unsigned long long* buf, size_t count, int peer, cudaStream_t, std::string* err) override {
        if (!in_group_ || peer < 0 || peer >= hub_->world) { *err = "hub: send outside a group or bad peer"; return SINET_E_INVAL; }
        hub_->slot[(size_t)rank_].sends.push_back({peer, buf, count});
        return SINET_OK;
    }
    int recv_u64(unsigned long long* buf, size_t count, int peer, cudaStream_t, std::string* err) override {
        if (!in_group_ || peer < 0 || peer >= hub_->world) { *err = "hub: recv outside a group or bad peer"; return SINET_E_INVAL; }
        recvs_.push_back({peer, buf, count});
        return SINET_OK;
    }
    int group_end(cudaStream_t st, std::string* err) override {
        in_group_ = false;
        int rc = post(nullptr, 0, st, err);
        if (rc) return rc;
        // the k-th recv from peer q matches q's k-th send to this rank
        std::vector<size_t> taken((size_t)hub_->world, 0);
        for (const auto& rv : recvs_) {
            const auto& s = hub_->slot[(size_t)rv.peer];
            size_t k = 0, want = taken[(size_t)rv.peer]++;
            const sinet_hub::P2P* m = nullptr;
            for (const auto& sd : s.sends)
                if (sd.peer == rank_ && k++ == want) { m = &sd; break; }
            if (!m || m->count != rv.count) {
                *err = "hub: unmatched or size-mismatched send/recv";
                rc = SINET_E_INVAL;
                break;
            }
            if (rv.peer != rank_) rc = cu(cudaStreamWaitEvent(st, s.ready[par_], 0), err);
            if (!rc) rc = cu(cudaMemcpyAsync(const_cast<unsigned long long*>(rv.ptr), m->ptr, rv.count * 8u,
                                             cudaMemcpyDefault, st), err);
            if (rc) break;
        }
        return finish(rc, st, err);
    }
    int reduce_scatter_u64(const unsigned long long* send, unsigned long long* recv, size_t recvcount, cudaStream_t st,
                           std::string* err) override {
        if (hub_->world > kMaxPeers) { *err = "hub: more than 64 ranks"; return SINET_E_INVAL; }
        int rc = post(send, recvcount, st, err);
        if (rc) return rc;
        PeerPtrs pp{};
        for (int r = 0; r < hub_->world && !rc; ++r) {
            const auto& s = hub_->slot[(size_t)r];
            if (r != rank_) {
                rc = cu(cudaStreamWaitEvent(st, s.ready[par_], 0), err);
                if (!rc && s.device != device_) rc = enable_peer(s.device, err);
            }
            pp.p[r] = static_cast<const unsigned long long*>(s.ptr) + (size_t)rank_ * recvcount;
        }
        if (!rc) rc = cu(launch_sum_peers(recv, pp, hub_->world, recvcount, sm_count(), st), err);
        return finish(rc, st, err);
    }
    int all_reduce_u64(const unsigned long long* send, unsigned long long* recv, size_t count,
                       unsigned long long* scratch, cudaStream_t st, std::string* err) override {
        if (!scratch) { *err = "hub: all-reduce needs scratch"; return SINET_E_INVAL; }
        // phase 1: gather every rank's vector (nobody writes until everyone has read)
        int rc = post(send, count, st, err);
        if (rc) return rc;
        for (int r = 0; r < hub_->world && !rc; ++r) {
            const auto& s = hub_->slot[(size_t)r];
            if (r != rank_) rc = cu(cudaStreamWaitEvent(st, s.ready[par_], 0), err);
            if (!rc) rc = cu(cudaMemcpyAsync(scratch + (size_t)r * count, s.ptr, count * 8u, cudaMemcpyDefault, st), err);
        }
        rc = finish(rc, st, err);
        if (rc) return rc;
        // phase 2: sum the gathered rows locally
        PeerPtrs pp{};
        for (int r = 0; r < hub_->world && r < kMaxPeers; ++r) pp.p[r] = scratch + (size_t)r * count;
        return cu(launch_sum_peers(recv, pp, hub_->world < kMaxPeers ? hub_->world : kMaxPeers, count, 1, st), err);
    }

private:
    static int cu(cudaError_t e, std::string* err) {
        if (e == cudaSuccess) return SINET_OK;
        *err = std::string("hub: ") + cudaGetErrorString(e);
        return SINET_E_CUDA;
    }
    int sm_count() {
        int n = 0;
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device_);
        return n > 0 ? n : 1;
    }
    int enable_peer(int dev, std::string* err) {
        int can = 0;
        cudaDeviceCanAccessPeer(&can, device_, dev);
        if (!can) { *err = "hub: no peer access between the ranks' devices"; return SINET_E_CUDA; }
        cudaError_t e = cudaDeviceEnablePeerAccess(dev, 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled) { cudaGetLastError(); return SINET_OK; }
        return cu(e, err);
    }
    // publish this rank's buffer and its ready event, then meet the peers (barrier 1)
    int post(const void* ptr, size_t count, cudaStream_t st, std::string* err) {
        par_ ^= 1;
        auto& s = hub_->slot[(size_t)rank_];
        s.ptr = ptr;
        s.count = count;
        int rc = cu(cudaEventRecord(s.ready[par_], st), err);
        hub_->barrier();   // always: a failing rank must not strand its peers
        return rc;
    }
    // record done, meet the peers (barrier 2), wait for every peer's done
    int finish(int rc, cudaStream_t st, std::string* err) {
        auto& s = hub_->slot[(size_t)rank_];
        int rc2 = cu(cudaEventRecord(s.done[par_], st), err);
        hub_->barrier();
        if (rc) return rc;
        if (rc2) return rc2;
        for (int r = 0; r < hub_->world; ++r)
            if (r != rank_) {
                int w = cu(cudaStreamWaitEvent(st, hub_->slot[(size_t)r].done[par_], 0), err);
                if (w) return w;
            }
        return SINET_OK;
    }

    sinet_hub* hub_;
    int rank_, device_;
    int par_ = 0;
    bool in_group_ = false;
    std::vector<sinet_hub::P2P> recvs_;
};

}  // namespace

std::unique_ptr<Transport> make_hub_transport(sinet_hub* hub, int rank, int device, std::string* err) {
    if (!hub || rank < 0 || rank >= hub->world) { *err = "hub: bad hub or rank"; return nullptr; }
    {
        std::lock_guard<std::mutex> lk(hub->mu);
        if (hub->slot[(size_t)rank].attached) { *err = "hub: rank already attached"; return nullptr; }
        hub->slot[(size_t)rank].attached = true;
        ++hub->refs;
    }
    std::unique_ptr<HubTransport> t(new HubTransport(hub, rank, device));
    if (t->init(err) != SINET_OK) return nullptr;
    return std::unique_ptr<Transport>(t.release());
}

}  // namespace sinet

extern "C" {

int sinet_hub_create(sinet_hub** out, int32_t world) {
    if (!out || world < 1 || world > sinet::kMaxPeers) return SINET_E_INVAL;
    *out = new (std::nothrow) sinet_hub(world);
    return *out ? SINET_OK : SINET_E_INVAL;
}

void sinet_hub_destroy(sinet_hub* hub) {
    if (!hub) return;
    bool last;
    {
        std::lock_guard<std::mutex> lk(hub->mu);
        last = --hub->refs == 0;
    }
    if (last) delete hub;   // else the last attached ctx frees it when it closes
}

}  // extern "C"
