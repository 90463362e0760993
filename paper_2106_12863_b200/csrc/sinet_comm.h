// Transports of the cross-GPU merge (merge-scatter P:L216-222).
//
// sinet_reduce() is written once against this interface.  Two implementations:
//   * NCCL (one process per GPU, torchrun ranks): the NCCL C API loaded at run time;
//   * HUB  (one process, one host thread per GPU -- the paper's own layout: "we assign
//     one thread for each GPU"): ranks rendezvous on a host barrier, device order
//     is kept with CUDA events, data moves by peer copies (cudaMemcpyAsync over UVA) and
//     the dense reduce-scatter is one kernel per owner that reads its slice from every
//     peer's bins directly (NVLink P2P loads across GPUs; plain loads on one GPU).
// Every call enqueues on `st` and returns SINET_OK or a SINET_E_* code with *err set.
// Semantics follow NCCL: when `st` passes a call, its data movement is complete on every
// rank that takes part (peers have finished reading this rank's send buffers).
#pragma once
#include <cstddef>
#include <cstdint>
#include <memory>
#include <string>

#include <cuda_runtime.h>

struct sinet_hub;

namespace sinet {

class Transport {
public:
    virtual ~Transport() = default;
    virtual const char* name() const = 0;
    // recv[r * count + i] = send_r[i] for every rank r
    virtual int all_gather_u32(const uint32_t* send, uint32_t* recv, size_t count, cudaStream_t st,
                               std::string* err) = 0;
    // point-to-point, matched in call order per (sender, receiver) pair; only between group_start / group_end
    virtual int group_start(std::string* err) = 0;
    virtual int send_u64(const unsigned long long* buf, size_t count, int peer, cudaStream_t st, std::string* err) = 0;
    virtual int recv_u64(unsigned long long* buf, size_t count, int peer, cudaStream_t st, std::string* err) = 0;
    virtual int group_end(cudaStream_t st, std::string* err) = 0;
    // recv[i] = sum over ranks r of send_r[rank * recvcount + i]  (u64, mod 2^64; recv may alias)
    virtual int reduce_scatter_u64(const unsigned long long* send, unsigned long long* recv, size_t recvcount,
                                   cudaStream_t st, std::string* err) = 0;
    // recv[i] = sum over ranks of send_r[i]; scratch: world * count u64 of device memory (HUB only)
    virtual int all_reduce_u64(const unsigned long long* send, unsigned long long* recv, size_t count,
                               unsigned long long* scratch, cudaStream_t st, std::string* err) = 0;
};

// NCCL transport over the libnccl.so.2 already loaded in the process (else loaded by name).
std::unique_ptr<Transport> make_nccl_transport(int world, int rank, const void* unique_id128, std::string* err);
int nccl_unique_id(void* out128, std::string* err);

// In-process transport: rank `rank` of `hub`, whose ctx lives on CUDA device `device`.
std::unique_ptr<Transport> make_hub_transport(sinet_hub* hub, int rank, int device, std::string* err);
int hub_world(const sinet_hub* hub);

// merge kernels (sinet_merge.cu)
constexpr int kMaxPeers = 64;
struct PeerPtrs { const unsigned long long* p[kMaxPeers]; };
cudaError_t launch_add_bins(unsigned long long* bins, const unsigned long long* in, uint64_t first, uint64_t n,
                            int sm_count, cudaStream_t st);
// dst[i] = sum_{r < npeers} src.p[r][i] for i < n (u64)
cudaError_t launch_sum_peers(unsigned long long* dst, const PeerPtrs& src, int npeers, uint64_t n, int sm_count,
                             cudaStream_t st);

}  // namespace sinet
