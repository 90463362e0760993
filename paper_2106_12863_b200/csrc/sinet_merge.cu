// Merge kernels of the cross-GPU combine: the paper merges the per-GPU
// <timestamp,count> / <timestamp,bytes> partials with "associative and commutative
// operators" (merge-scatter).  Bins are u64 sums, so merging is addition.
#include "sinet_comm.h"
#include "sinet_params.h"

namespace sinet {

namespace {

int grid_for(uint64_t n_vec, int sm_count) {
    const uint64_t blocks = (n_vec + 255u) / 256u;
    const uint64_t cap = (uint64_t)(sm_count > 0 ? sm_count : 1) * 8u;
    return (int)(blocks < cap ? (blocks ? blocks : 1) : cap);
}

}  // namespace

// Sparse exchange: owned bins [first, first+n) += received partial bins (staging).
__global__ void __launch_bounds__(256) k_add_bins(unsigned long long* bins, const unsigned long long* in,
                                                  uint64_t first, uint64_t n) {
    const uint64_t total = n * 4u;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x)
        bins[first * 4u + i] += in[i];
}

cudaError_t launch_add_bins(unsigned long long* bins, const unsigned long long* in, uint64_t first, uint64_t n,
                            int sm_count, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    k_add_bins<<<grid_for(n * 4u, sm_count), 256, 0, st>>>(bins, in, first, n);
    return cudaGetLastError();
}

// Dense reduce-scatter over peer memory (in-process transport): the owner reads its slice
// from every rank's partial bins -- NVLink loads when the ranks are different GPUs -- and
// writes the sum once.  128-bit streaming loads; dst may alias one of the sources (each
// element is read by the thread that writes it).
__global__ void __launch_bounds__(256) k_sum_peers(unsigned long long* dst, PeerPtrs src, int npeers, uint64_t n) {
    const uint64_t nv = n / 2u;
    ulonglong2* d2 = reinterpret_cast<ulonglong2*>(dst);
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += (uint64_t)gridDim.x * blockDim.x) {
        unsigned long long a = 0ull, b = 0ull;
        for (int r = 0; r < npeers; ++r) {
            const ulonglong2 v = __ldcs(reinterpret_cast<const ulonglong2*>(src.p[r]) + i);
            a += v.x;
            b += v.y;
        }
        d2[i] = make_ulonglong2(a, b);
    }
    if ((n & 1u) && blockIdx.x == 0 && threadIdx.x == 0) {
        unsigned long long a = 0ull;
        for (int r = 0; r < npeers; ++r) a += src.p[r][n - 1];
        dst[n - 1] = a;
    }
}

cudaError_t launch_sum_peers(unsigned long long* dst, const PeerPtrs& src, int npeers, uint64_t n, int sm_count,
                             cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    k_sum_peers<<<grid_for(n / 2u + 1u, sm_count), 256, 0, st>>>(dst, src, npeers, n);
    return cudaGetLastError();
}

}  // namespace sinet
