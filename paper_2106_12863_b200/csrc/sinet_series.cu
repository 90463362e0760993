// NEXT-1 of SURVEY §8(f): series read-out on the device.
//   * re-binning of the ms bins to coarser frames -- "Session data is grouped
//     into one-hour frame bins", counts "in 10 minutes";
//   * sparse export of the nonzero bins of one direction as (bin start ms,
//     count, bytes) -- the paper's key/value namespaces X1<timestamp>,
//     X1<count>, X2<timestamp>, X2<bytes>.
// Both read the bins once (32 B/bin: all four planes share a sector, so the
// rebin kernel reduces all of them in the same pass).
#include "sinet_device.cuh"
#include "sinet_kernels.h"

namespace sinet {

// One thread reduces kRun consecutive bins, then a warp-segmented inclusive
// scan over ascending coarse keys; the last lane of each segment adds its
// four u64 sums to the (zeroed) output with RED.ADD.64.
constexpr int kRun = 4;

__global__ void __launch_bounds__(256) k_rebin(const ulonglong2* __restrict__ bins, uint64_t lo, uint64_t hi,
                                               uint64_t factor, unsigned long long* out) {
    const uint64_t nb = hi - lo;
    const uint64_t nthreads_needed = (nb + kRun - 1) / kRun;
    const uint32_t lane = threadIdx.x & 31u;
    for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x; base < nthreads_needed;
         base += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t t = base + threadIdx.x;
        unsigned long long v[4] = {0ull, 0ull, 0ull, 0ull};
        uint64_t key = ~0ull;
        const uint64_t b0 = t * kRun;
#pragma unroll
        for (int r = 0; r < kRun; ++r) {
            const uint64_t i = b0 + r;
            if (t < nthreads_needed && i < nb) {
                const uint64_t k = (lo + i) / factor - lo / factor;   // absolute frame, from the first one met
                if (key != ~0ull && k != key) {   // coarse boundary inside this thread's run
                    for (int m = 0; m < 4; ++m) if (v[m]) atomicAdd(out + key * 4 + m, v[m]);
                    v[0] = v[1] = v[2] = v[3] = 0ull;
                }
                key = k;
                const ulonglong2 a = __ldcs(bins + (lo + i) * 2);
                const ulonglong2 c = __ldcs(bins + (lo + i) * 2 + 1);
                v[0] += a.x; v[1] += a.y; v[2] += c.x; v[3] += c.y;
            }
        }
        // warp-segmented inclusive scan (keys ascend with the lane index)
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const uint64_t ku = __shfl_up_sync(kFull, key, off);
            unsigned long long vu[4];
#pragma unroll
            for (int m = 0; m < 4; ++m) vu[m] = __shfl_up_sync(kFull, v[m], off);
            if (lane >= (uint32_t)off && ku == key && key != ~0ull)
                for (int m = 0; m < 4; ++m) v[m] += vu[m];
        }
        const uint64_t kd = __shfl_down_sync(kFull, key, 1);
        const bool tail = key != ~0ull && (lane == 31u || kd != key);
        if (tail)
            for (int m = 0; m < 4; ++m) if (v[m]) atomicAdd(out + key * 4 + m, v[m]);
    }
}

// Sparse export, pass 1: nonzero-count bins of one direction per 8192-bin block.
constexpr uint32_t kSparseBlock = 8192;

__global__ void __launch_bounds__(256) k_sparse_count(const unsigned long long* __restrict__ bins, uint64_t lo,
                                                      uint64_t hi, uint32_t dir, uint32_t* counts) {
    __shared__ uint32_t s;
    if (threadIdx.x == 0) s = 0;
    __syncthreads();
    const uint64_t b0 = lo + (uint64_t)blockIdx.x * kSparseBlock;
    uint32_t c = 0;
    for (uint32_t i = threadIdx.x; i < kSparseBlock; i += blockDim.x) {
        const uint64_t b = b0 + i;
        if (b < hi && __ldg(bins + b * 4 + dir * 2) != 0ull) ++c;
    }
    c = __reduce_add_sync(kFull, c);
    if ((threadIdx.x & 31u) == 0 && c) atomicAdd(&s, c);
    __syncthreads();
    if (threadIdx.x == 0) counts[blockIdx.x] = s;
}

// Pass 2: exclusive scan of the block counts (one block; nblk is small) and the total.
__global__ void __launch_bounds__(1024) k_sparse_scan(uint32_t* counts, uint32_t nblk, unsigned long long* total) {
    __shared__ unsigned long long s_carry;
    __shared__ unsigned long long s_warp[32];
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    for (uint32_t base = 0; base < nblk; base += blockDim.x) {
        const uint32_t i = base + threadIdx.x;
        const unsigned long long v = (i < nblk) ? counts[i] : 0ull;
        unsigned long long x = v;   // inclusive warp scan
        for (int off = 1; off < 32; off <<= 1) {
            const unsigned long long y = __shfl_up_sync(kFull, x, off);
            if (lane >= (uint32_t)off) x += y;
        }
        if (lane == 31u) s_warp[warp] = x;
        __syncthreads();
        if (warp == 0) {
            unsigned long long w = (lane < (blockDim.x >> 5)) ? s_warp[lane] : 0ull;
            for (int off = 1; off < 32; off <<= 1) {
                const unsigned long long y = __shfl_up_sync(kFull, w, off);
                if (lane >= (uint32_t)off) w += y;
            }
            s_warp[lane] = w;   // inclusive over warps
        }
        __syncthreads();
        const unsigned long long before = s_carry + (warp ? s_warp[warp - 1] : 0ull) + x - v;
        if (i < nblk) counts[i] = (uint32_t)before;   // exclusive offset (< 2^32 entries per export)
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) s_carry += s_warp[(blockDim.x >> 5) - 1];
        __syncthreads();
    }
    if (threadIdx.x == 0) *total = s_carry;
}

// Pass 3: ordered scatter of (start + bin*w, count, bytes) of every nonzero-count bin.
__global__ void __launch_bounds__(256) k_sparse_write(const unsigned long long* __restrict__ bins, uint64_t lo,
                                                      uint64_t hi, uint32_t dir, const uint32_t* offsets,
                                                      uint64_t start, uint32_t width, unsigned long long* o_ts,
                                                      unsigned long long* o_cnt, unsigned long long* o_bytes,
                                                      uint64_t capacity) {
    __shared__ uint32_t s_warp[8];
    __shared__ uint32_t s_base;
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_base = offsets[blockIdx.x];
    const uint64_t b0 = lo + (uint64_t)blockIdx.x * kSparseBlock;
    for (uint32_t step = 0; step < kSparseBlock; step += blockDim.x) {
        const uint64_t b = b0 + step + threadIdx.x;
        unsigned long long c = 0;
        if (b < hi) c = __ldg(bins + b * 4 + dir * 2);
        const bool nz = c != 0ull;
        const unsigned m = __ballot_sync(kFull, nz);
        if (lane == 0) s_warp[warp] = __popc(m);
        __syncthreads();
        uint32_t before = s_base;
        for (uint32_t w = 0; w < warp; ++w) before += s_warp[w];
        before += __popc(m & ((1u << lane) - 1u));
        if (nz && before < capacity) {
            o_ts[before] = start + b * (uint64_t)width;
            o_cnt[before] = c;
            o_bytes[before] = __ldg(bins + b * 4 + dir * 2 + 1);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t add = 0;
            for (uint32_t w = 0; w < (blockDim.x >> 5); ++w) add += s_warp[w];
            s_base += add;
        }
        __syncthreads();
    }
}

cudaError_t launch_rebin(const unsigned long long* bins, uint64_t lo, uint64_t hi, uint64_t factor,
                         unsigned long long* out, uint64_t n_out, int sm_count, cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(out, 0, n_out * 32u, st);
    if (e != cudaSuccess || hi <= lo) return e;
    const uint64_t threads = (hi - lo + kRun - 1) / kRun;
    uint64_t blocks = (threads + 255) / 256;
    const uint64_t cap = (uint64_t)sm_count * 8u;
    k_rebin<<<(int)(blocks < cap ? blocks : cap), 256, 0, st>>>(reinterpret_cast<const ulonglong2*>(bins), lo, hi,
                                                               factor, out);
    return cudaGetLastError();
}

uint32_t sparse_blocks(uint64_t nbins) { return (uint32_t)((nbins + kSparseBlock - 1) / kSparseBlock); }

cudaError_t launch_sparse(const unsigned long long* bins, uint64_t lo, uint64_t hi, uint32_t dir, uint32_t* scratch,
                          unsigned long long* d_total, uint64_t start, uint32_t width, unsigned long long* o_ts,
                          unsigned long long* o_cnt, unsigned long long* o_bytes, uint64_t capacity,
                          cudaStream_t st) {
    const uint32_t nblk = sparse_blocks(hi - lo);
    if (nblk == 0) return cudaMemsetAsync(d_total, 0, 8, st);
    k_sparse_count<<<nblk, 256, 0, st>>>(bins, lo, hi, dir, scratch);
    k_sparse_scan<<<1, 1024, 0, st>>>(scratch, nblk, d_total);
    if (capacity)
        k_sparse_write<<<nblk, 256, 0, st>>>(bins, lo, hi, dir, scratch, start, width, o_ts, o_cnt, o_bytes, capacity);
    return cudaGetLastError();
}

}  // namespace sinet
