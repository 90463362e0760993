// NEXT-4 comparator: the paper's own histogram design on B200.
//
// The paper discriminates with a Thrust transform and histograms with
// "pairwise reduction" over key/value pairs (<timestamp,count>,
// <timestamp,bytes>), i.e. sort by key + reduce_by_key, then merges the
// per-GPU partials.  This file reproduces that pipeline with CUB
// so the bench can time it on the same box and the same input as the fused
// kernels.  It produces bit-identical bins (parity-tested).
//   1. k_map_keys: classify + map every record to key = bin*2+dir (sentinel
//      2B for records not binned), value = bytes; side totals as usual.
//   2. cub::DeviceRadixSort::SortPairs on the key bits that are used.
//   3. cub::DeviceReduce::ReduceByKey (bytes) + DeviceRunLengthEncode::Encode (counts).
//   4. k_scatter_runs: add each run into its (bin, dir) (keys unique: no races).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_run_length_encode.cuh>

#include "sinet_device.cuh"
#include "sinet_kernels.h"

namespace sinet {

template <bool kSmall>
__global__ void __launch_bounds__(256) k_map_keys(KernelParams p, uint32_t sentinel, uint32_t* keys,
                                                  unsigned long long* vals) {
    extern __shared__ __align__(16) uint32_t smem[];
    __shared__ unsigned long long s_tot[32 * 12];
    const Table T = stage_table<kSmall>(p, smem);
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t wpb = blockDim.x >> 5;
    const uint64_t gw = (uint64_t)blockIdx.x * wpb + (threadIdx.x >> 5);
    const uint64_t stride = (uint64_t)gridDim.x * wpb * 128ull;
    WarpTotals tot;
    tot.zero();
    uint32_t tmin = 0xFFFFFFFFu, tmax = 0u;
    for (uint64_t wbase = gw * 128ull; wbase < p.nv; wbase += stride) {
        const uint64_t base = wbase + lane * 4ull;
        Rec4 r;
        load4(p, base, r);
        uint32_t addr[8], in8[8];
#pragma unroll
        for (int j = 0; j < 4; ++j) { addr[2 * j] = r.src[j]; addr[2 * j + 1] = r.dst[j]; }
        member_batch<8>(addr, in8, T);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const bool inrange = vvalid(p, base + j);
            const bool valid = inrange && watch_pass(r.src[j], r.dst[j], p);
            const uint32_t s_in = in8[2 * j];
            const uint32_t d_in = in8[2 * j + 1];
            const uint32_t cell = s_in * 2u + d_in;
            const uint32_t dir = (p.lut >> (cell * 2u)) & 3u;
            uint32_t bin = 0;
            const bool inw = map_bin(r.ts[j], p, bin);
            const bool directed = valid && dir < 2u;
            if (directed && inw) { tmin = min(tmin, bin); tmax = max(tmax, bin); }
            if (inrange) {   // every record gets a key: filtered or unbinned ones the sentinel
                const uint64_t a = base + j - p.head;
                keys[a] = (directed && inw) ? bin * 2u + dir : sentinel;
                vals[a] = r.by[j];
            }
            tot.add(valid, cell, directed && !inw, dir, r.by[j]);
        }
    }
    note_touched_warp(p, tmin, tmax);
    flush_totals(tot, p.totals, s_tot);
}

__global__ void __launch_bounds__(256) k_scatter_runs(const uint32_t* keys, const uint32_t* counts,
                                                      const unsigned long long* sums, const int* num_runs,
                                                      uint32_t sentinel, unsigned long long* bins) {
    const int n = *num_runs;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint32_t k = keys[i];
        if (k == sentinel) continue;
        unsigned long long* slot = bins + (size_t)(k >> 1) * 4u + (k & 1u) * 2u;
        slot[0] += counts[i];
        slot[1] += sums[i];
    }
}

namespace {
struct SrLayout {
    size_t keys_in, keys_out, vals_in, vals_out, uniq, sums, counts, nruns, temp, total;
};

size_t au(size_t x) { return (x + 255) / 256 * 256; }

SrLayout sr_layout(uint64_t n, size_t temp_bytes) {
    SrLayout L{};
    size_t off = 0;
    L.keys_in = off;  off += au(n * 4);
    L.keys_out = off; off += au(n * 4);
    L.vals_in = off;  off += au(n * 8);
    L.vals_out = off; off += au(n * 8);
    L.uniq = off;     off += au(n * 4);
    L.sums = off;     off += au(n * 8);
    L.counts = off;   off += au(n * 4);
    L.nruns = off;    off += 256;
    L.temp = off;     off += au(temp_bytes);
    L.total = off;
    return L;
}

size_t cub_temp_bytes(uint64_t n, int end_bit) {
    size_t a = 0, b = 0, c = 0;
    const int ni = (int)n;
    cub::DeviceRadixSort::SortPairs(nullptr, a, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                    (unsigned long long*)nullptr, (unsigned long long*)nullptr, ni, 0, end_bit);
    cub::DeviceReduce::ReduceByKey(nullptr, b, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                   (unsigned long long*)nullptr, (unsigned long long*)nullptr, (int*)nullptr,
                                   cuda::std::plus<unsigned long long>{}, ni);
    cub::DeviceRunLengthEncode::Encode(nullptr, c, (uint32_t*)nullptr, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                       (int*)nullptr, ni);
    size_t m = a > b ? a : b;
    return m > c ? m : c;
}

int key_bits(uint64_t nbins) {
    uint64_t s = nbins * 2;   // sentinel
    int b = 1;
    while ((s >> b) != 0) ++b;
    return b;
}
}  // namespace

size_t sortreduce_scratch_bytes(uint64_t n, uint64_t nbins) {
    if (n == 0) return 0;
    return sr_layout(n, cub_temp_bytes(n, key_bits(nbins))).total;
}

cudaError_t launch_sortreduce(const KernelParams& p, void* scratch, size_t scratch_bytes, int sm_count,
                              cudaStream_t st, int* launches) {
    const uint64_t n = p.n;
    const int eb = key_bits(p.nbins);
    const uint32_t sentinel = p.nbins * 2u;
    const size_t tb = cub_temp_bytes(n, eb);
    SrLayout L = sr_layout(n, tb);
    if (scratch_bytes < L.total) return cudaErrorInvalidValue;
    unsigned char* s = static_cast<unsigned char*>(scratch);
    uint32_t* keys_in = reinterpret_cast<uint32_t*>(s + L.keys_in);
    uint32_t* keys_out = reinterpret_cast<uint32_t*>(s + L.keys_out);
    unsigned long long* vals_in = reinterpret_cast<unsigned long long*>(s + L.vals_in);
    unsigned long long* vals_out = reinterpret_cast<unsigned long long*>(s + L.vals_out);
    uint32_t* uniq = reinterpret_cast<uint32_t*>(s + L.uniq);
    unsigned long long* sums = reinterpret_cast<unsigned long long*>(s + L.sums);
    uint32_t* counts = reinterpret_cast<uint32_t*>(s + L.counts);
    int* nruns = reinterpret_cast<int*>(s + L.nruns);
    void* temp = s + L.temp;
    const size_t smem = table_smem_bytes(p.nbnd, p.n_mixed, p.small);
    cudaError_t e = p.small ? cudaFuncSetAttribute(k_map_keys<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)
                            : cudaFuncSetAttribute(k_map_keys<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    if (p.small) k_map_keys<true><<<sm_count * 4, 256, smem, st>>>(p, sentinel, keys_in, vals_in);
    else k_map_keys<false><<<sm_count * 4, 256, smem, st>>>(p, sentinel, keys_in, vals_in);
    size_t t = tb;
    const int ni = (int)n;
    if ((e = cub::DeviceRadixSort::SortPairs(temp, t, keys_in, keys_out, vals_in, vals_out, ni, 0, eb, st))) return e;
    t = tb;
    if ((e = cub::DeviceReduce::ReduceByKey(temp, t, keys_out, uniq, vals_out, sums, nruns,
                                            cuda::std::plus<unsigned long long>{}, ni, st))) return e;
    t = tb;
    // run lengths = <timestamp,count>; unique keys written again into keys_in (same order)
    if ((e = cub::DeviceRunLengthEncode::Encode(temp, t, keys_out, keys_in, counts, nruns, ni, st))) return e;
    k_scatter_runs<<<sm_count * 8, 256, 0, st>>>(uniq, counts, sums, nruns, sentinel, p.bins);
    *launches = 5;   // map, sort (>=1), reduce-by-key, run-length-encode, scatter (CUB adds internal launches)
    return cudaGetLastError();
}

}  // namespace sinet
