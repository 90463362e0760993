// sinet kernels for sm_100a: bin materialisation and the L2-atomic histogram path.
//
// The fused kernel does SURVEY §8 rows a2-a7 in one pass over the records:
// 128-bit streaming loads of the four Table 1 columns (a2), membership of
// src and dst (a3, a4; Alg. 1 l.6-9), the direction LUT (a4),
// Map to a millisecond bin (a5), Reduce by u64 addition
// into the bins (a6) and the side totals (a7).
#include "sinet_device.cuh"
#include "sinet_kernels.h"

namespace sinet {

// Zero-fill every tile whose state word is not "initialised in this epoch"
// and mark it initialised.  One warp per 32 tiles: the state words are read
// coalesced, so a pass over an all-initialised histogram costs ~n_tiles*4 B.
__global__ void __launch_bounds__(256) k_materialize(ulonglong2* bins, uint32_t* flags,
                                                     uint32_t n_tiles, uint32_t init_word) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t base = gw * 32u; base < n_tiles; base += nw * 32u) {
        uint32_t t = base + lane;
        uint32_t f = (t < n_tiles) ? flags[t] : init_word;
        unsigned need = __ballot_sync(kFull, f != init_word);
        while (need) {
            int k = __ffs(need) - 1;
            need &= need - 1;
            uint32_t tile = base + (uint32_t)k;
            ulonglong2* b = bins + (size_t)tile * (kTileBins * 2u);
            const ulonglong2 z = make_ulonglong2(0ull, 0ull);
#pragma unroll 8
            for (uint32_t i = lane; i < kTileBins * 2u; i += 32u) b[i] = z;
            if (lane == (uint32_t)k) flags[tile] = init_word;
        }
    }
}

// Histogram by L2 atomics onto materialised bins: any record order.
// Persistent grid; each warp takes 128 consecutive records per step (4 per
// lane, vector loads), so the loop is warp-uniform and the totals can use
// warp ballots/reductions.
template <bool kSmall>
__global__ void __launch_bounds__(256) k_hist_atomic(KernelParams p) {
    extern __shared__ __align__(16) uint32_t smem[];
    __shared__ unsigned long long s_tot[32 * 12];
    const Table T = stage_table<kSmall>(p, smem);
    __syncthreads();

    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t warps_per_block = blockDim.x >> 5;
    const uint64_t gw = (uint64_t)blockIdx.x * warps_per_block + (threadIdx.x >> 5);
    const uint64_t stride = (uint64_t)gridDim.x * warps_per_block * 128ull;
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
        uint32_t tag4 = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const bool valid = vvalid(p, base + j) && watch_pass(r.src[j], r.dst[j], p);
            const uint32_t s_in = in8[2 * j];
            const uint32_t d_in = in8[2 * j + 1];
            const uint32_t cell = s_in * 2u + d_in;
            const uint32_t dir = (p.lut >> (cell * 2u)) & 3u;
            uint32_t bin = 0;
            const bool inw = map_bin(r.ts[j], p, bin);
            const bool directed = valid && dir < 2u;
            if (directed && inw) { tmin = min(tmin, bin); tmax = max(tmax, bin); }
            if (directed && inw) {
                unsigned long long* slot = p.bins + ((size_t)bin * 4u + dir * 2u);
                atomicAdd(slot, 1ull);
                atomicAdd(slot + 1, (unsigned long long)r.by[j]);
            }
            tag4 |= (s_in | (d_in << 1) | ((inw ? 0u : 1u) << 2)) << (8 * j);
            tot.add(valid, cell, directed && !inw, dir, r.by[j]);
        }
        if (p.tags) store_tags4(p, base, tag4);
    }
    note_touched_warp(p, tmin, tmax);
    flush_totals(tot, p.totals, s_tot);
}

// AUTO order probe: run k of kProbeRun consecutive ts starting at (n - kProbeRun) * k / (kProbeRuns - 1)
__global__ void k_probe_gather(const uint64_t* __restrict__ ts, uint64_t n, uint64_t* __restrict__ out) {
    const uint64_t at = (n - kProbeRun) * (uint64_t)blockIdx.x / (kProbeRuns - 1);
    out[blockIdx.x * kProbeRun + threadIdx.x] = ts[at + threadIdx.x];
}

cudaError_t launch_probe_gather(const uint64_t* ts, uint64_t n, uint64_t* out, cudaStream_t st) {
    k_probe_gather<<<kProbeRuns, kProbeRun, 0, st>>>(ts, n, out);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- launchers
cudaError_t launch_materialize(unsigned long long* bins, uint32_t* flags, uint32_t n_tiles,
                               uint32_t init_word, int grid, cudaStream_t st) {
    return launch_materialize_range(bins, flags, 0, n_tiles, init_word, grid, st);
}

// tiles [t_lo, t_hi) only (the sparse multi-GPU merge materialises what it sends and owns)
cudaError_t launch_materialize_range(unsigned long long* bins, uint32_t* flags, uint32_t t_lo, uint32_t t_hi,
                                     uint32_t init_word, int grid, cudaStream_t st) {
    if (t_hi <= t_lo) return cudaSuccess;
    const uint32_t n = t_hi - t_lo;
    uint32_t need = (n + 255u) / 256u;   // 8 warps x 32 tiles per block per step
    int g = (int)((need < (uint32_t)grid) ? need : (uint32_t)grid);
    if (g < 1) g = 1;
    k_materialize<<<g, 256, 0, st>>>(reinterpret_cast<ulonglong2*>(bins) + (size_t)t_lo * kTileBins * 2u,
                                     flags + t_lo, n, init_word);
    return cudaGetLastError();
}

cudaError_t setup_hist_atomic() {
    cudaError_t e = cudaFuncSetAttribute(k_hist_atomic<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kMaxTableSmem);
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(k_hist_atomic<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxTableSmem);
}

int hist_atomic_blocks_per_sm(const KernelParams& p) {
    int nb = 0;
    const size_t sm = table_smem_bytes(p.nbnd, p.n_mixed, p.small);
    cudaError_t e = p.small ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_hist_atomic<true>, 256, sm)
                            : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_hist_atomic<false>, 256, sm);
    return (e == cudaSuccess && nb > 0) ? nb : 1;
}

cudaError_t launch_hist_atomic(const KernelParams& p, int grid, cudaStream_t st) {
    const size_t sm = table_smem_bytes(p.nbnd, p.n_mixed, p.small);
    if (p.small) k_hist_atomic<true><<<grid, 256, sm, st>>>(p);
    else k_hist_atomic<false><<<grid, 256, sm, st>>>(p);
    return cudaGetLastError();
}

}  // namespace sinet
