// k_hist_stream: the fused discrimination + ms-histogram kernel for
// approximately time-ordered input (strategy STREAM).
//
// The paper tiles its two-stage map-reduce so that "a whole problem [that]
// does not fit in the cache" is reduced piece by piece (§4) and
// reduces each GPU's chunk into <timestamp,count>/<timestamp,bytes>.
// Here the tile is a window of WS consecutive millisecond bins held in shared
// memory by one CTA, which streams a contiguous range of records:
//   * records are read once with 128-bit loads, the next chunk prefetched into
//     registers while the current one is binned;
//   * each record is classified (Alg. 1 l.6-9) and mapped to its ms bin;
//   * count and bytes are accumulated with native shared-memory u32 atomics
//     (bytes as lo/hi words with an exact carry), equal keys of a warp are
//     aggregated first (hot bins);
//   * when the window slides past a 512-bin tile, the tile is retired to HBM
//     exactly once: the first CTA to claim it (state word CAS) stores its bins
//     with plain 128-bit stores (no memset, no read-modify-write), later
//     contributors wait until it is initialised and add with RED.ADD.64.
// Records outside the window (late beyond the window, or a chunk wider than
// it) take the same claim-then-RED path one at a time, so the result is exact
// for any record order; only speed depends on time locality.
#include "sinet_device.cuh"
#include "sinet_kernels.h"

namespace sinet {

namespace {

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release_u32(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// true: the caller won the tile and must initialise + release it;
// false: the tile is initialised in this epoch (possibly after waiting).
__device__ bool claim_or_wait(uint32_t* flag, uint32_t epoch) {
    const uint32_t claimed = (epoch << 2) | kTileClaimed, init = (epoch << 2) | kTileInit;
    uint32_t f = ld_acquire_u32(flag);
    for (;;) {
        if (f == init) return false;
        if (f == claimed) {
            __nanosleep(100);
            f = ld_acquire_u32(flag);
            continue;
        }
        const uint32_t old = atomicCAS(flag, f, claimed);
        if (old == f) return true;
        f = old;
    }
}

// One thread makes sure tile t is initialised (zero-filling it alone if it wins).
__device__ void ensure_tile_single(const KernelParams& p, uint32_t t) {
    uint32_t* flag = p.tile_flags + t;
    if (claim_or_wait(flag, p.epoch)) {
        ulonglong2* b = reinterpret_cast<ulonglong2*>(p.bins + (size_t)t * kTileBins * 4u);
        const ulonglong2 z = make_ulonglong2(0ull, 0ull);
        for (uint32_t i = 0; i < kTileBins * 2u; ++i) b[i] = z;
        __threadfence();
        st_release_u32(flag, (p.epoch << 2) | kTileInit);
    }
}

__device__ void spill(const KernelParams& p, uint32_t bin, uint32_t dir, uint32_t cnt, uint64_t bytes) {
    ensure_tile_single(p, bin / kTileBins);
    unsigned long long* slot = p.bins + ((size_t)bin * 4u + dir * 2u);
    atomicAdd(slot, (unsigned long long)cnt);
    if (bytes) atomicAdd(slot + 1, (unsigned long long)bytes);
}

}  // namespace

// Shared-memory window layout: 6 u32 per bin = {cnt_out, cnt_in, lo_out, lo_in, hi_out, hi_in}.
template <int THREADS, int WS, bool kBndSmem, bool kAgg>
__global__ void __launch_bounds__(THREADS, 1) k_hist_stream(KernelParams p) {
    constexpr int NW = THREADS / 32;
    constexpr uint32_t NTILE = WS / kTileBins;
    static_assert((WS & (WS - 1)) == 0 && WS % kTileBins == 0, "window must be a power of two of tiles");
    static_assert((NTILE & (NTILE - 1)) == 0, "tiles per window must be a power of two");
    extern __shared__ __align__(16) uint32_t smem[];
    uint32_t* s_win = smem;
    uint32_t* s_cls2 = s_win + WS * 6;
    __shared__ uint32_t s_red[2][2][NW];
    __shared__ uint32_t s_touched[NTILE];
    __shared__ uint32_t s_claim;
    __shared__ unsigned long long s_tot[NW * 12];

    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    for (uint32_t i = tid; i < (uint32_t)WS * 6u / 4u; i += THREADS)
        reinterpret_cast<uint4*>(s_win)[i] = make_uint4(0u, 0u, 0u, 0u);
    if (tid < NTILE) s_touched[tid] = 0u;
    const uint32_t* bnd = stage_table(p, s_cls2, s_cls2 + kClsWords, kBndSmem);
    __syncthreads();

    // accumulate (cnt, bytes) of one (bin, dir) into the window, or spill it
    auto accumulate = [&](uint32_t bin, uint32_t dir, uint32_t cnt, uint64_t bytes, uint32_t wb) {
        if (bin - wb < (uint32_t)WS) {
            uint32_t* s = s_win + (bin & (WS - 1)) * 6u + dir;
            atomicAdd(s, cnt);
            const uint32_t lo = (uint32_t)bytes;
            uint32_t hi = (uint32_t)(bytes >> 32);
            const uint32_t old = atomicAdd(s + 2, lo);
            hi += (old + lo < old) ? 1u : 0u;     // exact carry out of the low word
            if (hi) atomicAdd(s + 4, hi);
            s_touched[(bin / kTileBins) & (NTILE - 1)] = 1u;
        } else {
            spill(p, bin, dir, cnt, bytes);
        }
    };

    // retire tile t (absolute index) from the window to HBM; block-uniform call
    auto flush_tile = [&](uint32_t t) {
        const uint32_t slot_tile = t & (NTILE - 1);
        if (!s_touched[slot_tile]) return;
        if (tid == 0) s_claim = claim_or_wait(p.tile_flags + t, p.epoch) ? 1u : 0u;
        __syncthreads();
        const bool won = s_claim != 0u;
        // every thread has read s_touched[slot_tile] above; clear it before the
        // closing barrier so no accumulate of the next tile in this slot is lost
        if (tid == 0) s_touched[slot_tile] = 0u;
        for (uint32_t i = tid; i < kTileBins; i += THREADS) {
            const uint32_t bin = t * kTileBins + i;
            uint32_t* s = s_win + (bin & (WS - 1)) * 6u;
            const uint2 c = *reinterpret_cast<const uint2*>(s);
            const uint2 lo = *reinterpret_cast<const uint2*>(s + 2);
            const uint2 hi = *reinterpret_cast<const uint2*>(s + 4);
            const unsigned long long b_out = (unsigned long long)lo.x | ((unsigned long long)hi.x << 32);
            const unsigned long long b_in = (unsigned long long)lo.y | ((unsigned long long)hi.y << 32);
            ulonglong2* g = reinterpret_cast<ulonglong2*>(p.bins + (size_t)bin * 4u);
            if (won) {
                __stcg(g, make_ulonglong2(c.x, b_out));
                __stcg(g + 1, make_ulonglong2(c.y, b_in));
            } else {
                unsigned long long* g64 = p.bins + (size_t)bin * 4u;
                if (c.x) { atomicAdd(g64, (unsigned long long)c.x); if (b_out) atomicAdd(g64 + 1, b_out); }
                if (c.y) { atomicAdd(g64 + 2, (unsigned long long)c.y); if (b_in) atomicAdd(g64 + 3, b_in); }
            }
            *reinterpret_cast<uint2*>(s) = make_uint2(0u, 0u);
            *reinterpret_cast<uint2*>(s + 2) = make_uint2(0u, 0u);
            *reinterpret_cast<uint2*>(s + 4) = make_uint2(0u, 0u);
        }
        __syncthreads();
        if (tid == 0 && won) {
            __threadfence();
            st_release_u32(p.tile_flags + t, (p.epoch << 2) | kTileInit);
        }
    };

    // this CTA's contiguous range of 4-record groups (virtual index space)
    const uint64_t ngroups = (p.nv + 3) / 4;
    const uint64_t g0 = ngroups * blockIdx.x / gridDim.x;
    const uint64_t g1 = ngroups * (blockIdx.x + 1) / gridDim.x;

    WarpTotals tot;
    tot.zero();
    uint32_t wb = 0;          // window base bin (multiple of kTileBins), block-uniform
    bool have_window = false;
    Rec4 cur, nxt;
    if (g0 + tid < g1) load4(p, (g0 + tid) * 4, cur);
    uint32_t parity = 0;

    for (uint64_t cbase = g0; cbase < g1; cbase += THREADS, parity ^= 1u) {
        const uint64_t my_g = cbase + tid;
        const bool have = my_g < g1;
        if (cbase + THREADS + tid < g1) load4(p, (cbase + THREADS + tid) * 4, nxt);   // prefetch

        uint32_t bin4[4], dir4[4];
        bool binned4[4];
        uint32_t tag4 = 0, bmin = 0xFFFFFFFFu, bmax = 0u;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const bool valid = have && vvalid(p, my_g * 4 + j);
            const uint32_t s_in = member(cur.src[j], s_cls2, p.entry, bnd);
            const uint32_t d_in = member(cur.dst[j], s_cls2, p.entry, bnd);
            const uint32_t cell = s_in * 2u + d_in;
            const uint32_t dir = (p.lut >> (cell * 2u)) & 3u;
            uint32_t bin = 0;
            const bool inw = map_bin(cur.ts[j], p, bin);
            const bool directed = valid && dir < 2u;
            binned4[j] = directed && inw;
            bin4[j] = bin;
            dir4[j] = dir;
            if (binned4[j]) { bmin = min(bmin, bin); bmax = max(bmax, bin); }
            tag4 |= (s_in | (d_in << 1) | ((inw ? 0u : 1u) << 2)) << (8 * j);
            tot.add(valid, cell, directed && !inw, dir, cur.by[j]);
        }
        if (p.tags && have) store_tags4(p, my_g * 4, tag4);

        // block-wide extent of this chunk's bins
        bmin = __reduce_min_sync(kFull, bmin);
        bmax = __reduce_max_sync(kFull, bmax);
        if (lane == 0) { s_red[parity][0][warp] = bmin; s_red[parity][1][warp] = bmax; }
        __syncthreads();
        bmin = 0xFFFFFFFFu;
        bmax = 0u;
#pragma unroll
        for (int w = 0; w < NW; ++w) { bmin = min(bmin, s_red[parity][0][w]); bmax = max(bmax, s_red[parity][1][w]); }

        // slide the window so that it covers the chunk's newest bins
        if (bmin <= bmax) {
            if (!have_window) {
                wb = bmin & ~(kTileBins - 1u);
                if (bmax - wb >= (uint32_t)WS) wb = (bmax + 1u - WS + kTileBins - 1u) & ~(kTileBins - 1u);
                have_window = true;
            } else if (bmax >= wb && bmax - wb >= (uint32_t)WS) {
                const uint32_t nwb = (bmax + 1u - WS + kTileBins - 1u) & ~(kTileBins - 1u);
                const uint32_t t0 = wb / kTileBins, nt = nwb / kTileBins - t0;
                const uint32_t t1 = t0 + (nt < NTILE ? nt : NTILE);
                for (uint32_t t = t0; t < t1; ++t) flush_tile(t);
                wb = nwb;
            }
        }

        // Reduce the chunk into the window
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const bool b = binned4[j];
            if (kAgg) {
                const unsigned long long key = b ? (((unsigned long long)bin4[j] << 1) | dir4[j]) : ~0ull - lane;
                const unsigned m = __match_any_sync(kFull, key);
                const bool big = __popc(m) >= 3;
                if (__any_sync(kFull, big && b)) {
                    unsigned leaders = __ballot_sync(kFull, big && b && lane == (unsigned)(__ffs(m) - 1));
                    while (leaders) {
                        const int l = __ffs(leaders) - 1;
                        leaders &= leaders - 1;
                        const unsigned g = __shfl_sync(kFull, m, l);
                        const uint64_t s = warp_sum_u64(((g >> lane) & 1u) ? cur.by[j] : 0ull);
                        if (lane == (unsigned)l) accumulate(bin4[j], dir4[j], (uint32_t)__popc(g), s, wb);
                    }
                    if (b && !big) accumulate(bin4[j], dir4[j], 1u, cur.by[j], wb);
                    continue;
                }
            }
            if (b) accumulate(bin4[j], dir4[j], 1u, cur.by[j], wb);
        }
        cur = nxt;
    }

    // retire what is left in the window
    __syncthreads();
    if (have_window)
        for (uint32_t t = wb / kTileBins, k = 0; k < NTILE; ++t, ++k) flush_tile(t);
    flush_totals(tot, p.totals, s_tot);
}

// ---------------------------------------------------------------- launch
namespace {
constexpr int kStreamThreads = 512;
constexpr int kStreamWS = 8192;

size_t stream_smem(uint32_t nbnd) {
    return (size_t)kStreamWS * 6u * 4u + (size_t)kClsWords * 4u + ((nbnd <= kMaxSmemBnd) ? (size_t)nbnd * 4u : 0u);
}
}  // namespace

cudaError_t setup_hist_stream() {
    cudaError_t e;
#define SET(B, A)                                                                                   \
    e = cudaFuncSetAttribute(k_hist_stream<kStreamThreads, kStreamWS, B, A>,                       \
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)stream_smem(B ? kMaxSmemBnd : kMaxSmemBnd + 1)); \
    if (e != cudaSuccess) return e;
    SET(true, true) SET(true, false) SET(false, true) SET(false, false)
#undef SET
    return cudaSuccess;
}

cudaError_t launch_hist_stream(const KernelParams& p, int sm_count, bool agg, cudaStream_t st) {
    const size_t sm = stream_smem(p.nbnd);
    const bool small = p.nbnd <= kMaxSmemBnd;
    // one CTA per SM, but never more CTAs than chunks' worth of records
    uint64_t chunks = (p.nv / 4 + kStreamThreads - 1) / kStreamThreads;
    int grid = (int)((chunks < (uint64_t)sm_count) ? (chunks ? chunks : 1) : (uint64_t)sm_count);
    if (small && agg) k_hist_stream<kStreamThreads, kStreamWS, true, true><<<grid, kStreamThreads, sm, st>>>(p);
    else if (small) k_hist_stream<kStreamThreads, kStreamWS, true, false><<<grid, kStreamThreads, sm, st>>>(p);
    else if (agg) k_hist_stream<kStreamThreads, kStreamWS, false, true><<<grid, kStreamThreads, sm, st>>>(p);
    else k_hist_stream<kStreamThreads, kStreamWS, false, false><<<grid, kStreamThreads, sm, st>>>(p);
    return cudaGetLastError();
}

}  // namespace sinet
