// Tile-state protocol shared by the stream kernels (write-once tiles of 256 bins).
//
// A tile's state word is epoch << 2 | {claimed, initialised}; a tile whose word is from
// an older epoch is "virtually zero".  The first CTA to claim a tile (CAS) initialises it
// in HBM (stores or zero-fill) and publishes it (release); everyone else adds with RED
// once it is initialised.  Nothing waits on a tile while holding an unpublished claim,
// so the protocol cannot deadlock.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "sinet_params.h"

namespace sinet {
namespace {   // internal linkage: each kernel TU gets its own copy (no -rdc)

constexpr uint32_t kSpinLimit = 1u << 25;   // ~seconds of waiting on one tile: a protocol bug

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Predicated shared-memory updates of one (bin, dir) slot at shared address a (count word;
// low bytes word at a + LO): if take, count += 1 and low += lo, returning the
// low word's old value (0 if not taken).
template <uint32_t LO>
__device__ __forceinline__ uint32_t smem_count_and_add_lo(uint32_t a, bool take, uint32_t lo) {
    uint32_t old;
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\tmov.u32 %0, 0;\n\t"
                 "@q red.shared.add.u32 [%1], 1;\n\t@q atom.shared.add.u32 %0, [%1+%4], %3;\n\t}"
                 : "=r"(old) : "r"(a), "r"((uint32_t)take), "r"(lo), "n"(LO) : "memory");
    return old;
}

// One 32-byte bin {a, b, c, d} (u64 each, from u32 values) with a single 256-bit evict-first
// store (STG.E.EF.256, sm_100): the bins are written once and never re-read by the kernel.
__device__ __forceinline__ void st_cs_v4u64(unsigned long long* p, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("st.global.cs.v4.u64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"((unsigned long long)a),
                 "l"((unsigned long long)b), "l"((unsigned long long)c), "l"((unsigned long long)d) : "memory");
}

__device__ __forceinline__ void st_release_u32(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// true: the caller won the tile and must initialise + release it;
// false: the tile is initialised in this epoch (possibly after waiting).
__device__ bool claim_or_wait(uint32_t* flag, uint32_t epoch) {
    const uint32_t claimed = (epoch << 2) | kTileClaimed, init = (epoch << 2) | kTileInit;
    uint32_t f = ld_acquire_u32(flag);
    uint32_t spins = 0;
    for (;;) {
        if (f == init) return false;
        if (f == claimed) {
            __nanosleep(100);
            f = ld_acquire_u32(flag);
            if (++spins > kSpinLimit) __trap();   // a protocol bug must fail loudly, not hang the GPU
            continue;
        }
        const uint32_t old = atomicCAS(flag, f, claimed);
        if (old == f) return true;
        f = old;
    }
}

// Warp-cooperative spill (warp-uniform call): every lane with `need` adds
// (cnt, bytes) to (bin, dir) in HBM.  For each distinct tile one lane claims
// it (or waits until it is initialised); if it wins, the whole warp zero-fills
// the tile and the lane publishes it.  No lane ever waits on a lane of its own
// warp (a spin on a sibling lane could deadlock at the compiler's
// reconvergence point), only on other warps/CTAs, which never wait while
// holding a claim.
__device__ void spill_warp(const KernelParams& p, bool need, uint32_t bin, uint32_t dir, uint32_t cnt,
                           uint64_t bytes) {
    const uint32_t lane = threadIdx.x & 31u;
    unsigned pending = __ballot_sync(kFull, need);
    const uint32_t t = bin / kTileBins;
    while (pending) {
        const int l = __ffs(pending) - 1;
        const uint32_t tl = __shfl_sync(kFull, t, l);
        uint32_t won = 0;
        if (lane == 0) won = claim_or_wait(p.tile_flags + tl, p.epoch) ? 1u : 0u;
        won = __shfl_sync(kFull, won, 0);
        if (won) {
            ulonglong2* b = reinterpret_cast<ulonglong2*>(p.bins + (size_t)tl * kTileBins * 4u);
            const ulonglong2 z = make_ulonglong2(0ull, 0ull);
            for (uint32_t i = lane; i < kTileBins * 2u; i += 32u) b[i] = z;
            __syncwarp();
            // st.release is cumulative over the warp's zero stores ordered before it by __syncwarp
            if (lane == 0) st_release_u32(p.tile_flags + tl, (p.epoch << 2) | kTileInit);
        }
        __syncwarp();
        const bool mine = need && t == tl;
        if (mine) {
            unsigned long long* slot = p.bins + ((size_t)bin * 4u + dir * 2u);
            if (cnt) atomicAdd(slot, (unsigned long long)cnt);
            if (bytes) atomicAdd(slot + 1, (unsigned long long)bytes);
        }
        pending &= ~__ballot_sync(kFull, mine);
    }
}

// Outcome of a tile claim, stored per ring slot tagged with the tile: (t+1) << 2 | outcome.
constexpr uint32_t kWon = 1u;    // we initialise the tile: plain stores, then release
constexpr uint32_t kInit = 2u;   // already initialised by someone else: add with RED
constexpr uint32_t kBusy = 3u;   // claimed by someone else, not yet initialised: wait, then RED

// One non-blocking claim attempt.  `old` is the value the first CAS returned
// (expected = prev_word, the state most tiles are in); a tile still in an
// older epoch is retried with the value seen.
__device__ __forceinline__ uint32_t claim_outcome(uint32_t* flag, uint32_t epoch, uint32_t prev_word, uint32_t old) {
    const uint32_t claimed = (epoch << 2) | kTileClaimed, init = (epoch << 2) | kTileInit;
    uint32_t expect = prev_word;
    for (;;) {
        if (old == expect) return kWon;
        if (old == init) return kInit;
        if (old == claimed) return kBusy;
        expect = old;
        old = atomicCAS(flag, expect, claimed);
    }
}

}  // namespace
}  // namespace sinet
