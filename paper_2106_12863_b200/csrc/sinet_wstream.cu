// k_hist_ws: a warp-specialised variant of the stream kernel (strategy
// STREAM) -- EXPERIMENTAL, opt-in (knob stream_kernel = 2); k_hist_stream stays the default
// because it is faster on B200 (DESIGN.md §6.3 has the measurements and why).
//
// Same method as k_hist_stream (sinet_stream.cu): the paper's tiling of the reduce "when a
// whole problem does not fit in the cache" (§4) applied to the time axis -- a
// window of ms bins is privatised in shared memory while the records stream through, and each
// 256-bin tile leaves the window exactly once, written by the first CTA that claims it.  Here
// no warp that processes records ever waits at a barrier:
//   * 15 WORKER warps take 128-record chunks from a shared counter, classify them (Alg. 1
//     l.6-9 on the staged table), map them (§4.1), and add the records
//     inside the window [lo, top) to the ring in a short critical section (flag store + fence +
//     window load ... ring atomics ... flag release); records outside go to HBM through the
//     tile protocol (sinet_tiles.cuh).  After a chunk a worker flushes one retiring tile if any
//     is posted, and publishes its newest tile.
//   * 1 MANAGER warp raises lo to kHist tiles below the slowest worker's newest tile, waits
//     until it has seen every worker outside its critical section (Dekker against the workers'
//     flag stores), claims the tiles below the new lo with one CAS each, posts them to the
//     flush queue (won tiles first), helps flush, and raises top once all are flushed.
// Deadlock freedom: every wait is for a tile claimed elsewhere, and a claimed tile is flushed
// and published after bounded work (won tiles are handed out before tiles that may wait).
#include <type_traits>

#include "sinet_device.cuh"
#include "sinet_kernels.h"
#include "sinet_tiles.cuh"

namespace sinet {

namespace {

constexpr int kWsThreads = 512;
constexpr uint32_t kWorkers = 15;                 // worker warps; warp kWorkers manages the window
constexpr uint32_t kDone = 0xFFFFFFFFu;           // "no worker left": the identity of the head minimum
constexpr uint32_t kChunk = 128;                  // records per worker chunk (4 per lane)

__device__ __forceinline__ uint32_t lds_acquire(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"((uint32_t)__cvta_generic_to_shared(p)) : "memory");
    return v;
}
__device__ __forceinline__ void sts_release(uint32_t* p, uint32_t v) {
    asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(p)), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t lds_volatile(const uint32_t* p) { return *reinterpret_cast<const volatile uint32_t*>(p); }

// count += cnt and low += lo of one ring slot (count word a, low word a + LO), returning
// the high word owed to HBM: (bytes >> 32) + the carry out of the low word
template <uint32_t LO>
__device__ __forceinline__ uint32_t ring_add(uint32_t a, uint32_t cnt, uint64_t bytes) {
    uint32_t old;
    const uint32_t lo = (uint32_t)bytes;
    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a), "r"(cnt) : "memory");
    asm volatile("atom.shared.add.u32 %0, [%1+%3], %2;" : "=r"(old) : "r"(a), "r"(lo), "n"(LO) : "memory");
    return (uint32_t)(bytes >> 32) + ((old + lo < old) ? 1u : 0u);
}

}  // namespace

// diagnostics (sinet_debug_counters): [0] late records, [1] early records, [2] high-word spills,
// [3] retire batches, [4] tiles retired, [5] manager idle polls, [6] chunks, [7] hot chunks,
// [8] polls waiting on heads, [9] polls waiting on the handshake, [10] sum of (tile - top) of early records, [11] max spread of heads
__device__ unsigned long long g_ws_dbg[12];
template <int WS, int kTab, bool kW1, bool kWatch>
__global__ void __launch_bounds__(kWsThreads, 1) k_hist_ws(KernelParams p) {
    constexpr uint32_t NT = WS / kTileBins;       // resident tiles
    constexpr uint32_t kHist = 8;                 // tiles kept below the slowest worker's newest (2048 ms >= the capture disorder)
    constexpr uint32_t kLoOff = WS * 2u;          // u32 offset of the low-bytes array
    constexpr uint32_t kBatch = NT / 8u;          // tiles retired per window slide, at least
    constexpr uint32_t kAhead = NT / 4u + 1u;     // tiles of room kept above the fastest worker's newest
    static_assert((WS & (WS - 1)) == 0 && NT <= 32u && NT > kHist + 4u, "ring of 16 or 32 tiles");
    extern __shared__ __align__(128) uint32_t smem[];
    uint32_t* s_win = smem;                                                    // cnt[WS][2] | lo[WS][2]
    uint32_t* s_tab = smem + WS * 4u;
    // per worker: newest tile (a hint), inside the ring critical section, done flag
    __shared__ uint32_t s_head[kWorkers], s_busy[kWorkers], s_done[kWorkers], s_min[kWorkers], s_max[kWorkers];
    __shared__ uint32_t s_lo, s_top, s_next;
    // the flush queue: one batch of tiles [s_q_t0, s_q_t0 + s_q_n) with their claim outcomes, taken
    // tile by tile by whichever warp is free (workers after a chunk, the manager while it waits)
    // (handed out won tiles first, then initialised ones, then busy ones: a warp waiting for a busy
    // tile never holds up a won tile of its own batch that another CTA may be waiting for)
    __shared__ uint32_t s_q_t0, s_q_n, s_q_won, s_q_add, s_q_gen, s_q_next, s_q_done;
    __shared__ uint8_t s_q_perm[32];
    __shared__ uint32_t s_range;
    __shared__ unsigned long long s_tot[16 * 12];

    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    const bool manager = warp == kWorkers;
    for (uint32_t i = threadIdx.x; i < WS; i += kWsThreads) reinterpret_cast<uint4*>(s_win)[i] = make_uint4(0u, 0u, 0u, 0u);
    const auto T = stage_stream_table<kTab>(p, s_tab);
    if (threadIdx.x == 0) { s_q_n = 0u; s_q_gen = 0u; s_q_next = 0u; s_q_done = 0u; }
    __syncthreads();

    const uint32_t prev_word = p.epoch > 1 ? (((p.epoch - 1u) << 2) | kTileInit) : 0u;
    const uint32_t init_word = (p.epoch << 2) | kTileInit, claimed_word = (p.epoch << 2) | kTileClaimed;
    const uint32_t win_base = (uint32_t)__cvta_generic_to_shared(s_win);
    const uint64_t ngroups = (p.nv + 3) / 4;
    const uint64_t nranges = (uint64_t)p.n_ranges;
    const bool tags_on = p.tags != nullptr;
    const bool key32 = p.nbins < 0x40000000u;   // 2*bin+dir keys stay below the lane sentinels

    WarpTotals tot;
    tot.zero();
    uint32_t gmin = 0xFFFFFFFFu, gmax = 0u;   // extent of this warp's binned records

    // ring tile t -> HBM, its ring slots zeroed (warp-uniform call): kind 0 = won (plain 128-bit
    // stores of all 256 bins, one 32-byte sector each, evict-first, then publish), 1 = initialised
    // by another CTA (RED.ADD.64 of the nonzero counters), 2 = claimed by another CTA and not yet
    // initialised (wait -- holding nothing unpublished -- then as 1)
    auto flush_tile = [&](uint32_t t, uint32_t kind) {
        if (kind == 2u) {
            if (lane == 0) {
                uint32_t spins = 0;
                while (ld_acquire_u32(p.tile_flags + t) != init_word) {
                    __nanosleep(200);
                    if (++spins > kSpinLimit) __trap();
                }
            }
            __syncwarp();
        }
        const uint32_t s0 = (t * kTileBins) & (WS - 1);
        unsigned long long* g = p.bins + (size_t)t * kTileBins * 4u;
#pragma unroll 4
        for (uint32_t i = lane; i < kTileBins; i += 32u) {
            uint2* sc = reinterpret_cast<uint2*>(s_win + (s0 + i) * 2u);
            uint2* sl = reinterpret_cast<uint2*>(s_win + kLoOff + (s0 + i) * 2u);
            const uint2 c = *sc, l = *sl;
            *sc = make_uint2(0u, 0u);
            *sl = make_uint2(0u, 0u);
            unsigned long long* b = g + i * 4u;
            if (kind == 0u) {
                __stcs(reinterpret_cast<ulonglong2*>(b), make_ulonglong2(c.x, l.x));
                __stcs(reinterpret_cast<ulonglong2*>(b) + 1, make_ulonglong2(c.y, l.y));
            } else {   // a record always adds a count, so zero count => zero bytes
                if (c.x) { atomicAdd(b, (unsigned long long)c.x); if (l.x) atomicAdd(b + 1, (unsigned long long)l.x); }
                if (c.y) { atomicAdd(b + 2, (unsigned long long)c.y); if (l.y) atomicAdd(b + 3, (unsigned long long)l.y); }
            }
        }
        __syncwarp();
        // the release is cumulative over the warp's stores ordered before it by __syncwarp
        if (kind == 0u && lane == 0) st_release_u32(p.tile_flags + t, init_word);
    };
    // take one tile of the posted batch, if any is left, and flush it (warp-uniform call)
    auto help_flush = [&]() -> bool {
        uint32_t v = 0, ok = 0, t0 = 0, won = 0, add = 0;
        if (lane == 0 && (lds_volatile(&s_q_next) & 0xFFu) < lds_volatile(&s_q_n)) {
            asm volatile("atom.acquire.cta.shared::cta.add.u32 %0, [%1], 1;" : "=r"(v)
                         : "r"((uint32_t)__cvta_generic_to_shared(&s_q_next)) : "memory");
            const uint32_t idx = v & 0xFFu;
            if ((v >> 8) == lds_volatile(&s_q_gen) && idx < lds_volatile(&s_q_n)) {
                const uint32_t k = s_q_perm[idx];
                ok = 1u;
                t0 = s_q_t0 + k;
                won = (s_q_won >> k) & 1u;
                add = (s_q_add >> k) & 1u;
            }
        }
        ok = __shfl_sync(kFull, ok, 0);
        if (!ok) return false;
        t0 = __shfl_sync(kFull, t0, 0);
        won = __shfl_sync(kFull, won, 0);
        add = __shfl_sync(kFull, add, 0);
        flush_tile(t0, won ? 0u : (add ? 1u : 2u));
        if (lane == 0) asm volatile("red.release.cta.shared::cta.add.u32 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&s_q_done)) : "memory");
        return true;
    };

    for (;;) {   // record ranges handed out dynamically (one atomic per range)
        if (threadIdx.x == 0) s_range = atomicAdd(p.range_counter, 1u);
        __syncthreads();
        const uint64_t range = s_range;
        if (range >= nranges) break;
        const uint64_t r0 = (ngroups * range / nranges) * 4, r1 = (ngroups * (range + 1) / nranges) * 4;
        const uint32_t nchunks = (uint32_t)((r1 - r0 + kChunk - 1) / kChunk);
        const uint64_t full_lo = (p.head != 0u) ? 4u : 0u;        // chunks whose every record is valid
        const uint64_t full_hi = (r1 > p.nv) ? r1 - 4 : r1;

        // ---- window start: every worker loads its first chunk; the window opens at the
        // oldest in-window bin among them
        typename RecN<4>::T cur, nxt;
        uint32_t k = warp;
        if (!manager) {
            const uint64_t v = r0 + (uint64_t)k * kChunk + lane * 4u;
            uint32_t mn = 0xFFFFFFFFu, mx = 0u;
            if (k < nchunks && v < r1) {
                load4(p, v, cur);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    uint32_t b;
                    if (vvalid(p, v + j) && map_bin(cur.ts[j], p, b)) { mn = min(mn, b); mx = max(mx, b); }
                }
            }
            mn = __reduce_min_sync(kFull, mn);
            mx = __reduce_max_sync(kFull, mx);
            if (lane == 0) { s_min[warp] = mn; s_max[warp] = mx; }
        }
        if (threadIdx.x == 0) s_next = kWorkers;
        __syncthreads();
        if (manager) {
            uint32_t mn = (lane < kWorkers) ? s_min[lane] : 0xFFFFFFFFu;
            uint32_t mx = (lane < kWorkers && s_min[lane] != 0xFFFFFFFFu) ? s_max[lane] : 0u;
            mn = __reduce_min_sync(kFull, mn);
            mx = __reduce_max_sync(kFull, mx);
            uint32_t lo0 = 0u;
            if (mn <= mx) {
                const uint32_t tmin = mn / kTileBins, tmax = mx / kTileBins;
                lo0 = (tmax >= tmin + (NT - 2u)) ? tmax - (NT - 2u) : tmin;
            }
            if (lane == 0) { s_lo = lo0; s_top = lo0 + NT; }
            if (lane < kWorkers) { s_head[lane] = lo0; s_done[lane] = 0u; s_busy[lane] = 0u; }   // tiles (s_max: bins)
        }
        __syncthreads();

        if (!manager) {
            // ================================================================ worker
            uint32_t head = s_lo;   // newest tile this warp has binned into (monotone)
            if (s_min[warp] != 0xFFFFFFFFu) head = max(head, s_max[warp] / kTileBins);
            uint32_t kn = 0;
            if (lane == 0) kn = atomicAdd(&s_next, 1u);
            kn = __shfl_sync(kFull, kn, 0);
            if (kn < nchunks) {
                const uint64_t v = r0 + (uint64_t)kn * kChunk + lane * 4u;
                if (v < r1) load4(p, v, nxt);
            }
            while (k < nchunks) {
                const uint64_t cb = r0 + (uint64_t)k * kChunk;
                const uint64_t my_v = cb + lane * 4u;
                const bool have = my_v < r1;
                const bool full = cb >= full_lo && cb + kChunk <= full_hi;

                // ---- a3-a5: classify and map (dir4[j] = 0/1 binned in that direction, 3 = not binned)
                uint32_t bin4[4], dir4[4];
                uint32_t tag4 = 0;
                uint32_t addr[8], in8[8];
#pragma unroll
                for (int j = 0; j < 4; ++j) { addr[2 * j] = cur.src[j]; addr[2 * j + 1] = cur.dst[j]; }
                member_batch_tab<kTab, 8>(addr, in8, T);
                auto classify = [&](auto kFullTag) {
                    constexpr bool kAllValid = decltype(kFullTag)::value;
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const bool valid = kAllValid || ((full || (have && vvalid(p, my_v + j))) &&
                                                         (!kWatch || watched(cur.src[j], p) || watched(cur.dst[j], p)));
                        const uint32_t cell = in8[2 * j] * 2u + in8[2 * j + 1];
                        const uint32_t dir = (p.lut >> (cell * 2u)) & 3u;
                        uint32_t bin = 0;
                        bool inw;
                        if (kW1) {
                            const uint64_t d = cur.ts[j] - p.start;
                            inw = d < (uint64_t)p.window;
                            bin = (uint32_t)d;
                        } else {
                            inw = map_bin(cur.ts[j], p, bin);
                        }
                        const bool directed = valid && dir < 2u;
                        const bool binned = directed && inw;
                        bin4[j] = bin;
                        dir4[j] = binned ? dir : 3u;
                        if (!kAllValid && tags_on)
                            tag4 |= (in8[2 * j] | (in8[2 * j + 1] << 1) | ((inw ? 0u : 1u) << 2)) << (8 * j);
                        if (kAllValid) tot.add_valid(cell, directed && !inw, dir, cur.by[j]);
                        else tot.add(valid, cell, directed && !inw, dir, cur.by[j]);
                    }
                };
                if (full && !kWatch && !tags_on) classify(std::true_type{});
                else classify(std::false_type{});
                if (tags_on && have) store_tags4(p, my_v, tag4);

                // ---- a6: accumulate into the ring, or to HBM when outside [lo, top)
                uint32_t bmax = 0u, bmin = 0xFFFFFFFFu;
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (dir4[j] < 2u) { bmax = max(bmax, bin4[j]); bmin = min(bmin, bin4[j]); }
                gmin = min(gmin, bmin);
                gmax = max(gmax, bmax);
                // hot chunk (first and last record in the same (bin, dir)): aggregate equal keys first
                const uint32_t key0 = __shfl_sync(kFull, dir4[0] < 2u ? bin4[0] * 2u + dir4[0] : 0xFFFFFFFFu, 0);
                const uint32_t key3 = __shfl_sync(kFull, dir4[3] < 2u ? bin4[3] * 2u + dir4[3] : 0xFFFFFFFEu, 31);
                const bool hot = key0 == key3 && key32;
                uint32_t cnt4[4];
                uint64_t by4[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) { cnt4[j] = 1u; by4[j] = cur.by[j]; }
                if (hot) {   // one accumulation per distinct key of the warp (its leader), count = group size
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const bool b = dir4[j] < 2u;
                        const unsigned m = __match_any_sync(kFull, b ? bin4[j] * 2u + dir4[j] : 0xFFFFFFFFu - lane);
                        const bool leader = lane == (uint32_t)(__ffs(m) - 1);
                        unsigned groups = __ballot_sync(kFull, b && leader && __popc(m) > 1);
                        while (groups) {
                            const int l = __ffs(groups) - 1;
                            groups &= groups - 1u;
                            const unsigned g = __shfl_sync(kFull, m, l);
                            const uint64_t sum = warp_sum_u64(((g >> lane) & 1u) ? cur.by[j] : 0ull);
                            if (lane == (uint32_t)l) { by4[j] = sum; cnt4[j] = (uint32_t)__popc(g); }
                        }
                        if (b && !leader) dir4[j] |= 4u;   // folded into its leader
                    }
                }
                // ---- critical section (Dekker with the manager): announce, read the window, add
                // the records inside it to the ring, leave with a release.  A manager that saw this
                // warp outside the section after raising lo knows its ring adds below lo are done.
                uint32_t lo = 0, top = 0;
                if (lane == 0) {
                    *reinterpret_cast<volatile uint32_t*>(&s_busy[warp]) = 1u;
                    __threadfence_block();
                    lo = lds_acquire(&s_lo);
                    top = lds_acquire(&s_top);
                }
                lo = __shfl_sync(kFull, lo, 0);
                top = __shfl_sync(kFull, top, 0);
                uint32_t hi4[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const bool take = dir4[j] < 2u && (bin4[j] / kTileBins) - lo < top - lo;
                    const uint32_t a = win_base + ((bin4[j] & (WS - 1)) * 2u + (dir4[j] & 1u)) * 4u;
                    uint32_t old;
                    if (!hot) {
                        old = smem_count_and_add_lo<kLoOff * 4u>(a, take, (uint32_t)by4[j]);
                    } else {
                        old = 0u;
                        if (take) {
                            asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a), "r"(cnt4[j]) : "memory");
                            asm volatile("atom.shared.add.u32 %0, [%1+%3], %2;" : "=r"(old) : "r"(a), "r"((uint32_t)by4[j]), "n"(kLoOff * 4u) : "memory");
                        }
                    }
                    const uint32_t l32 = (uint32_t)by4[j];
                    hi4[j] = take ? (uint32_t)(by4[j] >> 32) + ((old + l32 < old) ? 1u : 0u) : 0u;
                    dir4[j] |= take ? 4u : 0u;   // 4|dir: accumulated (or folded)
                }
                __syncwarp();
                if (lane == 0) sts_release(&s_busy[warp], 0u);
                // ---- outside the section: records outside [lo, top) and owed high words to HBM
                bool any = false;
#pragma unroll
                for (int j = 0; j < 4; ++j) any |= dir4[j] < 2u || hi4[j] != 0u;
                if (p.debug) {
                    uint32_t late = 0, early = 0, hiw = 0;
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        if (dir4[j] < 2u) {
                            if (bin4[j] / kTileBins < lo) ++late;
                            else { ++early; atomicAdd(&g_ws_dbg[10], (unsigned long long)(bin4[j] / kTileBins - top)); }
                        }
                        if (hi4[j]) ++hiw;
                    }
                    late = __reduce_add_sync(kFull, late); early = __reduce_add_sync(kFull, early);
                    hiw = __reduce_add_sync(kFull, hiw);
                    if (lane == 0) { atomicAdd(&g_ws_dbg[0], late); atomicAdd(&g_ws_dbg[1], early); atomicAdd(&g_ws_dbg[2], hiw); }
                }
                if (__any_sync(kFull, any)) {
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const bool out = dir4[j] < 2u;
                        if (__any_sync(kFull, out || hi4[j] != 0u))
                            spill_warp(p, out || hi4[j] != 0u, bin4[j], dir4[j] & 1u, out ? cnt4[j] : 0u,
                                       out ? by4[j] : ((uint64_t)hi4[j] << 32));
                    }
                }
                help_flush();   // at most one retiring tile per chunk
                // ---- progress: the newest tile this warp has binned (a hint for the manager)
                bmax = __reduce_max_sync(kFull, bmax);
                head = max(head, bmax / kTileBins);
                __syncwarp();
                if (p.debug && lane == 0) { atomicAdd(&g_ws_dbg[6], 1ull); if (key0 == key3) atomicAdd(&g_ws_dbg[7], 1ull); }
                if (lane == 0) *reinterpret_cast<volatile uint32_t*>(&s_head[warp]) = head;
                k = kn;
                cur = nxt;
                if (lane == 0) kn = atomicAdd(&s_next, 1u);
                kn = __shfl_sync(kFull, kn, 0);
                if (kn < nchunks) {
                    const uint64_t v = r0 + (uint64_t)kn * kChunk + lane * 4u;
                    if (v < r1) load4(p, v, nxt);
                }
            }
            __syncwarp();
            if (lane == 0) sts_release(&s_done[warp], 1u);   // s_head keeps this warp's final newest tile
        } else {
            // ================================================================ manager
            // retired: the oldest resident tile.  The manager raises lo to kHist tiles below the
            // slowest worker's newest tile, waits until it has seen every worker outside its
            // ring section once (Dekker: lo store + fence vs the worker's flag store + fence),
            // then retires everything below the new lo in one batch (one claim round trip).
            uint32_t retired = s_lo, hull_hi = retired;
            uint32_t pend = 0u;    // a raised lo awaiting the handshake (0: none)
            bool seen = false;     // this lane's worker was seen outside the ring section since the raise
            uint32_t posted = 0u;  // a posted flush batch ends at this tile (0: none)
            uint32_t gen = lds_volatile(&s_q_gen);
            uint32_t spins = 0;
            for (;;) {
                if (posted) {   // help flush the batch; once every tile is flushed, open the slots
                    if (++spins > kSpinLimit) __trap();   // a protocol bug must fail loudly, not hang
                    const bool did = help_flush();
                    if (lds_acquire(&s_q_done) == lds_volatile(&s_q_n)) {
                        __syncwarp();
                        retired = posted;
                        posted = 0u;
                        spins = 0;
                        if (lane == 0) sts_release(&s_top, retired + NT);
                        continue;
                    }
                    if (!did) __nanosleep(32);
                    continue;
                }
                const bool dn = (lane < kWorkers) ? lds_acquire(&s_done[lane]) != 0u : true;
                const uint32_t hd = (lane < kWorkers) ? lds_volatile(&s_head[lane]) : 0u;
                const bool all_done = __all_sync(kFull, dn);
                const uint32_t hmin = __reduce_min_sync(kFull, dn ? kDone : hd);   // finished workers do not pin the window
                hull_hi = max(hull_hi, __reduce_max_sync(kFull, hd));
                const uint32_t hmax = __reduce_max_sync(kFull, dn ? 0u : hd);
                if (pend) {
                    seen |= dn || lds_acquire(&s_busy[lane < kWorkers ? lane : 0]) == 0u || lane >= kWorkers;
                    if (__all_sync(kFull, seen)) {
                        __syncwarp();   // every lane's ring reads after the workers' releases (acquired above)
                        // claim [retired, end) (tiles above the hull hold no data), post the batch
                        const uint32_t end = min(pend, max(retired, hull_hi + 1u));
                        const uint32_t n = end - retired;
                        uint32_t o = 0u;
                        if (lane < n) {
                            uint32_t* f = p.tile_flags + retired + lane;
                            o = claim_outcome(f, p.epoch, prev_word, atomicCAS(f, prev_word, claimed_word));
                        }
                        const unsigned won_m = __ballot_sync(kFull, o == kWon), add_m = __ballot_sync(kFull, o == kInit);
                        if (p.debug && lane == 0) { atomicAdd(&g_ws_dbg[3], 1ull); atomicAdd(&g_ws_dbg[4], (unsigned long long)n); }
                        if (n) {
                            ++gen;
                            // hand-out order: won, then initialised, then busy tiles
                            const unsigned busy_m = __ballot_sync(kFull, o == kBusy);
                            const unsigned below = (1u << lane) - 1u;
                            const uint32_t nw = __popc(won_m), na = __popc(add_m);
                            const uint32_t pos = (o == kWon) ? __popc(won_m & below)
                                               : (o == kInit) ? nw + __popc(add_m & below) : nw + na + __popc(busy_m & below);
                            if (lane < n) s_q_perm[pos] = (uint8_t)lane;
                            __syncwarp();
                            if (lane == 0) {
                                s_q_t0 = retired;
                                s_q_won = won_m;
                                s_q_add = add_m;
                                s_q_n = n;
                                s_q_done = 0u;
                                s_q_gen = gen;
                                sts_release(&s_q_next, gen << 8);
                            }
                            __syncwarp();
                            posted = pend;
                        } else {
                            retired = pend;
                            if (lane == 0) sts_release(&s_top, retired + NT);
                        }
                        pend = 0u;
                        continue;
                    }
                } else {
                    // raise the lower edge as far as the slowest worker's history allows
                    // (or, when one worker lags -- descheduled, or waiting in the spill path -- far enough
                    // that the fastest would run out of room, keep kAhead tiles ahead of the fastest:
                    // the laggard's few late records then go to HBM instead of everyone's early ones)
                    uint32_t target = retired;
                    if (all_done) {
                        target = min(retired + NT, hull_hi + 1u);
                    } else {
                        uint32_t want = hmin >= kHist ? hmin - kHist : 0u;
                        if (hmax + kAhead >= NT && hmax + kAhead - NT > want) want = hmax + kAhead - NT;
                        if (want >= retired + kBatch) target = min(retired + NT, want);
                    }
                    if (target > retired) {
                        if (lane == 0) {
                            *reinterpret_cast<volatile uint32_t*>(&s_lo) = target;
                            __threadfence_block();
                        }
                        __syncwarp();
                        __threadfence_block();   // Dekker: the lo store before every lane's busy reads
                        pend = target;
                        seen = false;
                        continue;
                    }
                    if (all_done) break;
                }
                if (p.debug && lane == 0) {
                    atomicAdd(&g_ws_dbg[5], 1ull);
                    atomicAdd(&g_ws_dbg[pend ? 9 : 8], 1ull);
                }
                __nanosleep(32);
            }
            __syncwarp();
        }
        __syncthreads();   // range done: the ring is all zero again
    }
    if (!manager) {
        const uint32_t mn = __reduce_min_sync(kFull, gmin), mx = __reduce_max_sync(kFull, gmax);
        if (lane == 0 && mn <= mx) { atomicMin(p.touched, mn); atomicMax(p.touched + 1, mx); }
    }
    flush_totals(tot, p.totals, s_tot);
}

// ---------------------------------------------------------------- launch
namespace {
constexpr size_t ring_smem(int ws) { return (size_t)ws * 16u; }
constexpr size_t kMaxDynSmem = 227u * 1024u - 2048u;   // minus this kernel's static shared memory
}  // namespace

#define SINET_WS_KERNEL(WSB, S, W, WL) k_hist_ws<WSB, S, W, WL>

cudaError_t setup_hist_ws() {
    cudaError_t e;
#define SET(WSB, S, W, WL)                                                                                         \
    e = cudaFuncSetAttribute(SINET_WS_KERNEL(WSB, S, W, WL), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxDynSmem); \
    if (e != cudaSuccess) return e;
#define SETW(WSB, S) SET(WSB, S, true, false) SET(WSB, S, false, false) SET(WSB, S, true, true) SET(WSB, S, false, true)
#define SETT(WSB) SETW(WSB, kTabByte) SETW(WSB, kTabPacked) SETW(WSB, kTabPackedNoL2) SETW(WSB, kTabGlobal)
    SETT(8192) SETT(4096)
#undef SETT
#undef SETW
#undef SET
    return cudaSuccess;
}

// the ring this table leaves room for: 8192 bins (32 tiles), else 4096
extern "C" int sinet_debug_counters(unsigned long long* out8, int reset) {
    if (out8 && cudaMemcpyFromSymbol(out8, g_ws_dbg, sizeof(g_ws_dbg)) != cudaSuccess) return -4;
    if (reset) {
        static const unsigned long long z[12] = {0};
        if (cudaMemcpyToSymbol(g_ws_dbg, z, sizeof(z)) != cudaSuccess) return -4;
    }
    return 0;
}

int hist_ws_ring_bins(int tab, uint32_t nbnd, uint32_t n_mixed) {
    return (ring_smem(8192) + stream_table_bytes(tab, nbnd, n_mixed) <= kMaxDynSmem) ? 8192 : 4096;
}

bool hist_ws_fits(int tab, uint32_t nbnd, uint32_t n_mixed) {
    return ring_smem(4096) + stream_table_bytes(tab, nbnd, n_mixed) <= kMaxDynSmem;
}

cudaError_t launch_hist_ws(const KernelParams& p, int sm_count, cudaStream_t st) {
    const int tab = stream_table_mode(p.has_bytes != 0u, p.nbnd, p.n_mixed, p.tab_mode);
    const int ws = hist_ws_ring_bins(tab, p.nbnd, p.n_mixed);
    const size_t sm = ring_smem(ws) + stream_table_bytes(tab, p.nbnd, p.n_mixed);
    const uint64_t chunks = (p.nv + kChunk - 1) / kChunk;
    const uint64_t want = (chunks + kWorkers * 8u - 1) / (kWorkers * 8u);   // >= 8 chunks per worker
    const int grid = (int)(want < (uint64_t)sm_count ? (want ? want : 1) : (uint64_t)sm_count);
    KernelParams q = p;
    // record ranges per CTA (dynamic): a whole number per CTA, each >= 64 chunks
    const uint64_t per = (uint64_t)grid * (uint64_t)(p.ranges_per_group ? p.ranges_per_group : 4u);
    const uint64_t max_r = chunks / 64u + 1u;
    q.n_ranges = (uint32_t)(per < max_r ? per : max_r);
    cudaError_t e = cudaMemsetAsync(p.range_counter, 0, 8, st);
    if (e != cudaSuccess) return e;
    const bool w1 = p.width == 1u, wl = p.wn != 0u;
#define LAUNCH(WSB, S)                                                                                   \
    if (w1 && !wl) SINET_WS_KERNEL(WSB, S, true, false)<<<grid, kWsThreads, sm, st>>>(q);                 \
    else if (!wl) SINET_WS_KERNEL(WSB, S, false, false)<<<grid, kWsThreads, sm, st>>>(q);                 \
    else if (w1) SINET_WS_KERNEL(WSB, S, true, true)<<<grid, kWsThreads, sm, st>>>(q);                    \
    else SINET_WS_KERNEL(WSB, S, false, true)<<<grid, kWsThreads, sm, st>>>(q);
#define LAUNCH_T(WSB) switch (tab) {                         \
        case kTabByte: LAUNCH(WSB, kTabByte) break;          \
        case kTabPacked: LAUNCH(WSB, kTabPacked) break;      \
        case kTabPackedNoL2: LAUNCH(WSB, kTabPackedNoL2) break; \
        default: LAUNCH(WSB, kTabGlobal) break;              \
    }
    if (ws == 8192) { LAUNCH_T(8192) } else { LAUNCH_T(4096) }
#undef LAUNCH_T
#undef LAUNCH
    return cudaGetLastError();
}

}  // namespace sinet
