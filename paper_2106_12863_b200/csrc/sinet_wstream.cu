// k_hist_ws: the fused discrimination + ms-histogram kernel for approximately
// time-ordered input, warp-specialised (strategy STREAM).
//
// Same method as k_hist_stream (sinet_stream.cu): the paper's tiling of the reduce
// "when a whole problem does not fit in the cache" (§4) applied to the time
// axis -- a window of WS consecutive ms bins is privatised in shared memory while the
// records stream through, and each 256-bin tile leaves the window exactly once, written
// to HBM by the first CTA that claims it (no memset) and added by the others.  What
// differs is who does what, so that no record-processing warp ever waits at a barrier:
//
//   * 15 WORKER warps take 128-record chunks of the CTA's record range from a shared-
//     memory counter (4 records per lane, 128-bit streaming loads, the next chunk
//     prefetched into registers), classify them (Alg. 1 l.6-9 on the staged table,
//     P:L160-163), map them to ms bins (§4.1) and add count and bytes into
//     the shared-memory ring with native u32 atomics (bytes as a low word + exact carry,
//     the high word to HBM).  A record outside the resident tiles [lo, top) -- later
//     than the history kept or ahead of the window -- goes to HBM through the tile
//     protocol (sinet_tiles.cuh).  After each chunk a worker publishes its newest tile
//     and the `lo` that chunk ran with; that is all the coordination it does.
//   * 1 MANAGER warp slides the window: once every worker's newest tile is kHist tiles
//     past a tile, it raises `lo` (workers see it at their next chunk), waits until every
//     worker has finished a chunk that ran with the new `lo` (polled, no fences), then
//     retires the tiles: claims them (one CAS per tile, all in flight at once), converts
//     each ring tile to the bins' u64 layout in a staging buffer, and hands it to the TMA
//     engine -- `cp.async.bulk` (a bulk store) for a tile it won, `cp.reduce.async.bulk
//     .add.u64` (a bulk reduce-add in L2) for a tile another CTA initialised -- then zeroes
//     the ring slots and raises `top`.  Won tiles are published (release of the state
//     word) once their bulk stores have completed.
//
// Deadlock freedom: a worker waits only for a claimed tile (spill path); a claimed tile
// is published after bounded work (TMA completion, a zero-fill), because the manager
// never blocks on its workers (the handshake is polled) and publishes everything before
// it waits for a tile claimed elsewhere.
#include <type_traits>

#include "sinet_device.cuh"
#include "sinet_kernels.h"
#include "sinet_tiles.cuh"

namespace sinet {

namespace {

constexpr int kWsThreads = 512;
constexpr uint32_t kWorkers = 15;                 // worker warps; warp kWorkers manages the window
constexpr uint32_t kDone = 0xFFFFFFFFu;           // "no worker left": the identity of the head minimum
constexpr uint32_t kStageBytes = kTileBins * 32u; // one tile in the bins' layout (8 KB)
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

// TMA bulk operations (issued by one thread; bulk groups are per thread)
__device__ __forceinline__ void bulk_store(void* g, uint32_t s, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g), "r"(s), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_add_u64(void* g, uint32_t s, uint32_t bytes) {
    asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.u64 [%0], [%1], %2;" ::"l"(g), "r"(s), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// generic-proxy shared-memory writes -> visible to the async proxy (the TMA engine)
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// async-proxy global writes (completed bulk stores) -> ordered before later generic accesses
__device__ __forceinline__ void fence_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

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
// [3] retire batches, [4] tiles retired, [5] manager idle polls, [6] chunks, [7] hot chunks
__device__ unsigned long long g_ws_dbg[8];

template <int WS, int kTab, bool kW1, bool kWatch>
__global__ void __launch_bounds__(kWsThreads, 1) k_hist_ws(KernelParams p) {
    constexpr uint32_t NT = WS / kTileBins;       // resident tiles
    constexpr uint32_t kHist = 8;                 // tiles kept below the slowest worker's newest (2048 ms >= the capture disorder)
    constexpr uint32_t kLoOff = WS * 2u;          // u32 offset of the low-bytes array
    constexpr uint32_t kBatch = NT / 8u;          // tiles retired per window slide, at least
    static_assert((WS & (WS - 1)) == 0 && NT <= 32u && NT > kHist + 4u, "ring of 16 or 32 tiles");
    extern __shared__ __align__(128) uint32_t smem[];
    uint32_t* s_win = smem;                                                    // cnt[WS][2] | lo[WS][2]
    unsigned long long* s_stage = reinterpret_cast<unsigned long long*>(smem + WS * 4u);   // 2 x u64[256][4]
    uint32_t* s_tab = smem + WS * 4u + 2u * kStageBytes / 4u;
    // per worker: newest tile (a hint), the `lo` its last finished chunk ran with, done flag
    __shared__ uint32_t s_head[kWorkers], s_used[kWorkers], s_done[kWorkers], s_min[kWorkers], s_max[kWorkers];
    __shared__ uint32_t s_lo, s_top, s_next;
    __shared__ uint32_t s_range;
    __shared__ unsigned long long s_tot[16 * 12];

    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    const bool manager = warp == kWorkers;
    for (uint32_t i = threadIdx.x; i < WS; i += kWsThreads) reinterpret_cast<uint4*>(s_win)[i] = make_uint4(0u, 0u, 0u, 0u);
    const auto T = stage_stream_table<kTab>(p, s_tab);
    __syncthreads();

    const uint32_t prev_word = p.epoch > 1 ? (((p.epoch - 1u) << 2) | kTileInit) : 0u;
    const uint32_t init_word = (p.epoch << 2) | kTileInit, claimed_word = (p.epoch << 2) | kTileClaimed;
    const uint32_t win_base = (uint32_t)__cvta_generic_to_shared(s_win);
    const uint32_t stage_base = (uint32_t)__cvta_generic_to_shared(s_stage);
    const uint64_t ngroups = (p.nv + 3) / 4;
    const uint64_t nranges = (uint64_t)p.n_ranges;
    const bool tags_on = p.tags != nullptr;
    const bool key32 = p.nbins < 0x40000000u;   // 2*bin+dir keys stay below the lane sentinels

    WarpTotals tot;
    tot.zero();
    uint32_t gmin = 0xFFFFFFFFu, gmax = 0u;   // extent of this warp's binned records
    uint32_t nstage = 0u;                     // manager: bulk operations issued (staging buffer parity)

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
            if (lane < kWorkers) { s_head[lane] = lo0; s_done[lane] = 0u; s_used[lane] = 0u; }   // tiles (s_max: bins)
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
                uint32_t lo = 0, top = 0;
                if (lane == 0) { lo = lds_acquire(&s_lo); top = lds_acquire(&s_top); }
                lo = __shfl_sync(kFull, lo, 0);
                top = __shfl_sync(kFull, top, 0);
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
                if (key0 != key3 || !key32) {
                    uint32_t hi4[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const bool take = dir4[j] < 2u && (bin4[j] / kTileBins) - lo < top - lo;
                        const uint32_t a = win_base + ((bin4[j] & (WS - 1)) * 2u + dir4[j]) * 4u;
                        const uint32_t old = smem_count_and_add_lo<kLoOff * 4u>(a, take, (uint32_t)cur.by[j]);
                        const uint32_t l32 = (uint32_t)cur.by[j];
                        hi4[j] = take ? (uint32_t)(cur.by[j] >> 32) + ((old + l32 < old) ? 1u : 0u) : 0u;
                        dir4[j] |= take ? 4u : 0u;   // 4|dir: accumulated
                    }
                    bool any = false;
#pragma unroll
                    for (int j = 0; j < 4; ++j) any |= dir4[j] < 2u || hi4[j] != 0u;
                    if (p.debug) {
                        uint32_t late = 0, early = 0, hiw = 0;
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            if (dir4[j] < 2u) { if (bin4[j] / kTileBins < lo) ++late; else ++early; }
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
                                spill_warp(p, out || hi4[j] != 0u, bin4[j], dir4[j] & 1u, out ? 1u : 0u,
                                           out ? cur.by[j] : ((uint64_t)hi4[j] << 32));
                        }
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const bool b = dir4[j] < 2u;
                        const uint32_t key = b ? bin4[j] * 2u + dir4[j] : 0xFFFFFFFFu - lane;
                        const unsigned m = __match_any_sync(kFull, key);
                        const bool leader = lane == (uint32_t)(__ffs(m) - 1);
                        uint32_t cnt = 1u;
                        uint64_t byt = cur.by[j];
                        unsigned groups = __ballot_sync(kFull, b && leader && __popc(m) > 1);
                        while (groups) {
                            const int l = __ffs(groups) - 1;
                            groups &= groups - 1u;
                            const unsigned g = __shfl_sync(kFull, m, l);
                            const uint64_t sum = warp_sum_u64(((g >> lane) & 1u) ? cur.by[j] : 0ull);
                            if (lane == (uint32_t)l) { byt = sum; cnt = (uint32_t)__popc(g); }
                        }
                        const bool act = b && leader;
                        const bool in_ring = act && (bin4[j] / kTileBins) - lo < top - lo;
                        const uint32_t hv = in_ring ? ring_add<kLoOff * 4u>(
                                                          win_base + ((bin4[j] & (WS - 1)) * 2u + dir4[j]) * 4u, cnt, byt)
                                                    : 0u;
                        const bool out = act && !in_ring;
                        if (__any_sync(kFull, out || hv != 0u))
                            spill_warp(p, out || hv != 0u, bin4[j], dir4[j], out ? cnt : 0u,
                                       out ? byt : ((uint64_t)hv << 32));
                    }
                }
                // ---- publish progress: the newest tile (a hint for the manager) and the `lo` this
                // chunk ran with (release: the warp's ring atomics happen before it).  Once a
                // worker has published lo' >= L, none of its chunks touches a tile below L again:
                // earlier chunks are finished, and later ones read lo >= lo' (read-read coherence).
                bmax = __reduce_max_sync(kFull, bmax);
                head = max(head, bmax / kTileBins);
                __syncwarp();
                if (p.debug && lane == 0) { atomicAdd(&g_ws_dbg[6], 1ull); if (key0 == key3) atomicAdd(&g_ws_dbg[7], 1ull); }
                if (lane == 0) {
                    *reinterpret_cast<volatile uint32_t*>(&s_head[warp]) = head;
                    sts_release(&s_used[warp], lo);
                }
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
            // retired: the oldest resident tile; lo_pub: the published lower edge (raised
            // eagerly); a tile below every worker's acknowledged lo (s_used) is retired.  The
            // batch is everything that became safe, so a manager that falls behind catches up
            // with larger batches (one claim round trip + one completion wait per batch).
            uint32_t retired = s_lo, lo_pub = retired, hull_hi = retired;
            unsigned pub_m = 0u;          // won tiles of the last batch, published after their bulk stores
            uint32_t pub_base = 0u;
            auto publish = [&]() {
                if (pub_m) {
                    if (lane == 0) {
                        bulk_wait_all();        // the bulk stores are complete in global memory
                        fence_async_global();
                        for (unsigned m = pub_m; m; m &= m - 1u)
                            st_release_u32(p.tile_flags + pub_base + (uint32_t)(__ffs(m) - 1), init_word);
                    }
                    __syncwarp();
                    pub_m = 0u;
                }
            };
            // ring tile t -> staging buffer (bins layout u64[256][2 dir][2 metric]), ring slots zeroed;
            // returns the buffer's shared address
            auto convert = [&](uint32_t t) -> uint32_t {
                const uint32_t b = nstage & 1u;
                if (lane == 0 && nstage >= 2u) bulk_wait_read<1>();   // the buffer's previous bulk read is done
                __syncwarp();
                ulonglong2* st = reinterpret_cast<ulonglong2*>(s_stage) + b * (kTileBins * 2u);
                const uint32_t s0 = (t * kTileBins) & (WS - 1);
#pragma unroll 4
                for (uint32_t i = lane; i < kTileBins; i += 32u) {
                    const uint2 c = *reinterpret_cast<const uint2*>(s_win + (s0 + i) * 2u);
                    const uint2 l = *reinterpret_cast<const uint2*>(s_win + kLoOff + (s0 + i) * 2u);
                    st[i * 2u] = make_ulonglong2(c.x, l.x);
                    st[i * 2u + 1u] = make_ulonglong2(c.y, l.y);
                }
                __syncwarp();
                // zero the tile's ring slots: 2 KB of counts + 2 KB of low words, 128-bit stores
                uint4* zc = reinterpret_cast<uint4*>(s_win + s0 * 2u);
                uint4* zl = reinterpret_cast<uint4*>(s_win + kLoOff + s0 * 2u);
#pragma unroll
                for (uint32_t i = lane; i < kTileBins / 2u; i += 32u) { zc[i] = make_uint4(0u, 0u, 0u, 0u); zl[i] = make_uint4(0u, 0u, 0u, 0u); }
                fence_async_smem();
                __syncwarp();
                return stage_base + b * kStageBytes;
            };
            auto issue = [&](uint32_t t, bool won, uint32_t sa) {
                if (lane == 0) {
                    void* g = p.bins + (size_t)t * kTileBins * 4u;
                    if (won) bulk_store(g, sa, kStageBytes);
                    else bulk_add_u64(g, sa, kStageBytes);
                    bulk_commit();
                }
                ++nstage;
            };
            // retire tiles [t0, t1), t1 - t0 <= NT <= 32 (no worker touches them any more)
            auto retire = [&](uint32_t t0, uint32_t t1) {
                const uint32_t n = t1 - t0;
                uint32_t o = 0u;
                if (lane < n && t0 + lane <= hull_hi) {   // tiles beyond the hull hold no data
                    uint32_t* f = p.tile_flags + t0 + lane;
                    o = claim_outcome(f, p.epoch, prev_word, atomicCAS(f, prev_word, claimed_word));
                }
                const unsigned won_m = __ballot_sync(kFull, o == kWon), add_m = __ballot_sync(kFull, o == kInit);
                const unsigned busy_m = __ballot_sync(kFull, o == kBusy);
                for (unsigned m = won_m | add_m; m; m &= m - 1u) {
                    const uint32_t kk = (uint32_t)(__ffs(m) - 1);
                    issue(t0 + kk, (won_m >> kk) & 1u, convert(t0 + kk));
                }
                pub_m = won_m;
                pub_base = t0;
                if (busy_m) {
                    // claimed elsewhere, not yet initialised: publish ours first (we then hold no
                    // claim), wait for the claimer, add
                    publish();
                    for (unsigned m = busy_m; m; m &= m - 1u) {
                        const uint32_t kk = (uint32_t)(__ffs(m) - 1);
                        if (lane == 0) {
                            uint32_t spins = 0;
                            while (ld_acquire_u32(p.tile_flags + t0 + kk) != init_word) {
                                __nanosleep(200);
                                if (++spins > kSpinLimit) __trap();
                            }
                        }
                        __syncwarp();
                        issue(t0 + kk, false, convert(t0 + kk));
                    }
                }
            };
            for (;;) {
                publish();
                const bool dn = (lane < kWorkers) ? lds_acquire(&s_done[lane]) != 0u : true;
                const uint32_t used = (lane < kWorkers) ? lds_acquire(&s_used[lane]) : kDone;
                const uint32_t hd = (lane < kWorkers) ? lds_volatile(&s_head[lane]) : 0u;
                const bool all_done = __all_sync(kFull, dn);
                const uint32_t hmin = __reduce_min_sync(kFull, dn ? kDone : hd);   // finished workers do not pin the window
                hull_hi = max(hull_hi, __reduce_max_sync(kFull, hd));
                // raise the lower edge as far as the slowest worker's history allows
                uint32_t target = retired;
                if (all_done) target = min(retired + NT, hull_hi + 1u);
                else if (hmin >= retired + kHist) target = min(retired + NT, hmin - kHist);
                if (target > lo_pub) {
                    lo_pub = target;
                    if (lane == 0) sts_release(&s_lo, lo_pub);
                }
                // retire what every worker has acknowledged
                const uint32_t safe = all_done ? lo_pub : min(lo_pub, __reduce_min_sync(kFull, dn ? kDone : used));
                if (safe >= retired + (all_done ? 1u : kBatch)) {
                    __syncwarp();   // every lane's ring reads after the workers' releases (acquired above)
                    if (p.debug && lane == 0) { atomicAdd(&g_ws_dbg[3], 1ull); atomicAdd(&g_ws_dbg[4], (unsigned long long)(safe - retired)); }
                    retire(retired, safe);
                    retired = safe;
                    __syncwarp();
                    if (lane == 0) sts_release(&s_top, retired + NT);
                    continue;
                }
                if (all_done && lo_pub == retired) break;
                if (p.debug && lane == 0) atomicAdd(&g_ws_dbg[5], 1ull);
                __nanosleep(32);
            }
            publish();
            if (lane == 0) bulk_wait_all();
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
constexpr size_t ring_smem(int ws) { return (size_t)ws * 16u + 2u * kStageBytes; }
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
        static const unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
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
