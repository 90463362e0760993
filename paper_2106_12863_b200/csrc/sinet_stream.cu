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
//   * when the window slides past a 256-bin tile, the tile is retired to HBM
//     exactly once: the first CTA to claim it (state word CAS) stores its bins
//     with one 256-bit store each (no memset, no read-modify-write), later
//     contributors wait until it is initialised and add with RED.ADD.64.
// Records outside the window (late beyond the window, or a chunk wider than
// it) take the same claim-then-RED path one at a time, so the result is exact
// for any record order; only speed depends on time locality.
#include <type_traits>

#include "sinet_device.cuh"
#include "sinet_kernels.h"
#include "sinet_tiles.cuh"

namespace sinet {

// Shared-memory window: a ring of NT tiles x 256 ms bins, 4 u32 per bin in two arrays,
// cnt[WS][2 dir] and lo[WS][2 dir] (the low 32 bits of the byte sums): the count words of
// a warp's 32 records spread over all 32 banks (16 with one 16-byte slot per bin).  A record whose bytes
// reach the high word (>= 2^32, or a carry out of the low word: elephants, very hot bins)
// adds that part straight to HBM through the spill path, after the chunk barrier, when
// the group holds no claim.  A thread retires one bin as one full 32-byte sector (one
// STG.E.EF.256), so a warp writes 1 KB contiguous per store.  Tiles [lo_t, lo_t + NT)
// are resident.  After a chunk is accumulated, tiles below the chunk's
// oldest bin (keeping >= NT/2-1 tiles of history) are claimed with one
// non-blocking CAS each; the CAS resolves while the next chunk is loaded and
// classified, and the tiles are retired (stored or added) right after.  A CTA
// never waits on another CTA's tile while it holds an unreleased claim, so
// the protocol cannot deadlock.
template <int THREADS, int NG, int WS, int RPT, bool kAgg, bool kW1, int kTab, bool kWatch>
__global__ void __launch_bounds__(THREADS, 1) k_hist_stream(KernelParams p) {
    // RPT records per thread per chunk; with RPT == 2 the side totals live in shared
    // memory per warp (registers for 1024 threads)
    constexpr bool kSmemTot = (RPT == 2 || THREADS > 512);   // totals per warp in shared memory (registers)
    using Rec = typename RecN<RPT>::T;
    constexpr int GT = THREADS / NG;          // threads per group
    constexpr int NW = THREADS / 32;
    constexpr int GW = GT / 32;               // warps per group
    constexpr uint32_t NT = WS / kTileBins;
    static_assert((WS & (WS - 1)) == 0 && WS % kTileBins == 0, "window must be a power of two of tiles");
    static_assert(NT <= (uint32_t)GT && (NT & (NT - 1)) == 0, "tiles per window: power of two <= group threads");
    static_assert(NG == 1 || NG == 2, "one or two groups per CTA");
    constexpr uint32_t kHist = NT / 2 - 1;   // tiles of history kept below a chunk's newest tile
    extern __shared__ __align__(16) uint32_t smem[];
    __shared__ __align__(16) uint32_t s_red_all[NG][2][2][GW];   // [group][parity][min, max][warp]
    __shared__ uint32_t s_state_all[NG][NT];   // (t+1) << 2 | claim outcome, per group
    __shared__ unsigned long long s_tot[(RPT == 2) ? 1 : NW * 12];

    // NG independent groups per CTA, each with its own ring and half of the CTA's records;
    // the lookup table is shared.  A group synchronises on its own named barrier.
    const uint32_t gid = threadIdx.x / GT, tid = threadIdx.x % GT, lane = tid & 31u, warp = tid >> 5;
    constexpr uint32_t kSlot = 4;             // u32 per ring bin
    uint32_t* s_win = smem + gid * (WS * kSlot);   // cnt[WS][2], then lo[WS][2]
    constexpr uint32_t kLoOff = WS * 2u;      // u32 offset of the lo array
    uint32_t (*s_red)[2][GW] = s_red_all[gid];
    uint32_t* s_state = s_state_all[gid];
    auto group_sync = [&]() {
        if (NG == 1) __syncthreads();
        else asm volatile("bar.sync %0, %1;" ::"r"(1u + gid), "r"((uint32_t)GT) : "memory");
    };
    const uint32_t prev_word = p.epoch > 1 ? (((p.epoch - 1u) << 2) | kTileInit) : 0u;
    for (uint32_t i = threadIdx.x; i < (uint32_t)NG * WS * kSlot / 4u; i += THREADS)
        reinterpret_cast<uint4*>(smem)[i] = make_uint4(0u, 0u, 0u, 0u);
    if (threadIdx.x < NG * NT) s_state_all[threadIdx.x / NT][threadIdx.x % NT] = 0u;
    const auto T = stage_stream_table<kTab>(p, smem + NG * WS * kSlot);
    __syncthreads();

    uint32_t lo_t = 0, act_t = 0;   // resident tiles [lo_t, lo_t+NT); [lo_t, act_t) claimed, to retire
    bool have_window = false;
    // hull of the tiles this CTA's chunks reached (block-uniform registers): a resident
    // tile inside it may hold data and is claimed + retired; outside it is empty
    uint32_t hull_lo = 0xFFFFFFFFu, hull_hi = 0u;
    auto touched = [&](uint32_t t) { return t >= hull_lo && t <= hull_hi; };
    // this thread's in-flight claim (issued after a chunk, resolved before the next barrier)
    uint32_t pend_t = 0xFFFFFFFFu, pend_old = 0u;

    auto resolve_pending = [&]() {
        if (pend_t != 0xFFFFFFFFu) {
            const uint32_t o = claim_outcome(p.tile_flags + pend_t, p.epoch, prev_word, pend_old);
            s_state[pend_t & (NT - 1)] = ((pend_t + 1u) << 2) | o;
            pend_t = 0xFFFFFFFFu;
        }
    };
    // thread k issues the claim CAS of tile t_from + k if it was touched (block-uniform call)
    auto issue_claims = [&](uint32_t t_from, uint32_t t_to) {
        if (tid < t_to - t_from) {
            const uint32_t t = t_from + tid;
            if (touched(t)) {
                pend_t = t;
                pend_old = atomicCAS(p.tile_flags + t, prev_word, (p.epoch << 2) | kTileClaimed);
            }
        }
    };
    // write (won: plain stores) or add (RED) 4 consecutive bins of the ring to HBM and zero them
    // write (won: plain stores) or add (RED) one bin of the ring to HBM and zero it
    auto flush_bin = [&](uint32_t bin, bool won) {
        uint2* sc = reinterpret_cast<uint2*>(s_win + (bin & (WS - 1)) * 2u);
        uint2* sl = reinterpret_cast<uint2*>(s_win + kLoOff + (bin & (WS - 1)) * 2u);
        const uint2 c = *sc, l = *sl;   // {cnt_out, cnt_in}, {lo_out, lo_in}
        *sc = make_uint2(0u, 0u);
        *sl = make_uint2(0u, 0u);
        unsigned long long* g64 = p.bins + (size_t)bin * 4u;
        if (won) {
            ulonglong2* g = reinterpret_cast<ulonglong2*>(g64);
            // evict-first: the kernel never re-reads a written bin (measured 1-2 % faster than .cg)
            __stcs(g, make_ulonglong2(c.x, l.x));
            __stcs(g + 1, make_ulonglong2(c.y, l.y));
        } else {
            // a record with bytes but no count never reaches the ring (counts are >= 1)
            if (c.x) { atomicAdd(g64, (unsigned long long)c.x); if (l.x) atomicAdd(g64 + 1, (unsigned long long)l.x); }
            if (c.y) { atomicAdd(g64 + 2, (unsigned long long)c.y); if (l.y) atomicAdd(g64 + 3, (unsigned long long)l.y); }
        }
    };

    // retire tiles [t_from, t_to) whose claims are resolved in s_state (block-uniform call;
    // must be preceded by a barrier after the claims were resolved)
    auto retire = [&](uint32_t t_from, uint32_t t_to) {
        const uint32_t nt = t_to - t_from;
        if (nt == 0) return;
        // lane k of every warp reads the outcome of tile t_from + k once (nt <= NT <= 32); the
        // warp's ballots give the won / initialised / busy tile masks (group-uniform: every warp
        // reads the same s_state), walked with ffs.  Thread k (warp 0) keeps its tile's outcome
        // for pass 2: after the barrier below, threads already in the next chunk may re-use the
        // slot for a newer claim.
        uint32_t my_o = 0u, o_l = 0u;
        if (lane < nt && touched(t_from + lane)) {
            const uint32_t t = t_from + lane, st = s_state[t & (NT - 1)];
            o_l = ((st >> 2) == t + 1u) ? (st & 3u) : kBusy;
        }
        if (warp == 0u) my_o = o_l;
        const unsigned won_m = __ballot_sync(kFull, o_l == kWon), init_m = __ballot_sync(kFull, o_l == kInit);
        const bool busy = __any_sync(kFull, o_l == kBusy);
        // pass 1a: WON tiles -> one 256-bit store per bin (no per-bin branch; the rare INIT tiles
        // follow in their own loop).  A round covers TPR = GT / 256 tiles: thread tid takes bin
        // tid % 256 of the round's (tid / 256)-th tile.
        {
            static_assert(GT % kTileBins == 0 && GT / kTileBins <= 2, "a round covers 1 or 2 tiles");
            constexpr uint32_t TPR = GT / kTileBins;
            const uint32_t sub = tid / kTileBins, i = tid % kTileBins;
            for (unsigned m = won_m; m;) {
                uint32_t k = (uint32_t)(__ffs(m) - 1);
                m &= m - 1u;
                bool ok = true;
                if (TPR == 2) {   // the round's second tile (if any) goes to threads 256..511
                    const uint32_t k1 = (uint32_t)(__ffs(m) - 1);
                    if (sub) { ok = m != 0u; k = k1; }
                    m &= m - 1u;
                }
                if (ok) {
                    const uint32_t bin = (t_from + k) * kTileBins + i, s = bin & (WS - 1);
                    uint2* sc = reinterpret_cast<uint2*>(s_win + s * 2u);
                    uint2* sl = reinterpret_cast<uint2*>(s_win + kLoOff + s * 2u);
                    const uint2 c = *sc, l = *sl;   // {cnt_out, cnt_in}, {lo_out, lo_in}
                    *sc = make_uint2(0u, 0u);
                    *sl = make_uint2(0u, 0u);
                    st_cs_v4u64(p.bins + (size_t)bin * 4u, c.x, l.x, c.y, l.y);
                }
            }
        }
        // pass 1b: INIT tiles (another CTA initialised them: rare) -> RED.ADD
        for (unsigned m = init_m; m; m &= m - 1u) {
            const uint32_t k = (uint32_t)(__ffs(m) - 1);
            for (uint32_t i = tid; i < kTileBins; i += GT) flush_bin((t_from + k) * kTileBins + i, false);
        }
        group_sync();
        // pass 2: publish WON tiles; wait (holding nothing unreleased) for BUSY ones
        if (tid < nt) {
            const uint32_t t = t_from + tid;
            if (my_o != 0u) {
                const uint32_t o = my_o;
                if (o == kWon) {
                    // the release is cumulative over the group's bin stores ordered before it
                    // by the barrier above (no separate fence)
                    st_release_u32(p.tile_flags + t, (p.epoch << 2) | kTileInit);
                } else if (o == kBusy) {
                    const uint32_t init = (p.epoch << 2) | kTileInit;
                    uint32_t spins = 0;
                    while (ld_acquire_u32(p.tile_flags + t) != init) {
                        __nanosleep(200);
                        if (++spins > kSpinLimit) __trap();
                    }
                }
            }
        }
        if (busy) {
            group_sync();
            for (uint32_t k = 0; k < nt; ++k) {
                const uint32_t t = t_from + k;
                if (!touched(t)) continue;
                const uint32_t st = s_state[t & (NT - 1)];
                if (((st >> 2) == t + 1u) && (st & 3u) != kBusy) continue;
                for (uint32_t i = tid; i < kTileBins; i += GT) flush_bin(t * kTileBins + i, false);
            }
            group_sync();
        }
    };
    // claim synchronously (non-blocking CASes, resolved at once) and retire [t_from, t_to)
    auto claim_and_retire = [&](uint32_t t_from, uint32_t t_to) {
        for (uint32_t base = t_from; base < t_to; base += NT) {
            const uint32_t e = (t_to - base < NT) ? t_to : base + NT;
            issue_claims(base, e);
            resolve_pending();
            group_sync();
            retire(base, e);
        }
    };

    // accumulate (cnt, bytes) of one (bin, dir) into the ring (caller checked residency);
    // returns the high word (bytes >> 32 + the carry out of the low word, mod 2^32) that the
    // caller must add to HBM as hi << 32 (exact mod 2^64)
    auto accumulate = [&](uint32_t bin, uint32_t dir, uint32_t cnt, uint64_t bytes) -> uint32_t {
        uint32_t* s = s_win + (bin & (WS - 1)) * 2u + dir;
        atomicAdd(s, cnt);
        const uint32_t lo = (uint32_t)bytes;
        const uint32_t old = atomicAdd(s + kLoOff, lo);
        return (uint32_t)(bytes >> 32) + ((old + lo < old) ? 1u : 0u);
    };

    // Branch-free accumulate of RPT records: record j is added to its ring slot iff take[j]
    // (predicated shared-memory RED / ATOM, no divergent branch).  The count uses a reduction
    // without a return value, the low word an atomic whose old value gives the exact carry.
    // Adds each taken record's high word (see accumulate) to hi[j].
    const uint32_t win_base = (uint32_t)__cvta_generic_to_shared(s_win);
    // Branch-free: EVERY record issues its two shared atomics, adding 0 when not taken (a
    // predicated atomic in inline asm compiles to BSSY/BRA/BSYNC around each ATOMS -- 4-5
    // instructions per atomic and a reconvergence point; measured in the C2 SASS).  The slot
    // address is always inside the ring (dir & 1), and adding 0 changes nothing.
    auto accumulate_all = [&](const bool (&take)[RPT], const uint32_t (&bin)[RPT], const uint32_t (&dir)[RPT],
                              const uint64_t (&by)[RPT], uint32_t (&hi)[RPT]) {
        uint32_t old[RPT];
#pragma unroll
        for (int j = 0; j < RPT; ++j) {
            const uint32_t a = win_base + ((bin[j] & (WS - 1)) * 2u + (dir[j] & 1u)) * 4u;
            const uint32_t lo = take[j] ? (uint32_t)by[j] : 0u;
            asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a), "r"(take[j] ? 1u : 0u) : "memory");
            asm volatile("atom.shared.add.u32 %0, [%1+%3], %2;" : "=r"(old[j]) : "r"(a), "r"(lo), "n"(kLoOff * 4u) : "memory");
        }
#pragma unroll
        for (int j = 0; j < RPT; ++j) {
            const uint32_t lo = (uint32_t)by[j];
            const uint32_t h = (uint32_t)(by[j] >> 32) + ((old[j] + lo < old[j]) ? 1u : 0u);
            hi[j] += take[j] ? h : 0u;
        }
    };
    auto accumulate_n = [&](const bool (&take)[RPT], const uint32_t (&bin)[RPT], const uint32_t (&dir)[RPT],
                            const uint64_t (&by)[RPT], uint32_t (&hi)[RPT]) {
        uint32_t old[RPT];
#pragma unroll
        for (int j = 0; j < RPT; ++j) {
            const uint32_t a = win_base + ((bin[j] & (WS - 1)) * 2u + dir[j]) * 4u;
            old[j] = smem_count_and_add_lo<kLoOff * 4u>(a, take[j], (uint32_t)by[j]);
        }
#pragma unroll
        for (int j = 0; j < RPT; ++j) {
            const uint32_t lo = (uint32_t)by[j];
            const uint32_t h = (uint32_t)(by[j] >> 32) + ((old[j] + lo < old[j]) ? 1u : 0u);
            hi[j] += take[j] ? h : 0u;
        }
    };

    // Contiguous ranges of 4-record groups (virtual index space) are handed out
    // dynamically (one atomic per range, counter zeroed before each launch) so that
    // groups that finish early take more.
    const uint64_t ngroups = (p.nv + 3) / 4;
    const uint64_t nranges = (uint64_t)p.n_ranges;
    __shared__ uint64_t s_range[NG];
    __shared__ unsigned long long s_wtot[kSmemTot ? NW : 1][12];   // per-warp totals (RPT == 2)
    if (kSmemTot) {
        for (uint32_t i = threadIdx.x; i < (uint32_t)NW * 12u; i += THREADS) (&s_wtot[0][0])[i] = 0ull;
    }
    WarpTotals tot;
    tot.zero();
    uint32_t gmin = 0xFFFFFFFFu, gmax = 0u;   // extent of this group's binned records (uniform)
    for (;;) {
    if (tid == 0) s_range[gid] = atomicAdd(p.range_counter, 1u);
    group_sync();
    const uint64_t range = s_range[gid];
    if (range >= nranges) break;
    // this range in virtual records [r0, r1) (a multiple of 4 apart)
    const uint64_t r0 = (ngroups * range / nranges) * 4, r1 = (ngroups * (range + 1) / nranges) * 4;
    lo_t = 0; act_t = 0; have_window = false; hull_lo = 0xFFFFFFFFu; hull_hi = 0u;

    // Chunk k of the range covers virtual records [r0 + k CH, r0 + (k+1) CH); all per-chunk
    // bounds are precomputed per range as 32-bit chunk indices (no 64-bit compares per chunk).
    constexpr uint32_t CH = (uint32_t)GT * RPT;   // records per chunk
    const uint32_t span = (uint32_t)(r1 - r0);     // < 2^31 (launch_hist_stream)
    const uint32_t nch = (span + CH - 1u) / CH;
    const uint32_t off = tid * (uint32_t)RPT;      // this thread's first record in a chunk
    // chunks where this thread has records: r0 + k CH + off < r1
    const uint32_t nhave = span > off ? (span - off + CH - 1u) / CH : 0u;
    // chunks whose every record is valid (not the batch's ragged first/last 4-record group)
    const uint64_t full_lo = (p.head != 0u) ? 4u : 0u;
    const uint64_t full_hi = (r1 > p.nv) ? r1 - 4 : r1;
    const uint32_t kf0 = r0 < full_lo ? 1u : 0u;
    const uint32_t kf1 = (uint32_t)((full_hi - r0) / CH);
    // chunks where this thread's 4 records are one 16-byte group of every column (128-bit loads)
    const uint64_t g0 = r0 + off;
    const uint32_t kv0 = g0 < p.head ? 1u : 0u;
    const uint32_t kv1 = p.nv >= g0 + RPT ? (uint32_t)((p.nv - g0 - RPT) / CH) + 1u : 0u;
    // column pointers of this thread's group in chunk 0 (may point before the column: only
    // dereferenced for chunks in [kv0, kv1))
    const int64_t e0 = (int64_t)g0 - (int64_t)p.head;
    const uint64_t* ts_b = p.ts + e0;
    const uint32_t* src_b = p.src + e0;
    const uint32_t* dst_b = p.dst + e0;
    const uint64_t* by_b = p.bytes + e0;
    auto load_chunk = [&](uint32_t k, Rec& r) {
        if constexpr (RPT == 4) {
            if (k >= kv0 && k < kv1) {
                const uint32_t a = k * CH;
                const ulonglong2 t0 = ldcs_v2u64(ts_b + a), t1 = ldcs_v2u64(ts_b + a + 2);
                const uint4 sv = ldcs_v4u32(src_b + a), dv = ldcs_v4u32(dst_b + a);
                const ulonglong2 b0 = ldcs_v2u64(by_b + a), b1 = ldcs_v2u64(by_b + a + 2);
                r.ts[0] = t0.x; r.ts[1] = t0.y; r.ts[2] = t1.x; r.ts[3] = t1.y;
                r.src[0] = sv.x; r.src[1] = sv.y; r.src[2] = sv.z; r.src[3] = sv.w;
                r.dst[0] = dv.x; r.dst[1] = dv.y; r.dst[2] = dv.z; r.dst[3] = dv.w;
                r.by[0] = b0.x; r.by[1] = b0.y; r.by[2] = b1.x; r.by[3] = b1.y;
                return;
            }
        }
        loadN<RPT>(p, g0 + (uint64_t)k * CH, r);
    };
    Rec cur, nxt;
    if (nhave) load_chunk(0u, cur);
    uint32_t parity = 0;

    for (uint32_t k = 0; k < nch; ++k, parity ^= 1u) {
        const uint64_t my_v = g0 + (uint64_t)k * CH;   // this thread's first record (general path only)
        const bool have = k < nhave;
        // every record of the chunk valid (all but the batch's ragged ends): no per-record checks
        const bool full = k >= kf0 && k < kf1;
        const bool tags_on = p.tags != nullptr;
        if (k + 1u < nhave) load_chunk(k + 1u, nxt);   // prefetch into registers

        // ---- a3-a5: classify and map this chunk (the claims issued last chunk resolve meanwhile)
        // dir4[j]: 0 / 1 = the record is binned in that direction and still to be accumulated,
        // 4 | dir = accumulated before the barrier, 3 = not binned (no per-record bool arrays:
        // they would live in a register as bit fields across the barrier)
        uint32_t bin4[RPT], dir4[RPT];
        uint32_t tag4 = 0, bmin = 0xFFFFFFFFu, bmax = 0u;
        WarpTotals ctot;   // this chunk's records (RPT == 2: reduced into shared memory below)
        if (kSmemTot) ctot.zero();
        WarpTotals& tt = kSmemTot ? ctot : tot;
        uint32_t addr[2 * RPT], in8[2 * RPT];
#pragma unroll
        for (int j = 0; j < RPT; ++j) { addr[2 * j] = cur.src[j]; addr[2 * j + 1] = cur.dst[j]; }
        member_batch_tab<kTab, 2 * RPT>(addr, in8, T);
        // kFull: every record of the chunk is valid (whole chunk in the batch, no watchlist),
        // so the per-record validity tests and masks drop out of the common path
        auto classify = [&](auto kFullTag) {
            constexpr bool kAllValid = decltype(kFullTag)::value;
#pragma unroll
            for (int j = 0; j < RPT; ++j) {
                const bool valid = kAllValid || ((full || (have && vvalid(p, my_v + j))) &&
                                                 (!kWatch || watched(cur.src[j], p) || watched(cur.dst[j], p)));
                const uint32_t cell = in8[2 * j] * 2u + in8[2 * j + 1];
                const uint32_t dir = (p.lut >> (cell * 2u)) & 3u;
                uint32_t bin = 0;
                bool inw;
                if (kW1) {   // 1 ms bins: the key is the offset itself
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
                if (!kAllValid && tags_on)   // tags: the general path only
                    tag4 |= (in8[2 * j] | (in8[2 * j + 1] << 1) | ((inw ? 0u : 1u) << 2)) << (8 * j);
                if (binned) { bmin = min(bmin, bin); bmax = max(bmax, bin); }
                if (kAllValid) tt.add_valid(cell, directed && !inw, dir, cur.by[j]);
                else tt.add(valid, cell, directed && !inw, dir, cur.by[j]);
            }
        };
        if (full && !kWatch && !tags_on) classify(std::true_type{});   // tags: the general path
        else classify(std::false_type{});
        if (tags_on && have) {
            if (RPT == 4) store_tags4(p, my_v, tag4);
            else for (int j = 0; j < RPT; ++j) if (vvalid(p, my_v + j)) p.tags[my_v + j - p.head] = (uint8_t)(tag4 >> (8 * j));
        }
        if (kSmemTot) {   // warp-reduce this chunk's totals into the warp's shared slots
            const unsigned long long cT = __reduce_add_sync(kFull, ctot.cT), cS = __reduce_add_sync(kFull, ctot.cS);
            const unsigned long long cD = __reduce_add_sync(kFull, ctot.cD), cSD = __reduce_add_sync(kFull, ctot.cSD);
            const unsigned long long bT = warp_sum_u64(ctot.bT), bS = warp_sum_u64(ctot.bS);
            const unsigned long long bD = warp_sum_u64(ctot.bD), bSD = warp_sum_u64(ctot.bSD);
            unsigned long long o[4] = {0ull, 0ull, 0ull, 0ull};
            if (__any_sync(kFull, (ctot.oc[0] | ctot.oc[1]) != 0u)) {
                o[0] = __reduce_add_sync(kFull, ctot.oc[0]); o[1] = __reduce_add_sync(kFull, ctot.oc[1]);
                o[2] = warp_sum_u64(ctot.ob[0]); o[3] = warp_sum_u64(ctot.ob[1]);
            }
            if (lane == 0) {
                const uint32_t w = threadIdx.x >> 5;
                s_wtot[w][0] += cT - cS - cD + cSD; s_wtot[w][1] += cD - cSD; s_wtot[w][2] += cS - cSD; s_wtot[w][3] += cSD;
                s_wtot[w][4] += bT - bS - bD + bSD; s_wtot[w][5] += bD - bSD; s_wtot[w][6] += bS - bSD; s_wtot[w][7] += bSD;
                s_wtot[w][8] += o[0]; s_wtot[w][9] += o[1]; s_wtot[w][10] += o[2]; s_wtot[w][11] += o[3];
            }
        }
        // Accumulate before the barrier every record whose tile is resident ([lo_t, lo_t + NT),
        // including the tiles claimed after the previous chunk, which retire right after the
        // barrier); only records outside the ring are left for after the retire.
        uint32_t hi4[RPT];   // high words owed to HBM (added after the barrier)
#pragma unroll
        for (int j = 0; j < RPT; ++j) hi4[j] = 0u;
        if (!kAgg && have_window) {
            bool take[RPT];
#pragma unroll
            for (int j = 0; j < RPT; ++j) take[j] = dir4[j] < 2u && bin4[j] / kTileBins - lo_t < NT;
            accumulate_all(take, bin4, dir4, cur.by, hi4);
#pragma unroll
            for (int j = 0; j < RPT; ++j) dir4[j] |= take[j] ? 4u : 0u;
        }
        bmin = __reduce_min_sync(kFull, bmin);
        bmax = __reduce_max_sync(kFull, bmax);
        if (lane == 0) { s_red[parity][0][warp] = bmin; s_red[parity][1][warp] = bmax; }
        resolve_pending();
        group_sync();
        bmin = 0xFFFFFFFFu;
        bmax = 0u;
        if constexpr (GW % 4 == 0) {   // 128-bit loads: GW/4 per array instead of GW scalar loads
#pragma unroll
            for (int w = 0; w < GW; w += 4) {
                const uint4 a = *reinterpret_cast<const uint4*>(&s_red[parity][0][w]);
                const uint4 b = *reinterpret_cast<const uint4*>(&s_red[parity][1][w]);
                bmin = min(bmin, min(min(a.x, a.y), min(a.z, a.w)));
                bmax = max(bmax, max(max(b.x, b.y), max(b.z, b.w)));
            }
        } else {
            for (int w = 0; w < GW; ++w) { bmin = min(bmin, s_red[parity][0][w]); bmax = max(bmax, s_red[parity][1][w]); }
        }
        const bool any = bmin <= bmax;
        const uint32_t bmin_t = bmin / kTileBins, bmax_t = bmax / kTileBins;

        // every tile this chunk reaches at or above the claim boundary joins the hull now,
        // before any retire: tiles that received pre-barrier accumulation must be seen as
        // touched by an emergency retire below (tiles in [lo_t, act_t) were claimed already)
        if (any) { gmin = min(gmin, bmin); gmax = max(gmax, bmax); }
        if (any && have_window) {
            hull_lo = min(hull_lo, bmin_t > act_t ? bmin_t : act_t);
            hull_hi = max(hull_hi, bmax_t);
        }

        // ---- a6 (retire): tiles claimed after the previous chunk
        retire(lo_t, act_t);
        lo_t = act_t;
        if (any) {
            if (!have_window) {
                have_window = true;
                lo_t = act_t = (bmax_t - bmin_t >= NT) ? bmax_t - NT + 1u : bmin_t;
                hull_lo = min(hull_lo, bmin_t > lo_t ? bmin_t : lo_t);
                hull_hi = max(hull_hi, bmax_t);
            } else if (bmax_t >= lo_t + NT) {   // the chunk reaches past the ring: retire now
                const uint32_t nlo = bmax_t - NT + 1u;
                claim_and_retire(lo_t, (nlo - lo_t < NT) ? nlo : lo_t + NT);
                lo_t = act_t = nlo;
            }
        }
        const bool key32 = p.nbins < 0x40000000u;   // keys 2*bin+dir stay below the lane sentinels

        // ---- a6 (accumulate): reduce the chunk into the ring
        // the whole chunk inside the ring (the common case): no per-record residency/spill checks
        const bool all_in = any && bmin_t >= lo_t && bmax_t - lo_t < NT;
        if (!kAgg && all_in) {
            bool rest[RPT];
            bool any_rest = false;
#pragma unroll
            for (int j = 0; j < RPT; ++j) { rest[j] = dir4[j] < 2u; any_rest |= rest[j]; }
            if (__any_sync(kFull, any_rest)) accumulate_n(rest, bin4, dir4, cur.by, hi4);
            bool any_hi = false;
#pragma unroll
            for (int j = 0; j < RPT; ++j) any_hi |= hi4[j] != 0u;
            if (__any_sync(kFull, any_hi)) {
#pragma unroll
                for (int j = 0; j < RPT; ++j)
                    if (__any_sync(kFull, hi4[j] != 0u))
                        spill_warp(p, hi4[j] != 0u, bin4[j], dir4[j] & 1u, 0u, (uint64_t)hi4[j] << 32);
            }
        } else
#pragma unroll
        for (int j = 0; j < RPT; ++j) {
            const bool b = dir4[j] < 2u;
            bool act = b;
            uint32_t cnt = 1u;
            uint64_t byt = cur.by[j];
            // warp aggregation of equal (bin, dir) keys (hot bins, bursts): only when a
            // cheap neighbour test finds a duplicate in the warp (records of one slot are
            // RPT apart in stream order, so hot keys show up in adjacent lanes)
            bool try_agg = false;
            if (kAgg) {
                const uint32_t k32 = b ? ((bin4[j] << 1) | dir4[j]) : 0xFFFFFFFFu - lane;
                const uint32_t kp = __shfl_up_sync(kFull, k32, 1);
                try_agg = __any_sync(kFull, b && lane > 0u && kp == k32);
            }
            if (try_agg) {
                unsigned m;
                if (key32) {
                    const uint32_t key = b ? ((bin4[j] << 1) | dir4[j]) : 0xFFFFFFFFu - lane;
                    m = __match_any_sync(kFull, key);
                } else {
                    const unsigned long long key = b ? (((unsigned long long)bin4[j] << 1) | dir4[j]) : ~0ull - lane;
                    m = __match_any_sync(kFull, key);
                }
                const bool grouped = b && __popc(m) > 1;
                if (__any_sync(kFull, grouped)) {
                    const bool leader = lane == (unsigned)(__ffs(m) - 1);
                    unsigned leaders = __ballot_sync(kFull, grouped && leader);
                    while (leaders) {
                        const int l = __ffs(leaders) - 1;
                        leaders &= leaders - 1;
                        const unsigned g = __shfl_sync(kFull, m, l);
                        const uint64_t sum = warp_sum_u64(((g >> lane) & 1u) ? cur.by[j] : 0ull);
                        if (lane == (unsigned)l) { byt = sum; cnt = (uint32_t)__popc(g); }
                    }
                    act = b && (!grouped || leader);
                }
            }
            const bool in_ring = act && (bin4[j] / kTileBins - lo_t < NT);
            // high word owed by this record (accumulated now, or before the barrier)
            const uint32_t hv = hi4[j] + (in_ring ? accumulate(bin4[j], dir4[j], cnt, byt) : 0u);
            const bool out = act && !in_ring;
            if (__any_sync(kFull, out || hv != 0u))
                spill_warp(p, out || hv != 0u, bin4[j], dir4[j] & 1u, out ? cnt : 0u, out ? byt : ((uint64_t)hv << 32));
        }
        cur = nxt;

        // ---- claim the tiles that fall out of the history kept below this chunk
        if (any) {
            const uint32_t keep = (bmax_t >= kHist) ? bmax_t - kHist : 0u;
            uint32_t nact = bmin_t < keep ? bmin_t : keep;
            if (nact < act_t) nact = act_t;
            if (nact > lo_t + NT) nact = lo_t + NT;
            issue_claims(act_t, nact);
            act_t = nact;
        }
    }

    // retire everything still resident
    resolve_pending();
    group_sync();
    if (have_window) {
        retire(lo_t, act_t);
        claim_and_retire(act_t, lo_t + NT);
    }
    }   // ranges
    if (tid == 0 && gmin <= gmax) { atomicMin(p.touched, gmin); atomicMax(p.touched + 1, gmax); }
    __syncthreads();
    if (kSmemTot) {
        if (threadIdx.x < 12) {
            unsigned long long acc = 0;
            for (int w = 0; w < NW; ++w) acc += s_wtot[w][threadIdx.x];
            if (acc) atomicAdd(p.totals + threadIdx.x, acc);
        }
    } else {
        flush_totals(tot, p.totals, s_tot);
    }
}

// ---------------------------------------------------------------- launch
namespace {
// ring layouts of the same 192 KB: one group with an 8192-bin ring (sparse input: a
// chunk spans many ms) or two independent groups with 4096-bin rings (dense input:
// one group's barrier/retire phase overlaps the other's loads and lookups)
constexpr int kRingBins1 = 8192;
constexpr int kRingBins2 = 4096;
}  // namespace

// 512 threads x 4 records per thread; one group (8192-bin ring) or two (4096-bin rings).
// (The kernel also supports 1024 threads x 2 records, measured 23 % slower: not instantiated.)
#define SINET_STREAM_KERNEL(G, A, W, S, WL) \
    k_hist_stream<512, G, (G == 1 ? kRingBins1 : kRingBins2), 4, A, W, S, WL>
constexpr size_t kRingSmem = (size_t)kRingBins1 * 4u * 4u;   // 128 KB: 4 u32 per bin

cudaError_t setup_hist_stream() {
    const int mx = (int)(kRingSmem + kStreamTableSmem);
    cudaError_t e;
#define SET(G, A, W, S, WL)                                                                                 \
    e = cudaFuncSetAttribute(SINET_STREAM_KERNEL(G, A, W, S, WL), cudaFuncAttributeMaxDynamicSharedMemorySize, mx); \
    if (e != cudaSuccess) return e;
#define SET4(G, S, WL) SET(G, true, true, S, WL) SET(G, true, false, S, WL) SET(G, false, true, S, WL) SET(G, false, false, S, WL)
#define SETT(G, WL) SET4(G, kTabByte, WL) SET4(G, kTabPacked, WL) SET4(G, kTabPackedNoL2, WL) SET4(G, kTabGlobal, WL)
    SETT(1, false) SETT(2, false) SETT(1, true) SETT(2, true)
#undef SETT
#undef SET4
#undef SET
    return cudaSuccess;
}

int stream_groups_for(const KernelParams& p) {
    if (p.stream_groups == 1 || p.stream_groups == 2) return (int)p.stream_groups;
    // records per bin of the window: >= 3/4 -> two groups (a 1024-record chunk spans few tiles)
    return (p.n * 4 >= (uint64_t)p.nbins * 3) ? 2 : 1;
}

cudaError_t launch_hist_stream(const KernelParams& p, int sm_count, bool agg, cudaStream_t st) {
    static_assert(kRingBins1 == 2 * kRingBins2, "both layouts use the same shared memory");
    const int tab = stream_table_mode(p.has_bytes != 0u, p.nbnd, p.n_mixed, p.tab_mode);
    const size_t sm = kRingSmem + stream_table_bytes(tab, p.nbnd, p.n_mixed);
    const uint64_t chunks = (p.nv / 4 + 511) / 512;
    const int grid = (int)((chunks < (uint64_t)sm_count) ? (chunks ? chunks : 1) : (uint64_t)sm_count);
    const bool w1 = p.width == 1u;
    const int g = stream_groups_for(p);
    KernelParams q = p;
    // record ranges handed out dynamically, a whole number per group (a partial last wave
    // leaves most groups idle: C2 with 625 ranges 1.72 ms vs 592 = 2 per group 1.36 ms), each
    // about kRangeRecords long: long ranges save window warm-up and drain (the boundary tiles
    // of a range are shared with its neighbours: RED instead of plain stores), short ones
    // balance bursty stretches.  Measured ranges per group (C2 100 M / C4 1.6 B bursty / C5
    // 400 M, ms): 2 -> 1.211 / - / -, 4 -> 1.217 / 12.87 / 4.78, 8 -> 1.246 / 12.53 / 4.81,
    // 16 -> - / 12.25 / 4.93, 32 -> - / 12.15 / -; C2 at 1 per group (338 k) 1.200, C3 1.2 B
    // at 10 / 20 per group 9.065 / 9.121: uniform input prefers ~300-400 k records per range,
    // bursty ~170 k (within 1 %): 300 k.
    constexpr uint64_t kRangeRecords = 300000;
    const uint64_t groups_total = (uint64_t)grid * (uint64_t)g;
    const uint64_t rpg = p.ranges_per_group ? p.ranges_per_group
                                            : (p.nv + groups_total * kRangeRecords / 2) / (groups_total * kRangeRecords);
    const uint64_t per = groups_total * (rpg ? rpg : 1u);
    const uint64_t max_r = p.nv / (4u * 512u * 4u) + 1u;
    q.n_ranges = (uint32_t)(per < max_r ? per : max_r);
    // a range spans < 2^31 records (the kernel indexes chunks of a range in 32 bits)
    if ((uint64_t)q.n_ranges < (p.nv >> 30) + 1u) q.n_ranges = (uint32_t)((p.nv >> 30) + 1u);
    cudaError_t e = cudaMemsetAsync(p.range_counter, 0, 8, st);
    if (e != cudaSuccess) return e;
#define LAUNCH(G, S, WL)                                                                                \
    if (agg && w1) SINET_STREAM_KERNEL(G, true, true, S, WL)<<<grid, 512, sm, st>>>(q);                  \
    else if (agg) SINET_STREAM_KERNEL(G, true, false, S, WL)<<<grid, 512, sm, st>>>(q);                  \
    else if (w1) SINET_STREAM_KERNEL(G, false, true, S, WL)<<<grid, 512, sm, st>>>(q);                   \
    else SINET_STREAM_KERNEL(G, false, false, S, WL)<<<grid, 512, sm, st>>>(q);
#define LAUNCH_G(S, WL) if (g == 2) { LAUNCH(2, S, WL) } else { LAUNCH(1, S, WL) }
#define LAUNCH_T(WL) switch (tab) {                              \
        case kTabByte: LAUNCH_G(kTabByte, WL) break;                  \
        case kTabPacked: LAUNCH_G(kTabPacked, WL) break;              \
        case kTabPackedNoL2: LAUNCH_G(kTabPackedNoL2, WL) break;      \
        default: LAUNCH_G(kTabGlobal, WL) break;                      \
    }
    if (p.wn) { LAUNCH_T(true) } else { LAUNCH_T(false) }
#undef LAUNCH_T
#undef LAUNCH_G
#undef LAUNCH
    return cudaGetLastError();
}

}  // namespace sinet
