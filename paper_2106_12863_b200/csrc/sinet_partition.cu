// Unordered input (strategy SHUFFLED with caller scratch): partition, then bin.
//
// The paper tiles its map-reduce because "a whole problem [that] does not fit in the cache"
// must be reduced piece by piece (§4).  For records in no particular time order
// the pieces are made explicitly: the records are radix-partitioned by time into buckets of
// 8192 ms bins (two passes of 7 bits: coarse buckets of 2^20 bins, then fine buckets), and
// every fine bucket is then reduced in shared memory and written to HBM once (SURVEY §8(d)
// strategy S4; §2.4 K2/K3).  Per sub-batch of at most `cap` records:
//
//   k_part_count  ts only (8 B/record): records per fine bucket (in-window records; the
//                 window test is Map, §4.1)
//   k_part_plan   one CTA: exclusive scans -> fine/coarse bucket bases, write cursors, the
//                 work units of the next passes
//   k_part_scatter  the full records (24 B/record): Alg. 1 membership of src and dst
//                 (P:L160-163), direction, Map, side totals and tags -- as the stream kernels
//                 -- then a block-local counting sort of 2048 records by coarse bucket and one
//                 write of each run (8 B bytes + 4 B key per record, key = bin | dir << 27 |
//                 binned << 28; NEITHER / filtered records stay as null keys)
//   k_part_fine   the same counting sort of each coarse bucket by fine bucket (12 B in, 12 B out)
//   k_part_bin    one fine bucket (or a part of a big one) at a time: count, low and high
//                 32-bit words of the byte sums per (bin, dir) in shared memory (exact mod 2^64),
//                 then each 256-bin tile with data goes to HBM through the tile protocol
//                 (sinet_tiles.cuh): plain stores if claimed first, RED.ADD otherwise.
// Algorithmic DRAM bytes: 24 + 8 + 4*12 B per record + 32 B per bin.
#include "sinet_device.cuh"
#include "sinet_kernels.h"
#include "sinet_tiles.cuh"

namespace sinet {

namespace {
constexpr int kPT = 512;                 // threads of the partition / bin kernels
constexpr uint32_t kPChunk = 2048;       // records per block-local counting sort (4 per thread)
constexpr uint32_t kFineShift = 13;      // 8192 bins per fine bucket
constexpr uint32_t kFineBins = 1u << kFineShift;
constexpr uint32_t kDigit = 7;           // 128 fine buckets per coarse bucket
constexpr uint32_t kPartRecords = 1u << 16;   // records per unit of the bin pass (big buckets split)
constexpr uint32_t kKeyDir = 1u << 27, kKeyBinned = 1u << 28, kBinMask = kKeyDir - 1u;
}  // namespace

// ---------------------------------------------------------------- scratch layout
PartLayout part_layout(uint64_t cap, uint32_t nbins) {
    PartLayout L{};
    L.cap = cap;
    L.nf = (nbins + kFineBins - 1) / kFineBins;
    L.nc = (L.nf + (1u << kDigit) - 1) >> kDigit;
    size_t o = 0;
    auto take = [&](size_t bytes) { size_t r = o; o = (o + bytes + 255) & ~(size_t)255; return r; };
    L.by_a = take(cap * 8);
    L.by_b = take(cap * 8);
    L.key_a = take(cap * 4);
    L.key_b = take(cap * 4);
    L.fine_cnt = take((size_t)kMaxFine * 4);
    L.fine_base = take((size_t)(kMaxFine + 1) * 4);
    L.fine_cur = take((size_t)kMaxFine * 4);
    L.unit_base = take((size_t)(kMaxFine + 1) * 4);
    L.coarse_base = take((size_t)(kMaxCoarse + 1) * 4);
    L.coarse_cur = take((size_t)kMaxCoarse * 4);
    L.cunit_base = take((size_t)(kMaxCoarse + 1) * 4);
    L.counters = take(64);
    L.total = o;
    return L;
}

struct PartArgs {
    unsigned long long* by_a;
    unsigned long long* by_b;
    uint32_t* key_a;
    uint32_t* key_b;
    uint32_t* fine_cnt;
    uint32_t* fine_base;
    uint32_t* fine_cur;
    uint32_t* unit_base;
    uint32_t* coarse_base;
    uint32_t* coarse_cur;
    uint32_t* cunit_base;
    uint32_t* counters;       // [0] fine-pass unit ticket, [1] bin-pass unit ticket
    uint32_t nf, nc;
};

// ---------------------------------------------------------------- pass 0: fine bucket sizes
__global__ void __launch_bounds__(kPT) k_part_count(KernelParams p, PartArgs a) {
    extern __shared__ uint32_t s_cnt[];   // [nf]
    for (uint32_t i = threadIdx.x; i < a.nf; i += kPT) s_cnt[i] = 0u;
    __syncthreads();
    const uint64_t stride = (uint64_t)gridDim.x * kPT * 4u;
    for (uint64_t v = ((uint64_t)blockIdx.x * kPT + threadIdx.x) * 4u; v < p.nv; v += stride) {
        uint64_t ts[4];
        if (v >= p.head && v + 4 <= p.nv) {
            const ulonglong2 t0 = ldcs_v2u64(p.ts + (v - p.head)), t1 = ldcs_v2u64(p.ts + (v - p.head) + 2);
            ts[0] = t0.x; ts[1] = t0.y; ts[2] = t1.x; ts[3] = t1.y;
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) ts[j] = vvalid(p, v + j) ? p.ts[v + j - p.head] : p.start - 1u;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            uint32_t bin;
            if (map_bin(ts[j], p, bin)) atomicAdd(&s_cnt[bin >> kFineShift], 1u);
        }
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < a.nf; i += kPT)
        if (s_cnt[i]) atomicAdd(&a.fine_cnt[i], s_cnt[i]);
}

// ---------------------------------------------------------------- plan (one CTA of 1024)
// block-wide exclusive scan of per-thread sums (1024 threads)
__device__ uint32_t block_excl_scan(uint32_t v, uint32_t* s_warp, uint32_t* total) {
    const uint32_t lane = threadIdx.x & 31u, w = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, x, d);
        if (lane >= (uint32_t)d) x += y;
    }
    if (lane == 31) s_warp[w] = x;
    __syncthreads();
    if (w == 0) {
        uint32_t s = s_warp[lane];
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t y = __shfl_up_sync(kFull, s, d);
            if (lane >= (uint32_t)d) s += y;
        }
        s_warp[lane] = s;   // inclusive per-warp prefix
    }
    __syncthreads();
    const uint32_t before = (w ? s_warp[w - 1] : 0u) + x - v;
    *total = s_warp[31];
    __syncthreads();
    return before;
}

__global__ void __launch_bounds__(1024) k_part_plan(PartArgs a) {
    __shared__ uint32_t s_warp[32];
    constexpr uint32_t kPer = kMaxFine / 1024;   // fine buckets per thread
    const uint32_t t = threadIdx.x;
    uint32_t c[kPer], u[kPer], sc = 0, su = 0;
#pragma unroll
    for (uint32_t k = 0; k < kPer; ++k) {
        const uint32_t f = t * kPer + k;
        c[k] = f < a.nf ? a.fine_cnt[f] : 0u;
        u[k] = (c[k] + kPartRecords - 1) / kPartRecords;
        sc += c[k];
        su += u[k];
    }
    uint32_t tot_c, tot_u;
    uint32_t bc = block_excl_scan(sc, s_warp, &tot_c);
    uint32_t bu = block_excl_scan(su, s_warp, &tot_u);
#pragma unroll
    for (uint32_t k = 0; k < kPer; ++k) {
        const uint32_t f = t * kPer + k;
        if (f < a.nf) {
            a.fine_base[f] = bc;
            a.fine_cur[f] = bc;
            a.unit_base[f] = bu;
            if ((f & ((1u << kDigit) - 1u)) == 0u) { a.coarse_base[f >> kDigit] = bc; a.coarse_cur[f >> kDigit] = bc; }
        }
        bc += c[k];
        bu += u[k];
    }
    if (t == 0) {
        a.fine_base[a.nf] = tot_c;
        a.unit_base[a.nf] = tot_u;
        a.coarse_base[a.nc] = tot_c;
        a.counters[0] = 0u;
        a.counters[1] = 0u;
    }
    __syncthreads();
    // units of the fine pass: chunks of kPChunk records inside each coarse bucket
    if (t < 32) {
        uint32_t carry = 0;
        for (uint32_t c0 = 0; c0 < a.nc; c0 += 32) {
            const uint32_t ci = c0 + t;
            const uint32_t n = ci < a.nc ? a.coarse_base[ci + 1 < a.nc ? ci + 1 : a.nc] - a.coarse_base[ci] : 0u;
            const uint32_t ch = (n + kPChunk - 1) / kPChunk;
            uint32_t x = ch;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t y = __shfl_up_sync(kFull, x, d);
                if (t >= (uint32_t)d) x += y;
            }
            if (ci < a.nc) a.cunit_base[ci] = carry + x - ch;
            carry += __shfl_sync(kFull, x, 31);
        }
        if (t == 0) a.cunit_base[a.nc] = carry;
    }
}

// ---------------------------------------------------------------- block-local counting sort
// 2048 records (4 per thread) with digits in [0, 128): returns nothing; writes the records
// to dst at cursor[digit] (reserved with one atomic per digit present), runs contiguous.
struct SortSmem {
    uint32_t cnt[128];
    uint32_t off[128];
    uint32_t gpos[128];
    uint32_t key[kPChunk];
    unsigned long long by[kPChunk];
};

__device__ __forceinline__ void sort_and_write(SortSmem& S, const uint32_t (&dig)[4], const uint32_t (&key)[4],
                                               const uint64_t (&by)[4], const bool (&has)[4], uint32_t* cursor,
                                               uint32_t digit_base, uint32_t* key_out, unsigned long long* by_out,
                                               uint32_t shift) {
    const uint32_t t = threadIdx.x;
    if (t < 128) S.cnt[t] = 0u;
    __syncthreads();
    uint32_t rank[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) rank[j] = has[j] ? atomicAdd(&S.cnt[dig[j]], 1u) : 0u;
    __syncthreads();
    if (t < 32) {   // exclusive scan of the 128 counters (4 per lane) + reservations
        uint32_t c4[4], s = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) { c4[k] = S.cnt[t * 4 + k]; s += c4[k]; }
        uint32_t x = s;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t y = __shfl_up_sync(kFull, x, d);
            if (t >= (uint32_t)d) x += y;
        }
        uint32_t o = x - s;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            S.off[t * 4 + k] = o;
            S.gpos[t * 4 + k] = c4[k] ? atomicAdd(cursor + digit_base + t * 4 + k, c4[k]) : 0u;
            o += c4[k];
        }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 4; ++j)
        if (has[j]) {
            const uint32_t q = S.off[dig[j]] + rank[j];
            S.key[q] = key[j];
            S.by[q] = by[j];
        }
    __syncthreads();
    const uint32_t n = S.off[127] + S.cnt[127];
    for (uint32_t q = t; q < n; q += kPT) {
        const uint32_t k = S.key[q];
        const uint32_t d = ((k & kBinMask) >> shift) & 127u;
        const uint32_t g = S.gpos[d] + (q - S.off[d]);
        key_out[g] = k;
        by_out[g] = S.by[q];
    }
    __syncthreads();
}

// ---------------------------------------------------------------- pass 1: classify + coarse partition
template <int kTab, bool kW1, bool kWatch>
__global__ void __launch_bounds__(kPT, 1) k_part_scatter(KernelParams p, PartArgs a) {
    extern __shared__ __align__(16) uint32_t smem[];
    __shared__ SortSmem S;
    __shared__ unsigned long long s_tot[16 * 12];
    const auto T = stage_stream_table<kTab>(p, smem);
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31u;
    WarpTotals tot;
    tot.zero();
    uint32_t gmin = 0xFFFFFFFFu, gmax = 0u;
    const bool tags_on = p.tags != nullptr;
    // the next chunk's records are loaded into registers while this one is sorted and written
    const uint64_t stride = (uint64_t)gridDim.x * kPChunk;
    Rec4 nxt;
    auto load_chunk = [&](uint64_t cb, Rec4& r) {
        const uint64_t v = cb + threadIdx.x * 4u;
        if (v < p.nv) load4(p, v, r);
        else { for (int j = 0; j < 4; ++j) { r.ts[j] = 0; r.src[j] = r.dst[j] = 0; r.by[j] = 0; } }
    };
    if ((uint64_t)blockIdx.x * kPChunk < p.nv) load_chunk((uint64_t)blockIdx.x * kPChunk, nxt);
    for (uint64_t cb = (uint64_t)blockIdx.x * kPChunk; cb < p.nv; cb += stride) {
        const uint64_t my_v = cb + threadIdx.x * 4u;
        const Rec4 r = nxt;
        if (cb + stride < p.nv) load_chunk(cb + stride, nxt);
        uint32_t addr[8], in8[8];
#pragma unroll
        for (int j = 0; j < 4; ++j) { addr[2 * j] = r.src[j]; addr[2 * j + 1] = r.dst[j]; }
        member_batch_tab<kTab, 8>(addr, in8, T);
        uint32_t dig[4], key[4], tag4 = 0;
        bool has[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const bool valid = vvalid(p, my_v + j) && (!kWatch || watched(r.src[j], p) || watched(r.dst[j], p));
            const bool present = vvalid(p, my_v + j);
            const uint32_t cell = in8[2 * j] * 2u + in8[2 * j + 1];
            const uint32_t dir = (p.lut >> (cell * 2u)) & 3u;
            uint32_t bin = 0;
            bool inw;
            if (kW1) {
                const uint64_t d = r.ts[j] - p.start;
                inw = d < (uint64_t)p.window;
                bin = (uint32_t)d;
            } else {
                inw = map_bin(r.ts[j], p, bin);
            }
            const bool directed = valid && dir < 2u;
            const bool binned = directed && inw;
            // every in-window record was counted by pass 0: it takes a slot (a null key if not binned)
            has[j] = present && inw;
            dig[j] = bin >> (kFineShift + kDigit);
            key[j] = bin | ((dir & 1u) * kKeyDir) | (binned ? kKeyBinned : 0u);
            if (binned) { gmin = min(gmin, bin); gmax = max(gmax, bin); }
            if (tags_on) tag4 |= (in8[2 * j] | (in8[2 * j + 1] << 1) | ((inw ? 0u : 1u) << 2)) << (8 * j);
            tot.add(valid, cell, directed && !inw, dir, r.by[j]);
        }
        if (tags_on && my_v < p.nv) store_tags4(p, my_v, tag4);
        sort_and_write(S, dig, key, r.by, has, a.coarse_cur, 0u, a.key_a, a.by_a, kFineShift + kDigit);
    }
    const uint32_t mn = __reduce_min_sync(kFull, gmin), mx = __reduce_max_sync(kFull, gmax);
    if (lane == 0 && mn <= mx) { atomicMin(p.touched, mn); atomicMax(p.touched + 1, mx); }
    flush_totals(tot, p.totals, s_tot);
}

// ---------------------------------------------------------------- pass 2: fine partition
__global__ void __launch_bounds__(kPT) k_part_fine(PartArgs a) {
    __shared__ SortSmem S;
    __shared__ uint32_t s_u;
    const uint32_t n_units = a.cunit_base[a.nc];
    for (;;) {
        if (threadIdx.x == 0) s_u = atomicAdd(&a.counters[0], 1u);
        __syncthreads();
        const uint32_t ticket = s_u;
        __syncthreads();
        if (ticket >= n_units) break;
        // tickets are spread over the coarse buckets (u = ticket * P mod n_units, P a prime
        // larger than any unit count: a bijection): consecutive units of one coarse bucket would
        // have every CTA reserve space on the same 128 fine cursors at once
        const uint32_t u = (uint32_t)(((uint64_t)ticket * 982451653ull) % n_units);
        // coarse bucket of unit u: the last c with cunit_base[c] <= u
        uint32_t lo = 0, len = a.nc;
        while (len) {
            const uint32_t h = len >> 1;
            if (a.cunit_base[lo + h] <= u) { lo += h + 1; len -= h + 1; } else len = h;
        }
        const uint32_t c = lo - 1;
        const uint32_t r0 = a.coarse_base[c] + (u - a.cunit_base[c]) * kPChunk;
        const uint32_t r1 = min(r0 + kPChunk, a.coarse_base[c + 1]);
        uint32_t dig[4], key[4];
        uint64_t by[4];
        bool has[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint32_t i = r0 + threadIdx.x + j * kPT;   // coalesced
            has[j] = i < r1;
            key[j] = has[j] ? __ldcs(a.key_a + i) : 0u;
            by[j] = has[j] ? __ldcs(a.by_a + i) : 0ull;
            dig[j] = ((key[j] & kBinMask) >> kFineShift) & 127u;
        }
        sort_and_write(S, dig, key, by, has, a.fine_cur, c << kDigit, a.key_b, a.by_b, kFineShift);
    }
}

// ---------------------------------------------------------------- pass 3: bin one fine bucket
// ring: cnt[8192][2], lo[8192][2], hi[8192][2] u32 (192 KB): count, low and high words of
// the byte sums; the high word absorbs (bytes >> 32) + the carry out of the low word, so the
// u64 sum is exact mod 2^64 without touching HBM before the flush.
__global__ void __launch_bounds__(kPT, 1) k_part_bin(KernelParams p, PartArgs a) {
    extern __shared__ __align__(16) uint32_t smem[];
    uint32_t* s_cnt = smem;
    uint32_t* s_lo = smem + kFineBins * 2u;
    uint32_t* s_hi = smem + kFineBins * 4u;
    __shared__ uint32_t s_u;
    for (uint32_t i = threadIdx.x; i < kFineBins * 6u / 4u; i += kPT) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const uint32_t n_units = a.unit_base[a.nf];
    const uint32_t prev_word = p.epoch > 1 ? (((p.epoch - 1u) << 2) | kTileInit) : 0u;
    const uint32_t init_word = (p.epoch << 2) | kTileInit, claimed_word = (p.epoch << 2) | kTileClaimed;
    const bool key32 = true;   // B < 2^27 on this path: 2*bin+dir keys never collide with sentinels
    for (;;) {
        if (threadIdx.x == 0) s_u = atomicAdd(&a.counters[1], 1u);
        __syncthreads();
        const uint32_t u = s_u;
        if (u >= n_units) break;
        uint32_t lo = 0, len = a.nf;
        while (len) {
            const uint32_t h = len >> 1;
            if (a.unit_base[lo + h] <= u) { lo += h + 1; len -= h + 1; } else len = h;
        }
        const uint32_t f = lo - 1;
        const uint32_t r0 = a.fine_base[f] + (u - a.unit_base[f]) * kPartRecords;
        const uint32_t r1 = min(r0 + kPartRecords, a.fine_base[f + 1]);
        // claim this warp's two tiles now: the CAS round trip overlaps the accumulation
        uint32_t oc[2] = {0u, 0u};
        if (lane == 0) {
#pragma unroll
            for (uint32_t kk = 0; kk < 2u; ++kk) {
                const uint32_t t = f * (kFineBins / kTileBins) + warp + kk * (kPT / 32u);
                if (t < p.n_tiles) {
                    uint32_t* fl = p.tile_flags + t;
                    oc[kk] = claim_outcome(fl, p.epoch, prev_word, atomicCAS(fl, prev_word, claimed_word));
                }
            }
        }
        // accumulate (warp-strided 128-record steps, 4 per lane, coalesced)
        for (uint32_t base = r0 + warp * 128u; base < r1; base += (kPT / 32u) * 128u) {
            uint32_t key[4];
            uint64_t by[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint32_t i = base + j * 32u + lane;
                key[j] = i < r1 ? __ldcs(a.key_b + i) : 0u;
                by[j] = i < r1 ? __ldcs(a.by_b + i) : 0ull;
            }
            const uint32_t k0 = __shfl_sync(kFull, key[0], 0), k3 = __shfl_sync(kFull, key[3], 31);
            const bool hot = key32 && k0 == k3 && (k0 & kKeyBinned);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const bool b = (key[j] & kKeyBinned) != 0u;
                const uint32_t slot = ((key[j] & (kFineBins - 1u)) << 1) | ((key[j] >> 27) & 1u);
                uint32_t cnt = 1u;
                uint64_t byt = by[j];
                bool act = b;
                if (hot) {   // a hot millisecond: aggregate equal keys of the warp first
                    const uint32_t kk = b ? (key[j] & (kKeyDir * 2u - 1u)) : 0xFFFFFFFFu - lane;
                    const unsigned m = __match_any_sync(kFull, kk);
                    const bool leader = lane == (uint32_t)(__ffs(m) - 1);
                    unsigned groups = __ballot_sync(kFull, b && leader && __popc(m) > 1);
                    while (groups) {
                        const int l = __ffs(groups) - 1;
                        groups &= groups - 1u;
                        const unsigned g = __shfl_sync(kFull, m, l);
                        const uint64_t s = warp_sum_u64(((g >> lane) & 1u) ? by[j] : 0ull);
                        if (lane == (uint32_t)l) { byt = s; cnt = (uint32_t)__popc(g); }
                    }
                    act = b && leader;
                }
                if (act) {
                    atomicAdd(s_cnt + slot, cnt);
                    const uint32_t l32 = (uint32_t)byt;
                    const uint32_t old = atomicAdd(s_lo + slot, l32);
                    const uint32_t h = (uint32_t)(byt >> 32) + ((old + l32 < old) ? 1u : 0u);
                    if (h) atomicAdd(s_hi + slot, h);
                }
            }
        }
        __syncthreads();
        // flush: warp w owns tiles w and w + 16 of the bucket (claimed when the unit started); its
        // won tiles go first (plain stores, then published), so a warp waits for a tile claimed
        // elsewhere only when it holds nothing unpublished
        const uint32_t oa = __shfl_sync(kFull, oc[0], 0), ob = __shfl_sync(kFull, oc[1], 0);
        const bool swap = ob == kWon && oa != kWon;
        for (uint32_t r = 0; r < 2u; ++r) {
            const uint32_t kk = (r == 0u) == !swap ? 0u : 1u;
            const uint32_t o = kk ? ob : oa;
            const uint32_t tt = warp + kk * (kPT / 32u);
            const uint32_t t = f * (kFineBins / kTileBins) + tt;
            if (o == 0u) continue;   // beyond the last tile
            uint32_t c[8][2], l[8][2], hh[8][2];
            bool nz = false;
#pragma unroll
            for (int m = 0; m < 8; ++m) {
                const uint32_t s = (tt * kTileBins + m * 32u + lane) * 2u;
                const uint2 cc = *reinterpret_cast<const uint2*>(s_cnt + s), ll = *reinterpret_cast<const uint2*>(s_lo + s),
                            hv = *reinterpret_cast<const uint2*>(s_hi + s);
                c[m][0] = cc.x; c[m][1] = cc.y; l[m][0] = ll.x; l[m][1] = ll.y; hh[m][0] = hv.x; hh[m][1] = hv.y;
                nz |= (cc.x | cc.y) != 0u;
                *reinterpret_cast<uint2*>(s_cnt + s) = make_uint2(0, 0);
                *reinterpret_cast<uint2*>(s_lo + s) = make_uint2(0, 0);
                *reinterpret_cast<uint2*>(s_hi + s) = make_uint2(0, 0);
            }
            const bool won = o == kWon;
            if (!won && !__any_sync(kFull, nz)) continue;   // nothing to add (a won tile is written even if empty)
            if (o == kBusy) {   // claimed elsewhere: initialised after bounded work
                if (lane == 0) {
                    uint32_t spins = 0;
                    while (ld_acquire_u32(p.tile_flags + t) != init_word) {
                        __nanosleep(200);
                        if (++spins > kSpinLimit) __trap();
                    }
                }
                __syncwarp();
            }
            unsigned long long* g = p.bins + (size_t)t * kTileBins * 4u;
#pragma unroll
            for (int m = 0; m < 8; ++m) {
                const uint32_t bin = m * 32u + lane;
                const unsigned long long bo = ((unsigned long long)hh[m][0] << 32) | l[m][0];
                const unsigned long long bi = ((unsigned long long)hh[m][1] << 32) | l[m][1];
                ulonglong2* gg = reinterpret_cast<ulonglong2*>(g + bin * 4u);
                if (won) {
                    __stcs(gg, make_ulonglong2(c[m][0], bo));
                    __stcs(gg + 1, make_ulonglong2(c[m][1], bi));
                } else {
                    if (c[m][0]) { atomicAdd(g + bin * 4u, (unsigned long long)c[m][0]); if (bo) atomicAdd(g + bin * 4u + 1, bo); }
                    if (c[m][1]) { atomicAdd(g + bin * 4u + 2, (unsigned long long)c[m][1]); if (bi) atomicAdd(g + bin * 4u + 3, bi); }
                }
            }
            __syncwarp();
            if (won && lane == 0) st_release_u32(p.tile_flags + t, init_word);
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------- host launch
namespace {
size_t part_ring_smem() { return (size_t)kFineBins * 6u * 4u; }
}  // namespace

cudaError_t setup_partition() {
    cudaError_t e = cudaFuncSetAttribute(k_part_bin, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)part_ring_smem());
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k_part_count, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(kMaxFine * 4u));
    if (e != cudaSuccess) return e;
#define SETP(S, W, WL)                                                                                            \
    e = cudaFuncSetAttribute(k_part_scatter<S, W, WL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kStreamTableSmem); \
    if (e != cudaSuccess) return e;
#define SETPW(S) SETP(S, true, false) SETP(S, false, false) SETP(S, true, true) SETP(S, false, true)
    SETPW(kTabByte) SETPW(kTabPacked) SETPW(kTabPackedNoL2) SETPW(kTabGlobal)
#undef SETPW
#undef SETP
    return cudaSuccess;
}

bool partition_supported(uint32_t nbins) { return (nbins + kFineBins - 1) / kFineBins <= kMaxFine; }

// one sub-batch of at most L.cap records (p describes it); 5 launches + 1 memset
cudaError_t launch_partitioned(const KernelParams& p, void* scratch, const PartLayout& L, int sm_count,
                               cudaStream_t st, int* launches) {
    auto* base = static_cast<unsigned char*>(scratch);
    PartArgs a{};
    a.by_a = reinterpret_cast<unsigned long long*>(base + L.by_a);
    a.by_b = reinterpret_cast<unsigned long long*>(base + L.by_b);
    a.key_a = reinterpret_cast<uint32_t*>(base + L.key_a);
    a.key_b = reinterpret_cast<uint32_t*>(base + L.key_b);
    a.fine_cnt = reinterpret_cast<uint32_t*>(base + L.fine_cnt);
    a.fine_base = reinterpret_cast<uint32_t*>(base + L.fine_base);
    a.fine_cur = reinterpret_cast<uint32_t*>(base + L.fine_cur);
    a.unit_base = reinterpret_cast<uint32_t*>(base + L.unit_base);
    a.coarse_base = reinterpret_cast<uint32_t*>(base + L.coarse_base);
    a.coarse_cur = reinterpret_cast<uint32_t*>(base + L.coarse_cur);
    a.cunit_base = reinterpret_cast<uint32_t*>(base + L.cunit_base);
    a.counters = reinterpret_cast<uint32_t*>(base + L.counters);
    a.nf = L.nf;
    a.nc = L.nc;
    cudaError_t e = cudaMemsetAsync(a.fine_cnt, 0, (size_t)L.nf * 4u, st);
    if (e != cudaSuccess) return e;
    k_part_count<<<sm_count * 2, kPT, (size_t)L.nf * 4u, st>>>(p, a);
    k_part_plan<<<1, 1024, 0, st>>>(a);
    const int tab = stream_table_mode(p.has_bytes != 0u, p.nbnd, p.n_mixed, p.tab_mode);
    const size_t tsm = stream_table_bytes(tab, p.nbnd, p.n_mixed);
    const uint64_t chunks = (p.nv + kPChunk - 1) / kPChunk;
    const int g1 = (int)(chunks < (uint64_t)sm_count ? (chunks ? chunks : 1) : (uint64_t)sm_count);
    const bool w1 = p.width == 1u, wl = p.wn != 0u;
#define SCAT(S)                                                                            \
    if (w1 && !wl) k_part_scatter<S, true, false><<<g1, kPT, tsm, st>>>(p, a);             \
    else if (!wl) k_part_scatter<S, false, false><<<g1, kPT, tsm, st>>>(p, a);             \
    else if (w1) k_part_scatter<S, true, true><<<g1, kPT, tsm, st>>>(p, a);                \
    else k_part_scatter<S, false, true><<<g1, kPT, tsm, st>>>(p, a);
    switch (tab) {
        case kTabByte: SCAT(kTabByte) break;
        case kTabPacked: SCAT(kTabPacked) break;
        case kTabPackedNoL2: SCAT(kTabPackedNoL2) break;
        default: SCAT(kTabGlobal) break;
    }
#undef SCAT
    k_part_fine<<<sm_count * 4, kPT, 0, st>>>(a);   // 4 x 26 KB smem, 32 registers: 4 CTAs per SM
    k_part_bin<<<sm_count, kPT, part_ring_smem(), st>>>(p, a);
    *launches += 5;
    return cudaGetLastError();
}

}  // namespace sinet
