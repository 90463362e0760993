// Device-side building blocks shared by the sinet kernels (sm_100a).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "sinet_params.h"

namespace sinet {

// ---------------------------------------------------------------- a3 + a4: membership
// Alg. 1 l.6-9 against the compiled union of the CIDR list
// (prefix_compile.cpp): one shared-memory load decides /16 blocks wholly
// inside or outside; a mixed block is resolved at /24 granularity by a level-2
// class table, and only a mixed /24 counts its boundaries <= ip.
struct Table {
    const uint32_t* cls2;    // smem
    const uint16_t* rank;    // smem
    const uint32_t* l2;      // smem (small lists) or global
    const uint32_t* mentry;  // smem (small lists) or global
    const uint32_t* bnd;     // smem (small lists) or global
    bool any_long = true;    // kTabPackedNoL2: some mixed /16 has more than 7 boundaries
};

// member(ip): 1 LDS for a /16 wholly in or out; a mixed /16 finds its index m among the
// mixed blocks by rank (prefix count of the class-table word + popcount of the mixed
// codes before it in the word already loaded), then 1 LDS of its /24 class; only a
// mixed /24 (prefixes longer than /24) searches the block's few boundaries.
__device__ __forceinline__ uint32_t member(uint32_t ip, const Table& T) {
    const uint32_t x = ip >> 16;
    const uint32_t w = T.cls2[x >> 4];
    const uint32_t sh = (x & 15u) * 2u;
    const uint32_t c = (w >> sh) & 3u;
    if (c < 2u) return c;
    const uint32_t mixed = (w >> 1) & ~w & 0x55555555u;          // bit 2i: block i of the word is mixed
    const uint32_t m = T.rank[x >> 4] + __popc(mixed & ((1u << sh) - 1u));
    const uint32_t y = (ip >> 8) & 0xFFu;
    const uint32_t c2 = (T.l2[m * 16u + (y >> 4)] >> ((y & 15u) * 2u)) & 3u;
    if (c2 < 2u) return c2;
    const uint32_t e = T.mentry[m];
    uint32_t cnt = e & 0xFFFFu, len = e >> 16;
    const uint32_t* b = T.bnd + cnt;
    while (len) {
        const uint32_t half = len >> 1;
        if (b[half] <= ip) { b += half + 1; cnt += half + 1; len -= half + 1; }
        else len = half;
    }
    return cnt & 1u;
}

// member() for K addresses at once, with the same result per address.  The class word
// and the rank of every address are loaded together (the rank's address depends on the ip
// only), then every mixed block's /24 class, so a thread has K independent loads in flight
// per level (2 dependent shared-memory round trips instead of 3 serial ones per address,
// and no per-address branch).  Only addresses in a mixed /24 take the boundary search.
template <int K>
__device__ __forceinline__ void member_batch(const uint32_t (&ip)[K], uint32_t (&in)[K], const Table& T) {
    uint32_t w[K], r[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        w[k] = T.cls2[ip[k] >> 20];
        r[k] = T.rank[ip[k] >> 20];
    }
    uint32_t c2[K];
    bool search = false;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const uint32_t sh = ((ip[k] >> 16) & 15u) * 2u;
        const uint32_t c = (w[k] >> sh) & 3u;
        const uint32_t mixed = (w[k] >> 1) & ~w[k] & 0x55555555u;
        r[k] += __popc(mixed & ((1u << sh) - 1u));     // index among the mixed blocks (if c == 2)
        const uint32_t y = (ip[k] >> 8) & 0xFFu;
        c2[k] = (c == 2u) ? ((T.l2[r[k] * 16u + (y >> 4)] >> ((y & 15u) * 2u)) & 3u) : c;
        search |= c2[k] == 2u;
    }
#pragma unroll
    for (int k = 0; k < K; ++k) in[k] = c2[k] & 1u;
    if (search) {   // rare: a prefix longer than /24 shares this /24 with non-members
#pragma unroll
        for (int k = 0; k < K; ++k) {
            if (c2[k] != 2u) continue;
            const uint32_t e = T.mentry[r[k]];
            uint32_t cnt = e & 0xFFFFu, len = e >> 16;
            const uint32_t* b = T.bnd + cnt;
            while (len) {
                const uint32_t half = len >> 1;
                if (b[half] <= ip[k]) { b += half + 1; cnt += half + 1; len -= half + 1; }
                else len = half;
            }
            in[k] = cnt & 1u;
        }
    }
}

// #boundaries <= ip of a mixed block (its entry: first boundary | count << 16), odd = member
__device__ __forceinline__ uint32_t block_search(uint32_t e, uint32_t ip, const uint32_t* bnd) {
    uint32_t cnt = e & 0xFFFFu, len = e >> 16;
    const uint32_t* b = bnd + cnt;
    while (len) {
        const uint32_t half = len >> 1;
        if (b[half] <= ip) { b += half + 1; cnt += half + 1; len -= half + 1; }
        else len = half;
    }
    return cnt & 1u;
}

// Byte encoding (stream kernel, kTabByte; prefix_compile.h): every level is one byte load.
struct TableB {
    const uint8_t* b16;      // smem [65536]: 0 out, 1 in, 2 + m mixed block m
    const uint8_t* b24;      // smem [n_mixed * 256 (>= 16)]: 0 / 1 / 2 (mixed /24: search)
    const uint32_t* mentry;  // smem
    const uint32_t* bnd;     // smem
    bool any_sub24 = true;   // some boundary is not /24-aligned (a prefix longer than /24)
};

// member() of K addresses with the byte encoding: K byte loads of the /16 classes, then K
// byte loads of the /24 classes (an address outside a mixed block loads b24[0] - the same
// byte for every such lane, a broadcast - and keeps its class), branch-free; a mixed /24
// (a prefix longer than /24) searches its block's boundaries.  (Measured: a predicated
// inline-asm load with a PRMT-formed index executed 10 % fewer instructions but ran 7 %
// slower - the volatile asm pinned the schedule.)
template <int K>
__device__ __forceinline__ void member_batch_byte(const uint32_t (&ip)[K], uint32_t (&in)[K], const TableB& T) {
    uint32_t c[K];
#pragma unroll
    for (int k = 0; k < K; ++k) c[k] = T.b16[ip[k] >> 16];
    uint32_t m[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const bool mixed = c[k] >= 2u;
        m[k] = c[k] - 2u;
        const uint32_t c2 = T.b24[mixed ? ((m[k] << 8) | ((ip[k] >> 8) & 0xFFu)) : 0u];
        c[k] = mixed ? c2 : c[k];
    }
#pragma unroll
    for (int k = 0; k < K; ++k) in[k] = c[k] & 1u;
    if (T.any_sub24) {   // CTA-uniform: only a list with prefixes longer than /24 has mixed /24s
#pragma unroll
        for (int k = 0; k < K; ++k)
            if (c[k] == 2u) in[k] = block_search(T.mentry[m[k]], ip[k], T.bnd);
    }
}

// member() of K addresses with the packed encoding without level 2 (kTabPackedNoL2: large
// lists whose level 2 does not fit in shared memory, e.g. the 4096-entry C5 list: 2023 mixed
// /16 blocks with 1.9 boundaries on average).  A mixed /16 with <= 7 boundaries decides from
// its 16-byte inline entry (one LDS.128, seven compares, branch-free; measured C5 5.67 -> 5.18
// ms against searching every mixed block, 5.32 ms with 3 inline boundaries + search, 5.40 ms
// with a second entry behind a branch); a block with more boundaries searches them, in a
// second pass taken only if the list has such a block (a CTA-uniform flag set while staging:
// C5 5.18 -> 5.03 ms without the per-address check).
template <int K>
__device__ __forceinline__ void member_batch_nol2(const uint32_t (&ip)[K], uint32_t (&in)[K], const Table& T) {
    uint32_t w[K], r[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        w[k] = T.cls2[ip[k] >> 20];
        r[k] = T.rank[ip[k] >> 20];
    }
    bool search = false;
    uint32_t c[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const uint32_t sh = ((ip[k] >> 16) & 15u) * 2u;
        c[k] = (w[k] >> sh) & 3u;
        const uint32_t mixed = (w[k] >> 1) & ~w[k] & 0x55555555u;
        r[k] += __popc(mixed & ((1u << sh) - 1u));
        in[k] = c[k] & 1u;
        search |= c[k] == 2u;
    }
    if (search) {
        // inline block entries (stage_stream_table), 16 bytes per mixed block: its boundaries
        // 0-6 as u16 (low half - 1; unused slots 0xFFFF, which no low half exceeds) in .x .y .z
        // and the low half of .w, the parity of the boundaries before the block at .w bit 16,
        // .w bit 31 = more than 7 boundaries (.x = its mentry: search).  Branch-free: a warp holds
        // 256 addresses, so a rare loop-carrying path would run in nearly every warp.
        // The entry's 7 u16 values are sorted (a block's boundaries ascend; unused slots are
        // 0xFFFF), so #values below x is a 3-step branch-free binary search over them (with an
        // implicit +inf eighth slot), and the count's parity is the last step's outcome: 3
        // compares and 3 selects instead of 7 compares and 7 adds (C5: the linear decode was 65
        // of 242 instructions per record).
        const uint4* me128 = reinterpret_cast<const uint4*>(T.mentry);
#pragma unroll
        for (int k = 0; k < K; ++k) {
            if (c[k] != 2u) continue;
            const uint4 e = me128[r[k]];
            const uint32_t x = ip[k] & 0xFFFFu;
            const uint32_t v0 = e.x & 0xFFFFu, v1 = e.x >> 16, v2 = e.y & 0xFFFFu, v3 = e.y >> 16;
            const uint32_t v4 = e.z & 0xFFFFu, v5 = e.z >> 16, v6 = e.w & 0xFFFFu;
            const bool p1 = v3 < x;                       // count >= 4
            const bool p2 = (p1 ? v5 : v1) < x;           // count >= base + 2
            const bool p3 = (p1 ? (p2 ? v6 : v4) : (p2 ? v2 : v0)) < x;
            // count = 4 p1 + 2 p2 + p3: its parity is p3
            in[k] = ((p3 ? 1u : 0u) ^ (e.w >> 16)) & 1u;
        }
        if (T.any_long) {   // CTA-uniform: the list has a mixed /16 with more than 7 boundaries
#pragma unroll
            for (int k = 0; k < K; ++k) {
                if (c[k] != 2u) continue;
                const uint4 e = me128[r[k]];
                if (e.w >> 31) in[k] = block_search(e.x, ip[k], T.bnd);
            }
        }
    }
}

// ---------------------------------------------------------------- NEXT-2: watchlist predicate
// Exact-address set (AbuseIPDB / GRIZZLY STEPPE lists): a /16 bitmap
// rejects most addresses with one cached load, a binary search confirms the rest.
__device__ __forceinline__ bool watched(uint32_t ip, const KernelParams& p) {
    if (!((__ldg(p.wbits + (ip >> 21)) >> ((ip >> 16) & 31u)) & 1u)) return false;
    uint32_t lo = 0, len = p.wn;
    while (len) {
        const uint32_t half = len >> 1;
        if (__ldg(p.wlist + lo + half) < ip) { lo += half + 1; len -= half + 1; }
        else len = half;
    }
    return lo < p.wn && __ldg(p.wlist + lo) == ip;
}

// a record passes the filter iff there is no watchlist or an endpoint is listed
__device__ __forceinline__ bool watch_pass(uint32_t src, uint32_t dst, const KernelParams& p) {
    return p.wn == 0u || watched(src, p) || watched(dst, p);
}

// ---------------------------------------------------------------- a5: Map to a ms bin
// key = (ts - start) / w for start <= ts < start + W (bins of 1 ms P:L217,
// half-open, reading A15).  d < W < 2^32, so a 32-bit quotient with one
// correction step after the multiply-high estimate is exact.
__device__ __forceinline__ bool map_bin(uint64_t ts, const KernelParams& p, uint32_t& bin) {
    uint64_t d = ts - p.start;          // wraps for ts < start -> fails the test below
    if (d >= (uint64_t)p.window) return false;
    uint32_t d32 = (uint32_t)d;
    if (p.width == 1u) { bin = d32; return true; }
    uint32_t q = __umulhi(d32, p.magic);
    if (d32 - q * p.width >= p.width) ++q;
    bin = q;
    return true;
}

// ---------------------------------------------------------------- a7: side totals
__device__ __forceinline__ uint64_t warp_sum_u64(uint64_t v) {
    // three exact 32-bit warp reductions of 24/24/16-bit pieces, recombined mod 2^64
    uint32_t a = __reduce_add_sync(kFull, (uint32_t)(v & 0xFFFFFFu));
    uint32_t b = __reduce_add_sync(kFull, (uint32_t)((v >> 24) & 0xFFFFFFu));
    uint32_t c = __reduce_add_sync(kFull, (uint32_t)(v >> 48));
    return (uint64_t)a + ((uint64_t)b << 24) + ((uint64_t)c << 48);
}

// Per-thread accumulators of the side totals.  Instead of one counter pair per
// membership cell, keep sums over {all, s_in, d_in, s_in&d_in} (fewer predicated
// adds); the 2x2 matrix follows by inclusion-exclusion (mod 2^64) at the end.
struct WarpTotals {
    uint32_t cT, cS, cD, cSD, oc[2];
    uint64_t bT, bS, bD, bSD, ob[2];
    __device__ __forceinline__ void zero() {
        cT = cS = cD = cSD = 0u;
        bT = bS = bD = bSD = 0ull;
        oc[0] = oc[1] = 0u;
        ob[0] = ob[1] = 0ull;
    }
    __device__ __forceinline__ void add(bool valid, uint32_t cell, bool oow, uint32_t dir, uint64_t b) {
        if (valid) add_valid(cell, oow, dir, b);
    }
    // a record known to be valid: predicated adds, the rare out-of-window case as a branch
    __device__ __forceinline__ void add_valid(uint32_t cell, bool oow, uint32_t dir, uint64_t b) {
        const uint32_t s = cell >> 1, d = cell & 1u, sd = s & d;
        cT += 1u; cS += s; cD += d; cSD += sd;
        bT += b;
        if (s) bS += b;
        if (d) bD += b;
        if (sd) bSD += b;
        if (oow) {
            if (dir == 0u) { oc[0] += 1u; ob[0] += b; } else { oc[1] += 1u; ob[1] += b; }
        }
    }
};

// Sum the per-thread totals of a block and add them to the global totals (one RED per counter).
__device__ __forceinline__ void flush_totals(const WarpTotals& t, unsigned long long* g_totals,
                                             unsigned long long* s_scratch /* [32][12] */) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    unsigned long long v[12];
    {
        const unsigned long long cT = __reduce_add_sync(kFull, t.cT), cS = __reduce_add_sync(kFull, t.cS);
        const unsigned long long cD = __reduce_add_sync(kFull, t.cD), cSD = __reduce_add_sync(kFull, t.cSD);
        const unsigned long long bT = warp_sum_u64(t.bT), bS = warp_sum_u64(t.bS);
        const unsigned long long bD = warp_sum_u64(t.bD), bSD = warp_sum_u64(t.bSD);
        // cells s_in*2+d_in: 0 = neither, 1 = d only, 2 = s only, 3 = both (mod 2^64)
        v[0] = cT - cS - cD + cSD; v[1] = cD - cSD; v[2] = cS - cSD; v[3] = cSD;
        v[4] = bT - bS - bD + bSD; v[5] = bD - bSD; v[6] = bS - bSD; v[7] = bSD;
    }
    v[8] = __reduce_add_sync(kFull, t.oc[0]);
    v[9] = __reduce_add_sync(kFull, t.oc[1]);
    v[10] = warp_sum_u64(t.ob[0]);
    v[11] = warp_sum_u64(t.ob[1]);
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < 12; ++k) s_scratch[warp * 12 + k] = v[k];
    }
    __syncthreads();
    if (threadIdx.x < 12) {
        unsigned long long acc = 0;
        for (int w = 0; w < nw; ++w) acc += s_scratch[w * 12 + threadIdx.x];
        if (acc) atomicAdd(g_totals + threadIdx.x, acc);
    }
}

// Record the extent of the bins this launch wrote (warp-uniform call): the multi-GPU
// reduce only exchanges the bins inside every rank's touched range.
__device__ __forceinline__ void note_touched_warp(const KernelParams& p, uint32_t tmin, uint32_t tmax) {
    tmin = __reduce_min_sync(kFull, tmin);
    tmax = __reduce_max_sync(kFull, tmax);
    if ((threadIdx.x & 31u) == 0 && tmin <= tmax) {
        atomicMin(p.touched, tmin);
        atomicMax(p.touched + 1, tmax);
    }
}

// ---------------------------------------------------------------- a2: columnar record load
struct Rec4 {
    uint64_t ts[4];
    uint32_t src[4], dst[4];
    uint64_t by[4];
};

// Four consecutive records of the virtual (16-byte aligned) index space,
// starting at virtual index vbase (vbase % 4 == 0): record vbase + j is column
// element vbase + j - head.  Complete groups use 6 x 128-bit streaming loads;
// the ragged first and last groups use scalar loads.
__device__ __forceinline__ bool vvalid(const KernelParams& p, uint64_t v) {
    return v >= p.head && v < p.nv;
}

__device__ __forceinline__ ulonglong2 ldcs_v2u64(const uint64_t* p) { return __ldcs(reinterpret_cast<const ulonglong2*>(p)); }
__device__ __forceinline__ uint4 ldcs_v4u32(const uint32_t* p) { return __ldcs(reinterpret_cast<const uint4*>(p)); }

__device__ __forceinline__ void load4(const KernelParams& p, uint64_t vbase, Rec4& r) {
    if (vbase >= p.head && vbase + 4 <= p.nv) {
        const uint64_t a = vbase - p.head;
        ulonglong2 t0 = ldcs_v2u64(p.ts + a);
        ulonglong2 t1 = ldcs_v2u64(p.ts + a + 2);
        uint4 s = ldcs_v4u32(p.src + a);
        uint4 d = ldcs_v4u32(p.dst + a);
        ulonglong2 b0 = ldcs_v2u64(p.bytes + a);
        ulonglong2 b1 = ldcs_v2u64(p.bytes + a + 2);
        r.ts[0] = t0.x; r.ts[1] = t0.y; r.ts[2] = t1.x; r.ts[3] = t1.y;
        r.src[0] = s.x; r.src[1] = s.y; r.src[2] = s.z; r.src[3] = s.w;
        r.dst[0] = d.x; r.dst[1] = d.y; r.dst[2] = d.z; r.dst[3] = d.w;
        r.by[0] = b0.x; r.by[1] = b0.y; r.by[2] = b1.x; r.by[3] = b1.y;
    } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const bool ok = vvalid(p, vbase + j);
            const uint64_t a = vbase + j - p.head;
            r.ts[j] = ok ? p.ts[a] : 0ull;
            r.src[j] = ok ? p.src[a] : 0u;
            r.dst[j] = ok ? p.dst[a] : 0u;
            r.by[j] = ok ? p.bytes[a] : 0ull;
        }
    }
}

// Two consecutive records at even virtual index vbase (RPT = 2 configuration).
struct Rec2 {
    uint64_t ts[2];
    uint32_t src[2], dst[2];
    uint64_t by[2];
};

__device__ __forceinline__ void load2(const KernelParams& p, uint64_t vbase, Rec2& r) {
    if (vbase >= p.head && vbase + 2 <= p.nv) {
        const uint64_t a = vbase - p.head;
        const ulonglong2 t = __ldcs(reinterpret_cast<const ulonglong2*>(p.ts + a));
        const uint2 s = __ldcs(reinterpret_cast<const uint2*>(p.src + a));
        const uint2 d = __ldcs(reinterpret_cast<const uint2*>(p.dst + a));
        const ulonglong2 b = __ldcs(reinterpret_cast<const ulonglong2*>(p.bytes + a));
        r.ts[0] = t.x; r.ts[1] = t.y; r.src[0] = s.x; r.src[1] = s.y;
        r.dst[0] = d.x; r.dst[1] = d.y; r.by[0] = b.x; r.by[1] = b.y;
    } else {
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const bool ok = vvalid(p, vbase + j);
            const uint64_t a = vbase + j - p.head;
            r.ts[j] = ok ? p.ts[a] : 0ull;
            r.src[j] = ok ? p.src[a] : 0u;
            r.dst[j] = ok ? p.dst[a] : 0u;
            r.by[j] = ok ? p.bytes[a] : 0ull;
        }
    }
}

template <int R> struct RecN;
template <> struct RecN<4> { using T = Rec4; };
template <> struct RecN<2> { using T = Rec2; };
template <int R> __device__ __forceinline__ void loadN(const KernelParams& p, uint64_t vbase, typename RecN<R>::T& r);
template <> __device__ __forceinline__ void loadN<4>(const KernelParams& p, uint64_t vbase, Rec4& r) { load4(p, vbase, r); }
template <> __device__ __forceinline__ void loadN<2>(const KernelParams& p, uint64_t vbase, Rec2& r) { load2(p, vbase, r); }

__device__ __forceinline__ void store_tags4(const KernelParams& p, uint64_t vbase, uint32_t tag4) {
    if (p.tags_vec && vbase >= p.head && vbase + 4 <= p.nv) {
        *reinterpret_cast<uint32_t*>(p.tags + (vbase - p.head)) = tag4;
    } else {
        for (int j = 0; j < 4; ++j)
            if (vvalid(p, vbase + j)) p.tags[vbase + j - p.head] = (uint8_t)(tag4 >> (8 * j));
    }
}

// Stage the /16 class table and the mixed-block rank (and, for small lists, the
// level-2 classes, entries and boundaries) into shared memory at `smem`
// (table_smem_bytes() bytes).
// kSmall (compile-time, = p.small) lets the compiler see the level-2 / entry / boundary
// pointers as shared memory (LDS) rather than generic loads.
template <bool kSmall>
__device__ __forceinline__ Table stage_table(const KernelParams& p, uint32_t* smem) {
    Table T;
    const uint4* g4 = reinterpret_cast<const uint4*>(p.cls2);
    uint4* s4 = reinterpret_cast<uint4*>(smem);
    for (uint32_t i = threadIdx.x; i < kClsWords / 4; i += blockDim.x) s4[i] = __ldg(g4 + i);
    uint32_t* s_rank = smem + kClsWords;
    for (uint32_t i = threadIdx.x; i < kRankWords; i += blockDim.x) s_rank[i] = __ldg(p.rank + i);
    T.cls2 = smem;
    T.rank = reinterpret_cast<const uint16_t*>(s_rank);
    if (kSmall) {
        uint32_t* s_l2 = s_rank + kRankWords;
        uint32_t* s_me = s_l2 + 16u * p.n_mixed;
        uint32_t* s_bnd = s_me + p.n_mixed;
        for (uint32_t i = threadIdx.x; i < 16u * p.n_mixed; i += blockDim.x) s_l2[i] = __ldg(p.l2 + i);
        for (uint32_t i = threadIdx.x; i < p.n_mixed; i += blockDim.x) s_me[i] = __ldg(p.mentry + i);
        for (uint32_t i = threadIdx.x; i < p.nbnd; i += blockDim.x) s_bnd[i] = __ldg(p.bnd + i);
        T.l2 = s_l2;
        T.mentry = s_me;
        T.bnd = s_bnd;
    } else {
        T.l2 = p.l2;
        T.mentry = p.mentry;
        T.bnd = p.bnd;
    }
    return T;
}

// Stream-kernel tables (kTab*, sinet_params.h), staged at `smem` (stream_table_bytes() bytes).
template <int kTab> struct StreamTab { using T = Table; };
template <> struct StreamTab<kTabByte> { using T = TableB; };

template <int kTab>
__device__ __forceinline__ typename StreamTab<kTab>::T stage_stream_table(const KernelParams& p, uint32_t* smem) {
    if constexpr (kTab == kTabByte) {
        TableB T;
        uint4* s4 = reinterpret_cast<uint4*>(smem);
        const uint4* g16 = reinterpret_cast<const uint4*>(p.b16);
        for (uint32_t i = threadIdx.x; i < 65536u / 16u; i += blockDim.x) s4[i] = __ldg(g16 + i);
        const uint32_t n24 = (p.n_mixed * 256u + 15u) / 16u + 1u;   // >= 16 bytes (b24[0] is always read)
        uint4* s24 = s4 + 65536u / 16u;
        const uint4* g24 = reinterpret_cast<const uint4*>(p.b24);
        for (uint32_t i = threadIdx.x; i < n24; i += blockDim.x) s24[i] = __ldg(g24 + i);
        uint32_t* s_me = reinterpret_cast<uint32_t*>(s24 + n24);
        uint32_t* s_bnd = s_me + p.n_mixed;
        for (uint32_t i = threadIdx.x; i < p.n_mixed; i += blockDim.x) s_me[i] = __ldg(p.mentry + i);
        int sub24 = 0;
        for (uint32_t i = threadIdx.x; i < p.nbnd; i += blockDim.x) {
            const uint32_t b = __ldg(p.bnd + i);
            s_bnd[i] = b;
            sub24 |= (b & 0xFFu) != 0u ? 1 : 0;
        }
        T.any_sub24 = __syncthreads_or(sub24) != 0;
        T.b16 = reinterpret_cast<const uint8_t*>(s4);
        T.b24 = reinterpret_cast<const uint8_t*>(s24);
        T.mentry = s_me;
        T.bnd = s_bnd;
        return T;
    } else if constexpr (kTab == kTabPackedNoL2) {
        Table T = stage_table<false>(p, smem);
        uint32_t* s_me = smem + kClsWords + kRankWords;
        uint32_t* s_bnd = s_me + 4u * p.n_mixed;
        int long_here = 0;
        for (uint32_t i = threadIdx.x; i < p.n_mixed; i += blockDim.x) {
            const uint32_t me = __ldg(p.mentry + i), lo = me & 0xFFFFu, len = me >> 16;
            long_here |= len > 7u ? 1 : 0;
            uint4 q = make_uint4(me, 0u, 0u, 0x80000000u);   // > 7 boundaries: search
            if (len <= 7u) {
                uint32_t v[8];
                for (uint32_t j = 0; j < 7u; ++j) v[j] = (j < len) ? ((__ldg(p.bnd + lo + j) & 0xFFFFu) - 1u) : 0xFFFFu;
                q = make_uint4(v[0] | (v[1] << 16), v[2] | (v[3] << 16), v[4] | (v[5] << 16), v[6] | ((lo & 1u) << 16));
            }
            reinterpret_cast<uint4*>(s_me)[i] = q;
        }
        for (uint32_t i = threadIdx.x; i < p.nbnd; i += blockDim.x) s_bnd[i] = __ldg(p.bnd + i);
        T.l2 = nullptr;
        T.any_long = __syncthreads_or(long_here) != 0;
        T.mentry = s_me;
        T.bnd = s_bnd;
        return T;
    } else {
        return stage_table<kTab == kTabPacked>(p, smem);
    }
}

template <int kTab, int K>
__device__ __forceinline__ void member_batch_tab(const uint32_t (&ip)[K], uint32_t (&in)[K],
                                                 const typename StreamTab<kTab>::T& T) {
    if constexpr (kTab == kTabByte) member_batch_byte<K>(ip, in, T);
    else if constexpr (kTab == kTabPackedNoL2) member_batch_nol2<K>(ip, in, T);
    else member_batch<K>(ip, in, T);
}

}  // namespace sinet
