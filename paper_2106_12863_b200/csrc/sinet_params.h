// Kernel parameter block and build constants shared by host launchers and device code.
#pragma once
#include <cstdint>
#include <vector_types.h>

namespace sinet {

constexpr uint32_t kTileBins = 256;        // bins per claim tile (8 KB of u64[4] bins)
constexpr uint32_t kClsWords = 4096;       // 65536 /16 blocks x 2 bits
constexpr uint32_t kRankWords = 2048;      // 4096 u16 prefix counts
// staged beyond the class table + rank (24 KB): level 2 + entries + boundaries if they fit here
constexpr uint32_t kSmallExtraBytes = 7 * 1024;
constexpr unsigned kFull = 0xFFFFFFFFu;

// tile state word: epoch << 2 | state
constexpr uint32_t kTileClaimed = 1u;
constexpr uint32_t kTileInit = 2u;

struct KernelParams {
    const uint64_t* ts;
    const uint32_t* src;
    const uint32_t* dst;
    const uint64_t* bytes;
    uint64_t n;                    // records in this batch
    uint64_t nv;                   // n + head: records in "virtual" 16-byte-aligned index space
    uint32_t head;                 // columns start `head` records past a 16-byte boundary (0..3)
    uint32_t tags_vec;             // 1 if tags - head is 4-byte aligned (u32 tag stores)
    uint8_t* tags;                 // nullable
    unsigned long long* bins;      // u64 [B_pad][2 dir][2 metric]
    unsigned long long* totals;    // 12 x u64
    uint32_t* tile_flags;          // [n_tiles]
    const uint32_t* cls2;          // [4096]
    const uint32_t* bnd;           // [nbnd]
    const uint32_t* rank;          // [2048] u16 pairs: mixed blocks before each class-table word
    const uint32_t* mentry;        // [n_mixed] entry of each mixed /16 block
    const uint32_t* l2;            // [n_mixed * 16] 2-bit /24 classes of the mixed /16 blocks
    const uint8_t* b16;            // [65536] byte /16 classes (2 + m: mixed block m), if has_bytes
    const uint8_t* b24;            // [n_mixed * 256] byte /24 classes of the mixed blocks
    uint32_t has_bytes;            // 1: the byte encoding exists (n_mixed <= kMaxByteMixed)
    int32_t tab_mode;              // stream kernel table encoding: -1 automatic, else forced (kTab*)
    uint32_t nbnd;
    uint32_t n_mixed;
    uint32_t small;                // 1: level 2, entries and boundaries fit in shared memory
    uint32_t stream_groups;        // 0 auto, 1 or 2: layout of the stream kernel's ring
    uint32_t stream_kernel;        // 0 auto, 1 group-barrier kernel (k_hist_stream), 2 warp-specialised (k_hist_ws)
    uint32_t debug;                // 1: k_hist_ws counts its slow paths (sinet_debug_counters)
    uint32_t ranges_per_group;     // 0 = default: record ranges handed out per group (load balance)
    uint32_t n_ranges;             // set by the launcher
    uint32_t* range_counter;       // zeroed by the launcher before each launch
    uint32_t* touched;             // [2] min / max binned bin of this epoch (sparse multi-GPU exchange)
    const uint32_t* wbits;         // NEXT-2 watchlist: [2048] bitmap of /16 blocks holding a listed address
    const uint32_t* wlist;         // sorted distinct listed addresses
    uint32_t wn;                   // 0 = no watchlist
    uint32_t lut;                  // 4 x 2 bits, index s_in*2+d_in
    uint64_t start;                // window start (ms)
    uint32_t window;               // W (ms) < 2^32
    uint32_t width;                // w (ms)
    uint32_t magic;                // floor(2^32 / w) for w >= 2
    uint32_t nbins;                // B
    uint32_t epoch;                // current epoch
    uint32_t n_tiles;
};

// Shared-memory bytes of the staged lookup table: class table + rank (+ small lists: level 2,
// entries, boundaries).
inline unsigned long table_extra_bytes(uint32_t nbnd, uint32_t n_mixed) {
    return (unsigned long)n_mixed * 68u + (unsigned long)nbnd * 4u;
}
inline bool table_small(uint32_t nbnd, uint32_t n_mixed) { return table_extra_bytes(nbnd, n_mixed) <= kSmallExtraBytes; }
inline unsigned long table_smem_bytes(uint32_t nbnd, uint32_t n_mixed, bool small) {
    return (unsigned long)(kClsWords + kRankWords) * 4u + (small ? table_extra_bytes(nbnd, n_mixed) : 0u);
}
constexpr unsigned long kMaxTableSmem = (unsigned long)(kClsWords + kRankWords) * 4u + kSmallExtraBytes;

// Lookup-table encodings of the stream kernel, all staged in shared memory except the last:
//   BYTE       byte /16 classes (64 KB) + byte /24 classes of the mixed blocks + entries + boundaries
//   PACKED     2-bit /16 classes + rank + 2-bit /24 level 2 + entries + boundaries
//   PACKED_NOL2  the same without level 2: a mixed /16 holds up to 7 boundaries inline (one
//                16-byte entry, decoded branch-free), else searches its boundaries
//   GLOBAL     2-bit /16 classes + rank in shared memory, the rest read from global memory
enum : int { kTabByte = 0, kTabPacked = 1, kTabPackedNoL2 = 2, kTabGlobal = 3 };
constexpr unsigned long kStreamTableSmem = 96ul * 1024ul;   // next to the 128 KB ring
inline unsigned long stream_table_bytes(int mode, uint32_t nbnd, uint32_t n_mixed) {
    const unsigned long tail = (unsigned long)n_mixed * 4u + (unsigned long)nbnd * 4u;   // entries + boundaries
    switch (mode) {
        case kTabByte: return 65536ul + (((unsigned long)n_mixed * 256u + 15u) & ~15ul) + 16u + tail;
        case kTabPacked: return (unsigned long)(kClsWords + kRankWords) * 4u + (unsigned long)n_mixed * 64u + tail;
        case kTabPackedNoL2: return (unsigned long)(kClsWords + kRankWords) * 4u + tail + (unsigned long)n_mixed * 12u;   // 16-byte entries
        default: return (unsigned long)(kClsWords + kRankWords) * 4u;
    }
}
// the fastest encoding that fits (forced: 0..3 if it fits, else the automatic choice)
inline int stream_table_mode(bool has_bytes, uint32_t nbnd, uint32_t n_mixed, int forced = -1) {
    auto fits = [&](int m) { return m == kTabGlobal || stream_table_bytes(m, nbnd, n_mixed) <= kStreamTableSmem; };
    if (forced >= 0 && forced <= 3 && (forced != kTabByte || has_bytes) && fits(forced)) return forced;
    if (has_bytes && fits(kTabByte)) return kTabByte;
    if (fits(kTabPacked)) return kTabPacked;
    if (fits(kTabPackedNoL2)) return kTabPackedNoL2;
    return kTabGlobal;
}

}  // namespace sinet
