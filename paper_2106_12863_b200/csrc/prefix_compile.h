// Host-side compilation of the CIDR list into the device lookup table.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace sinet {

// Device lookup table for membership of a u32 address in the union of the
// CIDR entries (Alg. 1 l.4-9).
//
//   bnd[K]     sorted, distinct u32 boundaries of the merged member intervals:
//              every interval [lo, hi] contributes lo and (if hi < 2^32-1) hi+1.
//              member(ip) == (number of boundaries <= ip) is odd.
//   cls2[4096] 2-bit class per /16 block x = ip >> 16, 16 per word:
//              0 = no address of the block is a member, 1 = all are, 2 = mixed.
//   entry[65536] for block x: lo | len << 16, where lo = #boundaries <= x<<16
//              and len = #boundaries in (x<<16, x<<16 | 0xFFFF]; a mixed block's
//              member(ip) = (lo + #{bnd[lo..lo+len) <= ip}) & 1.
struct CompiledTable {
    std::vector<uint32_t> bnd;
    std::vector<uint32_t> cls2;
    std::vector<uint32_t> entry;
    // mixed blocks, numbered m = 0.. in ascending x:
    //   rank[w]   = number of mixed blocks in cls2 words [0, w) (u16 pairs packed in u32)
    //   mentry[m] = entry[x] of mixed block m
    //   l2[m*16..] = 2-bit classes of its 256 /24 sub-blocks (0 out, 1 in, 2 mixed -> search)
    std::vector<uint32_t> rank;     // 2048 u32 = 4096 u16
    std::vector<uint32_t> mentry;
    std::vector<uint32_t> l2;
    // byte encoding (only when n_mixed <= kMaxByteMixed), read by the stream kernel from
    // shared memory with one byte load per level:
    //   b16[x]         0 = block x out, 1 = in, 2 + m = mixed block number m
    //   b24[m*256 + y] 0 / 1 / 2 (mixed -> search mentry[m]'s boundaries) for /24 y of block m
    std::vector<uint8_t> b16;
    std::vector<uint8_t> b24;
    uint32_t n_unique = 0;     // distinct normalised entries
    uint32_t n_intervals = 0;  // merged member intervals
    uint32_t n_mixed = 0;      // /16 blocks of class 2
};

constexpr uint32_t kMaxPrefixes = 16383;   // <= 4P+2 boundaries keeps lo and len in 16 bits each
constexpr uint32_t kMaxByteMixed = 253;    // 2 + m fits a byte

// Returns false (with *err set) on invalid input (n == 0, len > 32, n > kMaxPrefixes).
bool compile_prefixes(const uint32_t* net, const uint8_t* len, uint32_t n,
                      CompiledTable* out, std::string* err);

// NEXT-4: labelled table (label[i] = 1 inside, 0 carved out); an address is a member iff
// its longest matching entry is labelled inside.  label == nullptr: every entry inside.
bool compile_prefixes_labelled(const uint32_t* net, const uint8_t* len, const uint8_t* label, uint32_t n,
                               CompiledTable* out, std::string* err);

}  // namespace sinet
