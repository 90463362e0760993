// Prefix-table compiler.
//
// Alg. 1 tests one address against a CIDR entry Y.Y.Y.Y/Z by masking both
// with Z (l.6-7) and checking SB - CB == 0 (l.8-9);
// the input is a "CIDR list" (l.1) and a record is a member if any
// entry matches (reading A3).  For a normalised entry (CB = Y & mask(Z)),
// (ip & mask(Z)) == CB  <=>  CB <= ip <= CB | ~mask(Z), so the union of the
// list is a set of disjoint intervals, compiled here once per sinet_open into
// sorted boundaries plus a /16 class table.  The kernel then answers a
// membership query with one shared-memory load for blocks that are entirely
// inside or outside and a short search for mixed blocks.
#include "prefix_compile.h"

#include <algorithm>
#include <cstdio>
#include <utility>

namespace sinet {

bool compile_prefixes(const uint32_t* net, const uint8_t* len, uint32_t n,
                      CompiledTable* out, std::string* err) {
    if (n == 0) { *err = "empty CIDR list (n_prefixes == 0)"; return false; }
    if (n > kMaxPrefixes) { *err = "too many prefixes (max 32767)"; return false; }
    if (!net || !len) { *err = "NULL prefix array"; return false; }

    // normalise (Alg. 1 l.7: CB = bitmask(Y, Z)) and form [lo, hi] as u64
    std::vector<std::pair<uint64_t, uint64_t>> iv;
    iv.reserve(n);
    for (uint32_t i = 0; i < n; ++i) {
        if (len[i] > 32) {
            char buf[96];
            std::snprintf(buf, sizeof buf, "prefix_len[%u] = %u > 32", i, (unsigned)len[i]);
            *err = buf;
            return false;
        }
        uint64_t host = (len[i] == 0) ? 0xFFFFFFFFull : ((1ull << (32 - len[i])) - 1ull);
        uint64_t lo = (uint64_t)net[i] & ~host & 0xFFFFFFFFull;
        iv.emplace_back(lo, lo | host);
    }
    std::sort(iv.begin(), iv.end());
    iv.erase(std::unique(iv.begin(), iv.end()), iv.end());
    out->n_unique = (uint32_t)iv.size();

    // merge overlapping or adjacent intervals
    std::vector<std::pair<uint64_t, uint64_t>> merged;
    for (auto& p : iv) {
        if (!merged.empty() && p.first <= merged.back().second + 1)
            merged.back().second = std::max(merged.back().second, p.second);
        else
            merged.push_back(p);
    }
    out->n_intervals = (uint32_t)merged.size();

    out->bnd.clear();
    for (auto& p : merged) {
        out->bnd.push_back((uint32_t)p.first);
        if (p.second < 0xFFFFFFFFull) out->bnd.push_back((uint32_t)(p.second + 1));
    }
    const std::vector<uint32_t>& b = out->bnd;

    out->cls2.assign(4096, 0u);
    out->entry.assign(65536, 0u);
    out->n_mixed = 0;
    // two-pointer sweep over the 65536 /16 blocks
    size_t le_lo = 0;   // #boundaries <= block start
    size_t le_hi = 0;   // #boundaries <= block end
    for (uint32_t x = 0; x < 65536; ++x) {
        uint32_t blo = x << 16, bhi = blo | 0xFFFFu;
        while (le_lo < b.size() && b[le_lo] <= blo) ++le_lo;
        if (le_hi < le_lo) le_hi = le_lo;
        while (le_hi < b.size() && b[le_hi] <= bhi) ++le_hi;
        uint32_t lo = (uint32_t)le_lo, cnt = (uint32_t)(le_hi - le_lo);
        uint32_t cls = (cnt == 0) ? (lo & 1u) : 2u;
        if (cls == 2) ++out->n_mixed;
        out->cls2[x >> 4] |= cls << ((x & 15u) * 2u);
        out->entry[x] = lo | (cnt << 16);
    }
    out->rank.assign(2048, 0u);
    out->mentry.clear();
    out->l2.assign((size_t)out->n_mixed * 16u, 0u);
    uint32_t m = 0;
    for (uint32_t x = 0; x < 65536; ++x) {
        if ((x & 15u) == 0) {
            const uint32_t w = x >> 4;
            out->rank[w >> 1] |= (m & 0xFFFFu) << ((w & 1u) * 16u);
        }
        if (((out->cls2[x >> 4] >> ((x & 15u) * 2u)) & 3u) != 2u) continue;
        out->mentry.push_back(out->entry[x]);
        // /24 sub-blocks: the same uniform/mixed test one level down
        const uint32_t lo = out->entry[x] & 0xFFFFu, len = out->entry[x] >> 16;
        for (uint32_t y = 0; y < 256; ++y) {
            const uint32_t a = (x << 16) | (y << 8), z = a | 0xFFu;
            uint32_t le_a = lo, le_z = lo;   // #boundaries <= a, <= z
            for (uint32_t i = lo; i < lo + len; ++i) {
                if (b[i] <= a) ++le_a;
                if (b[i] <= z) ++le_z;
            }
            const uint32_t c2 = (le_a == le_z) ? (le_a & 1u) : 2u;
            out->l2[(size_t)m * 16u + (y >> 4)] |= c2 << ((y & 15u) * 2u);
        }
        ++m;
    }
    return true;
}

}  // namespace sinet
