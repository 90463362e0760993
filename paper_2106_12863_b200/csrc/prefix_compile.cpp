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

// NEXT-4, labelled longest-prefix match: member intervals of "the longest entry
// containing ip is labelled inside".  Prefix intervals are laminar (nested or
// disjoint), so a sweep with a stack of open intervals yields, between
// consecutive interval edges, the innermost (longest) enclosing entry.
static void lpm_member_intervals(std::vector<std::pair<uint64_t, uint64_t>>& iv_lo_hi,
                                 const std::vector<uint8_t>& lab_by_iv,
                                 std::vector<std::pair<uint64_t, uint64_t>>* members) {
    // order: start ascending, then wider (outer) first
    std::vector<size_t> order(iv_lo_hi.size());
    for (size_t i = 0; i < order.size(); ++i) order[i] = i;
    std::sort(order.begin(), order.end(), [&](size_t a, size_t b) {
        if (iv_lo_hi[a].first != iv_lo_hi[b].first) return iv_lo_hi[a].first < iv_lo_hi[b].first;
        return iv_lo_hi[a].second > iv_lo_hi[b].second;
    });
    std::vector<size_t> stack;
    uint64_t cur = 0;   // next address not yet emitted
    auto emit = [&](uint64_t lo, uint64_t hi_excl, bool in) {
        if (!in || lo >= hi_excl) return;
        if (!members->empty() && members->back().second + 1 == lo) members->back().second = hi_excl - 1;
        else members->emplace_back(lo, hi_excl - 1);
    };
    auto top_in = [&]() { return !stack.empty() && lab_by_iv[stack.back()] != 0; };
    for (size_t k : order) {
        const uint64_t lo = iv_lo_hi[k].first, hi = iv_lo_hi[k].second;
        // close every open interval that ends before this one starts
        while (!stack.empty() && iv_lo_hi[stack.back()].second < lo) {
            const uint64_t end = iv_lo_hi[stack.back()].second + 1;
            emit(cur, end, top_in());
            cur = end;
            stack.pop_back();
        }
        emit(cur, lo, top_in());
        cur = lo;
        stack.push_back(k);
        (void)hi;
    }
    while (!stack.empty()) {
        const uint64_t end = iv_lo_hi[stack.back()].second + 1;
        emit(cur, end, top_in());
        cur = end;
        stack.pop_back();
    }
}

bool compile_prefixes(const uint32_t* net, const uint8_t* len, uint32_t n,
                      CompiledTable* out, std::string* err) {
    return compile_prefixes_labelled(net, len, nullptr, n, out, err);
}

bool compile_prefixes_labelled(const uint32_t* net, const uint8_t* len, const uint8_t* label, uint32_t n,
                               CompiledTable* out, std::string* err) {
    if (n == 0) { *err = "empty CIDR list (n_prefixes == 0)"; return false; }
    if (n > kMaxPrefixes) { *err = "too many prefixes (max 16383)"; return false; }
    if (!net || !len) { *err = "NULL prefix array"; return false; }

    // normalise (Alg. 1 l.7: CB = bitmask(Y, Z)) and form [lo, hi] as u64
    std::vector<std::pair<uint64_t, uint64_t>> iv;
    std::vector<uint8_t> lab;
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
        lab.push_back(label ? (label[i] ? 1 : 0) : 1);
    }
    std::vector<std::pair<uint64_t, uint64_t>> merged;
    if (!label) {
        // plain list: match-any = union of the intervals (reading A3)
        std::sort(iv.begin(), iv.end());
        iv.erase(std::unique(iv.begin(), iv.end()), iv.end());
        out->n_unique = (uint32_t)iv.size();
        for (auto& p : iv) {
            if (!merged.empty() && p.first <= merged.back().second + 1)
                merged.back().second = std::max(merged.back().second, p.second);
            else
                merged.push_back(p);
        }
    } else {
        // labelled: equal entries -> the last one wins, then the LPM sweep
        std::vector<size_t> idx;
        for (size_t i = 0; i < iv.size(); ++i) idx.push_back(i);
        std::stable_sort(idx.begin(), idx.end(), [&](size_t a, size_t b) { return iv[a] < iv[b]; });
        std::vector<std::pair<uint64_t, uint64_t>> uiv;
        std::vector<uint8_t> ulab;
        for (size_t k = 0; k < idx.size(); ++k) {
            if (k + 1 < idx.size() && iv[idx[k + 1]] == iv[idx[k]]) continue;   // a later equal entry wins
            uiv.push_back(iv[idx[k]]);
            ulab.push_back(lab[idx[k]]);
        }
        out->n_unique = (uint32_t)uiv.size();
        lpm_member_intervals(uiv, ulab, &merged);
    }
    out->n_intervals = (uint32_t)merged.size();

    out->bnd.clear();
    for (auto& p : merged) {
        out->bnd.push_back((uint32_t)p.first);
        if (p.second < 0xFFFFFFFFull) out->bnd.push_back((uint32_t)(p.second + 1));
    }
    if (out->bnd.size() > 65535u) { *err = "compiled table too large (> 65535 boundaries)"; return false; }
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
    out->b16.clear();
    out->b24.clear();
    if (out->n_mixed <= kMaxByteMixed) {
        out->b16.assign(65536, 0u);
        out->b24.assign((size_t)out->n_mixed * 256u, 0u);
        uint32_t k = 0;
        for (uint32_t x = 0; x < 65536; ++x) {
            const uint32_t c = (out->cls2[x >> 4] >> ((x & 15u) * 2u)) & 3u;
            if (c != 2u) { out->b16[x] = (uint8_t)c; continue; }
            out->b16[x] = (uint8_t)(2u + k);
            for (uint32_t y = 0; y < 256; ++y)
                out->b24[(size_t)k * 256u + y] = (uint8_t)((out->l2[(size_t)k * 16u + (y >> 4)] >> ((y & 15u) * 2u)) & 3u);
            ++k;
        }
    }
    return true;
}

}  // namespace sinet
