// NEXT-3 text parser: launch interface (kernel in sinet_parse.cu).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace sinet {

constexpr uint32_t kParseChunk = 16u * 1024u;   // text bytes owned by one chunk (look-back unit)

// line status codes (= SINET_LINE_* in include/sinet.h)
constexpr uint32_t kLineOk = 0, kLineLong = 1, kLineColumns = 2, kLineTime = 3, kLineSrc = 4, kLineDst = 5,
                   kLineBytes = 6;

struct ParseParams {
    const uint8_t* text;
    uint64_t len;
    int32_t tz_offset_min;
    uint64_t* ts;
    uint32_t* src;
    uint32_t* dst;
    uint64_t* bytes;
    uint64_t cap;                      // output records capacity
    uint8_t* status;                   // nullable
    uint64_t status_cap;
    unsigned long long* ticket;        // chunk tickets (zeroed)
    unsigned long long* st_lines;      // [n_chunks] look-back words of the line counts (zeroed)
    unsigned long long* st_valid;      // [n_chunks] look-back words of the valid counts (zeroed)
    unsigned long long* result;        // [10]: lines, valid (host-filled from the look-back), first bad, count[7]
    uint64_t n_chunks;
    uint32_t packed;                   // 1: len < 2^31, one look-back of (lines << 31 | valid) in st_lines
};

size_t parse_smem_bytes();
cudaError_t launch_parse_text(const ParseParams& p, int sm_count, cudaStream_t st);

}  // namespace sinet
