// k_parse_text: PA-7080 session-log text -> the four columns the hot path reads (NEXT-3).
//
// Table 1 lists the 24 items of a session record; the path needs
// No. 1 capture_time, No. 5 source_ip, No. 8 destination_ip
// and No. 21 bytes.  The file syntax is DESIGN.md readings
// A27-A31: '\n'-separated lines (an optional '\r' before it), 24 comma-separated
// fields, capture_time "YYYY/MM/DD HH:MM:SS.mmm" in local time at tz_offset_min,
// dotted-quad IPv4 ("translated to a 32-bit sequence"), bytes a
// decimal u64; per-line status, valid lines written in line order.
//
// B200 design: one pass over the text in HBM.  Persistent CTAs (8 x 128 threads per SM)
// take 16 KB chunks by ticket; each chunk (+ a 2 KB tail for the line that crosses its
// end) is staged into shared memory by a TMA bulk copy (cp.async.bulk, mbarrier
// completion); once it is parsed (results in registers) the next ticket's chunk streams
// into the same buffer while the previous chunk looks back and writes.  A chunk owns the
// lines that start right after one of its newlines (chunk 0 also the line at offset 0).  Every thread first turns 32-byte words of
// the staged text into newline and comma bitmasks (structural index, 1 bit per
// byte); the CTA counts line starts (block scan); one thread per line then finds
// the line end and the commas around fields 1, 5, 8 and 21 with popcounts over the
// bitmask words and parses those four fields; the chunk's (lines, valid) counts go
// through a decoupled look-back (two chained scans) that gives the line index and
// the output index of its first line, so valid records are compacted in line order
// without a second pass over the text.
#include <cstdint>
#include <cuda_runtime.h>

#include "sinet_parse.h"

namespace sinet {
namespace {

constexpr int kPT = 128;                       // threads per CTA
constexpr uint32_t kChunk = kParseChunk;       // bytes owned per chunk
constexpr uint32_t kTail = 2048;               // staged beyond the chunk: max line 2047 + '\n'
constexpr uint32_t kBuf = kChunk + kTail;      // staged bytes per buffer
constexpr uint32_t kBufAlloc = kBuf + 16;      // + slack: the word loop may read 3 bytes past the text
constexpr int kLPT = 1;                        // lines per thread per round
constexpr uint32_t kLCap = kPT * kLPT;         // lines per round
constexpr uint32_t kMaxLine = 2047;
constexpr uint32_t kNoLine = 0xFFu;
constexpr uint64_t kFlagAgg = 1ull << 62, kFlagInc = 2ull << 62, kValMask = (1ull << 62) - 1;
constexpr uint64_t kHalfMask = (1ull << 31) - 1;   // packed look-back word: lines << 31 | valid
constexpr uint32_t kWords = kBuf / 32u;        // bitmask words of a staged buffer (1 bit per byte)
static_assert(kChunk % (16 * kPT) == 0, "each thread scans a whole number of 16-byte words");
static_assert(kBuf % 32u == 0, "whole bitmask words");

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared.b64 P, [%0], %1;\n\t"
        "@!P bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
// global -> shared bulk copy (TMA engine), completion counted on the mbarrier
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
// Look-back words pack (flag, value) into one u64, and nothing else is read on the strength
// of them (the records and statuses a chunk writes are consumed after the kernel), so
// relaxed gpu-scope accesses suffice: no fence per load or publish.
__device__ __forceinline__ uint64_t ld_relaxed_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// thread 0: stage text [off, min(off + kBuf, len)) into buf.  The 16-byte-aligned body
// goes by TMA; the last < 16 bytes of the text by plain loads before the arrive (the
// mbarrier's release/acquire makes them visible to the waiting threads).
__device__ __forceinline__ void stage_chunk(const ParseParams& p, uint64_t off, uint8_t* buf, uint64_t* bar) {
    const uint64_t end = min(off + (uint64_t)kBuf, p.len);
    const uint32_t n = (uint32_t)(end - off);
    const uint32_t body = n & ~15u;
    for (uint32_t i = body; i < n; ++i) buf[i] = p.text[off + i];
    mbar_expect_tx(bar, body);
    if (body) bulk_g2s(buf, p.text + off, body, bar);
}

__device__ __forceinline__ uint32_t is_digit(uint32_t c) { return c - 48u < 10u; }

// capture_time at buf[b, b+23): "YYYY/MM/DD HH:MM:SS.mmm" -> epoch ms (UTC) of that local time.
// Days since 1970-01-01 from the civil date in closed form (era of 400 years, March-based
// day of year); the oracle counts them year by year instead.
__device__ bool parse_time(const uint8_t* s, int64_t tz_ms, uint64_t& out) {
    uint32_t c[23];
#pragma unroll
    for (int i = 0; i < 23; ++i) c[i] = s[i];
    bool ok = c[4] == '/' && c[7] == '/' && c[10] == ' ' && c[13] == ':' && c[16] == ':' && c[19] == '.';
#pragma unroll
    for (int i = 0; i < 23; ++i)
        if (i != 4 && i != 7 && i != 10 && i != 13 && i != 16 && i != 19) ok &= is_digit(c[i]) != 0u;
    if (!ok) return false;
    auto d = [&](int i) { return c[i] - 48u; };
    const uint32_t Y = d(0) * 1000u + d(1) * 100u + d(2) * 10u + d(3);
    const uint32_t M = d(5) * 10u + d(6), D = d(8) * 10u + d(9);
    const uint32_t h = d(11) * 10u + d(12), mi = d(14) * 10u + d(15), sec = d(17) * 10u + d(18);
    const uint32_t ms = d(20) * 100u + d(21) * 10u + d(22);
    if (Y < 1970u || M - 1u > 11u || D == 0u || h > 23u || mi > 59u || sec > 59u) return false;
    const bool leap = (Y % 4u == 0u && Y % 100u != 0u) || Y % 400u == 0u;
    const uint32_t mdays = (M == 2u) ? (leap ? 29u : 28u) : (30u + ((M + (M >> 3)) & 1u));
    if (D > mdays) return false;
    const uint32_t y = Y - (M <= 2u ? 1u : 0u);
    const uint32_t era = y / 400u, yoe = y - era * 400u;
    const uint32_t doy = (153u * (M > 2u ? M - 3u : M + 9u) + 2u) / 5u + D - 1u;
    const uint32_t doe = yoe * 365u + yoe / 4u - yoe / 100u + doy;
    const int64_t days = (int64_t)era * 146097 + (int64_t)doe - 719468;
    const int64_t local = ((days * 24 + h) * 60 + mi) * 60000 + (int64_t)sec * 1000 + ms;
    const int64_t utc = local - tz_ms;
    if (utc < 0) return false;
    out = (uint64_t)utc;
    return true;
}

// dotted quad at s[0, n): four octets, 1-3 digits, no leading zero, <= 255
__device__ bool parse_ipv4(const uint8_t* s, uint32_t n, uint32_t& out) {
    if (n < 7u || n > 15u) return false;
    uint32_t v = 0, x = 0, nd = 0, dots = 0, first = 0;
    bool ok = true;
    for (uint32_t i = 0; i < n; ++i) {
        const uint32_t ch = s[i];
        if (ch == '.') {
            ok &= nd != 0u && x <= 255u && !(nd > 1u && first == '0');
            v = (v << 8) | x;
            x = 0; nd = 0; ++dots;
        } else {
            ok &= is_digit(ch) != 0u && nd < 3u;
            if (nd == 0u) first = ch;
            x = x * 10u + (ch - 48u);
            ++nd;
        }
    }
    ok &= dots == 3u && nd != 0u && x <= 255u && !(nd > 1u && first == '0');
    out = (v << 8) | x;
    return ok;
}

// bytes at s[0, n): 1-20 decimal digits, < 2^64
__device__ bool parse_u64(const uint8_t* s, uint32_t n, uint64_t& out) {
    if (n == 0u || n > 20u) return false;
    uint64_t x = 0;
    bool ok = true;
    for (uint32_t i = 0; i < n; ++i) {
        const uint32_t dgt = (uint32_t)s[i] - 48u;
        ok &= dgt < 10u;
        // x * 10 + dgt <= 2^64 - 1  <=>  x < 1844674407370955161, or x == that and dgt <= 5
        ok &= x < 1844674407370955161ull || (x == 1844674407370955161ull && dgt <= 5u);
        x = x * 10u + dgt;
    }
    out = x;
    return ok;
}

struct LineOut {
    uint64_t ts, bytes;
    uint32_t src, dst, status;
};

// 4-bit mask of the bytes of w equal to the byte pattern pat (bit i = byte i): exact
// per-byte zero test of w ^ pat, flags gathered by one multiply.
__device__ __forceinline__ uint32_t eq_nibble(uint32_t w, uint32_t pat) {
    const uint32_t x = w ^ pat;
    const uint32_t f = ~(((x & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | x) & 0x80808080u;   // bit 7 of each zero byte
    return ((f >> 7) * 0x01020408u) >> 24;
}
__device__ __forceinline__ uint32_t eq_mask32(const uint4& v0, const uint4& v1, uint32_t pat) {
    return eq_nibble(v0.x, pat) | (eq_nibble(v0.y, pat) << 4) | (eq_nibble(v0.z, pat) << 8) |
           (eq_nibble(v0.w, pat) << 12) | (eq_nibble(v1.x, pat) << 16) | (eq_nibble(v1.y, pat) << 20) |
           (eq_nibble(v1.z, pat) << 24) | (eq_nibble(v1.w, pat) << 28);
}

// position of the n-th (0-based) set bit of m (n < popc(m))
__device__ __forceinline__ uint32_t nth_bit(uint32_t m, uint32_t n) {
    uint32_t pos = 0;
#pragma unroll
    for (uint32_t w = 16; w >= 1; w >>= 1) {
        const uint32_t c = __popc(m & ((1u << w) - 1u));
        if (n >= c) { n -= c; m >>= w; pos += w; }
    }
    return pos;
}

// Parse the line starting at buf[s] (chunk-local), with the chunk's newline / comma bitmask
// words nlm / cmm; lim = bytes of text staged from s on (<= kMaxLine + 1 is enough to decide).
__device__ LineOut parse_line(const uint8_t* buf, const uint32_t* nlm, const uint32_t* cmm, uint32_t s,
                              uint32_t lim, int64_t tz_ms) {
    LineOut o;
    o.ts = 0; o.bytes = 0; o.src = 0; o.dst = 0;
    // the end and the commas that bound fields 1, 5, 8 and 21 (comma ordinals 0, 3-4, 6-7, 19-20)
    // the ordinals 0, 3, 4, 6, 7, 19, 20 packed as 5-bit fields (no indexed local array)
    constexpr uint64_t kT = 0ull | 3ull << 5 | 4ull << 10 | 6ull << 15 | 7ull << 20 | 19ull << 25 | 20ull << 30;
    auto target = [&](uint32_t i) { return (uint32_t)(kT >> (5u * i)) & 31u; };
    uint32_t nc = 0, ti = 0, c0 = 0, c3 = 0, c4 = 0, c6 = 0, c7 = 0, c19 = 0, c20 = 0;
    uint32_t e = 0xFFFFFFFFu;                         // offset of '\n' from s
    const uint32_t stop = min(lim, kMaxLine + 1u);
    for (uint32_t wi = s >> 5; wi * 32u < s + stop; ++wi) {
        const uint32_t base = wi * 32u;
        uint32_t valid = 0xFFFFFFFFu;
        if (base < s) valid <<= (s - base);           // bytes before the line start
        const uint32_t rem = s + stop - base;
        if (rem < 32u) valid &= (1u << rem) - 1u;
        const uint32_t nl = nlm[wi] & valid;
        uint32_t cm = cmm[wi] & valid;
        if (nl) {
            const uint32_t bp = __ffs(nl) - 1u;
            e = base + bp - s;
            cm &= (1u << bp) - 1u;                     // commas before the newline only
        }
        const uint32_t c = __popc(cm);
        while (ti < 7u && target(ti) < nc + c) {
            const uint32_t q = base + nth_bit(cm, target(ti) - nc);
            c0 = ti == 0u ? q : c0;
            c3 = ti == 1u ? q : c3;
            c4 = ti == 2u ? q : c4;
            c6 = ti == 3u ? q : c6;
            c7 = ti == 4u ? q : c7;
            c19 = ti == 5u ? q : c19;
            c20 = ti == 6u ? q : c20;
            ++ti;
        }
        nc += c;
        if (e != 0xFFFFFFFFu) break;
    }
    uint32_t len = (e == 0xFFFFFFFFu) ? stop : e;   // content length (no '\n')
    if (len > kMaxLine) { o.status = kLineLong; return o; }
    // a '\r' before the '\n' can only end field No. 24, which is not read
    if (nc != 23u) { o.status = kLineColumns; return o; }
    if (c0 - s != 23u || !parse_time(buf + s, tz_ms, o.ts)) { o.status = kLineTime; return o; }
    if (!parse_ipv4(buf + c3 + 1u, c4 - c3 - 1u, o.src)) { o.status = kLineSrc; return o; }
    if (!parse_ipv4(buf + c6 + 1u, c7 - c6 - 1u, o.dst)) { o.status = kLineDst; return o; }
    if (!parse_u64(buf + c19 + 1u, c20 - c19 - 1u, o.bytes)) { o.status = kLineBytes; return o; }
    o.status = kLineOk;
    return o;
}

// exclusive block scan of one u32 per thread; returns the exclusive prefix, *total the sum
__device__ __forceinline__ uint32_t block_scan(uint32_t v, uint32_t* s_w, uint32_t* total) {
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, d);
        if (lane >= (uint32_t)d) x += y;
    }
    if (lane == 31u) s_w[warp] = x;
    __syncthreads();
    uint32_t base = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < kPT / 32; ++w) {
        const uint32_t t = s_w[w];
        if ((uint32_t)w < warp) base += t;
        tot += t;
    }
    __syncthreads();
    *total = tot;
    return base + x - v;
}

// Decoupled look-back over one chained scan, in two steps so that a CTA can publish a
// chunk's aggregate as soon as it is parsed and look back later (after parsing its next
// chunk), when the predecessors have published theirs.
// publish_agg: thread 0; chunk 0 publishes its inclusive value at once.
__device__ __forceinline__ void publish_agg(unsigned long long* st, uint64_t c, uint64_t agg) {
    st_relaxed_u64(st + c, (c == 0 ? kFlagInc : kFlagAgg) | agg);
}
// finish_look_back: warp 0; returns the exclusive prefix of chunk c (the sum over all
// earlier chunks) and publishes its inclusive value.  A window covers 256 predecessors,
// 8 consecutive ones per lane loaded together (one round trip per window): the nearest
// chunk with an inclusive value is typically a wave of CTAs (hundreds of chunks) back.
__device__ uint64_t finish_look_back(unsigned long long* st, uint64_t c, uint64_t agg) {
    constexpr int kQ = 8;
    const uint32_t lane = threadIdx.x & 31u;
    if (c == 0) return 0;
    uint64_t excl = 0;
    int64_t j = (int64_t)c - 1;
    for (;;) {
        uint64_t w[kQ];
#pragma unroll
        for (int q = 0; q < kQ; ++q) {
            const int64_t idx = j - (int64_t)lane * kQ - q;   // q = 0: this lane's nearest
            w[q] = idx >= 0 ? ld_relaxed_u64(st + idx) : kFlagInc;
        }
        // wait until every inspected predecessor has published something
        for (;;) {
            bool missing = false;
#pragma unroll
            for (int q = 0; q < kQ; ++q) missing |= (w[q] >> 62) == 0ull;
            if (!__any_sync(0xFFFFFFFFu, missing)) break;
            __nanosleep(64);
#pragma unroll
            for (int q = 0; q < kQ; ++q)
                if ((w[q] >> 62) == 0ull) w[q] = ld_relaxed_u64(st + (j - (int64_t)lane * kQ - q));
        }
        uint32_t incm = 0;
#pragma unroll
        for (int q = 0; q < kQ; ++q) incm |= ((w[q] >> 62) == 2ull ? 1u : 0u) << q;
        const uint32_t inc_lanes = __ballot_sync(0xFFFFFFFFu, incm != 0u);
        // everything nearer than the nearest inclusive predecessor, and that one, contributes
        const uint32_t L = inc_lanes ? (uint32_t)(__ffs(inc_lanes) - 1) : 32u;
        const uint32_t qinc = incm ? (uint32_t)(__ffs(incm) - 1) : (uint32_t)kQ;
        uint64_t v = 0;
#pragma unroll
        for (int q = 0; q < kQ; ++q)
            if (lane < L || (lane == L && (uint32_t)q <= qinc)) v += w[q] & kValMask;
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, d);
        excl += v;
        if (inc_lanes) break;
        j -= 32 * kQ;
    }
    if (lane == 0) st_relaxed_u64(st + c, kFlagInc | (excl + agg));
    return excl;
}

#ifndef SINET_PARSE_CTAS
#define SINET_PARSE_CTAS 8   // resident CTAs per SM (registers <= 64 per thread; measured 1.00 ms vs 1.08 at 6)
#endif
__global__ void __launch_bounds__(kPT, SINET_PARSE_CTAS) k_parse_text(ParseParams p) {
    static_assert(kLPT == 1, "one line per thread per round (the pending chunk keeps one result per thread)");
    constexpr uint32_t kWPT = kChunk / 32u / kPT;       // owned bitmask words per thread
    extern __shared__ __align__(128) uint8_t s_buf[];   // kBufAlloc: the staged chunk
    __shared__ __align__(8) uint64_t s_bar;
    __shared__ uint16_t s_start[kLCap];
    __shared__ uint32_t s_nlm[kWords], s_cmm[kWords];   // newline / comma bitmasks of the current chunk
    __shared__ uint32_t s_w[kPT / 32];
    __shared__ uint64_t s_next, s_base[2];
    __shared__ uint32_t s_stat[8];
    __shared__ uint64_t s_firstbad;

    const uint32_t tid = threadIdx.x;
    // thread 0: take the next ticket and stage its chunk into the (single) buffer, once every
    // thread's reads of it are done (the proxy fence orders them before the TMA writes)
    auto next_chunk = [&]() {
        const uint64_t cn = atomicAdd(p.ticket, 1ull);
        s_next = cn;
        if (cn < p.n_chunks) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            stage_chunk(p, cn * kChunk, s_buf, &s_bar);
        }
    };
    if (tid == 0) {
        mbar_init(&s_bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        next_chunk();
    }
    if (tid < 8) s_stat[tid] = 0;
    if (tid == 0) s_firstbad = ~0ull;
    __syncthreads();
    uint64_t c = s_next;
    uint32_t phase = 0;
    const int64_t tz_ms = (int64_t)p.tz_offset_min * 60000;

    // write one parsed line: status, per-status count, the record (if valid) at output index o
    auto write_line = [&](const LineOut& r, uint64_t line, uint64_t o) {
        if (r.status == kNoLine) return;
        if (p.status && line < p.status_cap) p.status[line] = (uint8_t)r.status;
        atomicAdd(&s_stat[r.status], 1u);
        if (r.status == kLineOk) {
            if (o < p.cap) {
                p.ts[o] = r.ts;
                p.src[o] = r.src;
                p.dst[o] = r.dst;
                p.bytes[o] = r.bytes;
            }
        } else {
            atomicMin(reinterpret_cast<unsigned long long*>(&s_firstbad), (unsigned long long)line);
        }
    };

    // publish chunk c's (lines, valid) aggregates (thread 0): one packed word when the
    // text is < 2 GiB (both prefix sums then fit 31 bits), else one word per scan
    auto publish_counts = [&](uint32_t n_lines, uint32_t n_valid) {
        if (p.packed) {
            publish_agg(p.st_lines, c, ((uint64_t)n_lines << 31) | n_valid);
        } else {
            publish_agg(p.st_lines, c, n_lines);
            publish_agg(p.st_valid, c, n_valid);
        }
    };
    // the previous single-round chunk: parsed, aggregates published, look-back + writes pending
    bool pend = false;
    uint64_t pc = 0;
    uint32_t p_lines = 0, p_valid = 0, p_vpre = 0;
    LineOut pres;
    pres.status = kNoLine;
    auto finish_pending = [&]() {   // block-uniform
        if (!pend) return;
        if (tid < 32) {
            uint64_t lb, vb;
            if (p.packed) {   // one scan of (lines << 31 | valid)
                const uint64_t x = finish_look_back(p.st_lines, pc, ((uint64_t)p_lines << 31) | p_valid);
                lb = x >> 31;
                vb = x & kHalfMask;
            } else {
                lb = finish_look_back(p.st_lines, pc, p_lines);
                vb = finish_look_back(p.st_valid, pc, p_valid);
            }
            if (tid == 0) { s_base[0] = lb; s_base[1] = vb; }
        }
        __syncthreads();
        write_line(pres, s_base[0] + tid, s_base[1] + p_vpre);
        __syncthreads();                               // s_base is rewritten
        pend = false;
    };

    while (c < p.n_chunks) {
        mbar_wait(&s_bar, phase);
        phase ^= 1u;
        const uint8_t* buf = s_buf;
        const uint64_t off = c * kChunk;
        const uint32_t staged = (uint32_t)min((uint64_t)kBuf, p.len - off);
        // newline at chunk-local x starts a line iff x < kChunk and off + x < len - 1
        const uint32_t nl_lim = (uint32_t)min((uint64_t)kChunk, (uint64_t)(p.len - 1ull - off));
        const uint32_t head = (c == 0) ? 1u : 0u;      // the line at offset 0

        // ---- structural index: newline and comma bitmasks of the staged bytes
        for (uint32_t w = tid; w < kWords; w += kPT) {
            const uint32_t a = w * 32u;
            uint32_t nl = 0u, cm = 0u;
            if (a < staged) {
                const uint4 v0 = *reinterpret_cast<const uint4*>(buf + a);
                const uint4 v1 = *reinterpret_cast<const uint4*>(buf + a + 16u);
                nl = eq_mask32(v0, v1, 0x0A0A0A0Au);
                cm = eq_mask32(v0, v1, 0x2C2C2C2Cu);
                if (staged - a < 32u) {
                    const uint32_t keep = (1u << (staged - a)) - 1u;
                    nl &= keep;
                    cm &= keep;
                }
            }
            s_nlm[w] = nl;
            s_cmm[w] = cm;
        }
        __syncthreads();

        // ---- lines of this chunk: the newlines it owns, counted per thread, block scan
        auto owned = [&](uint32_t w) -> uint32_t {    // bits of word w at chunk-local x < nl_lim
            const uint32_t b0 = w * 32u;
            if (b0 + 32u <= nl_lim) return 0xFFFFFFFFu;
            return b0 >= nl_lim ? 0u : (1u << (nl_lim - b0)) - 1u;
        };
        uint32_t my_nl = 0;
#pragma unroll
        for (uint32_t k = 0; k < kWPT; ++k) my_nl += __popc(s_nlm[tid * kWPT + k] & owned(tid * kWPT + k));
        uint32_t n_lines;
        const uint32_t my_first = block_scan(my_nl, s_w, &n_lines) + head;
        n_lines += head;

        // ---- parse in rounds of kLCap lines (thread t: line t of a round)
        const uint32_t rounds = (n_lines + kLCap - 1u) / kLCap;
        LineOut res;
        auto parse_round = [&](uint32_t r) -> uint32_t {
            const uint32_t r0 = r * kLCap, r1 = min(r0 + kLCap, n_lines);
            if (head && r == 0 && tid == 0) s_start[0] = 0;
            uint32_t idx = my_first;
            for (uint32_t k = 0; k < kWPT && idx < r1; ++k) {
                uint32_t m = s_nlm[tid * kWPT + k] & owned(tid * kWPT + k);
                while (m) {
                    const uint32_t bpos = __ffs(m) - 1u;
                    m &= m - 1u;
                    if (idx >= r0 && idx < r1) s_start[idx - r0] = (uint16_t)((tid * kWPT + k) * 32u + bpos + 1u);
                    ++idx;
                }
            }
            __syncthreads();
            const uint32_t i = r0 + tid;
            res.status = kNoLine;
            if (i < r1) {
                const uint32_t st = s_start[i - r0];
                res = parse_line(buf, s_nlm, s_cmm, st, staged > st ? staged - st : 0u, tz_ms);
            }
            __syncthreads();                           // s_start is rewritten by the next round
            return res.status == kLineOk ? 1u : 0u;
        };
        if (rounds <= 1u) {
            // the common case: parse once, publish the chunk's counts, then finish the previous
            // chunk (whose predecessors have had a chunk's time to publish) and keep this one
            const uint32_t my_valid = rounds ? parse_round(0) : 0u;
            uint32_t n_valid;
            const uint32_t vpre = block_scan(my_valid, s_w, &n_valid);
            if (tid == 0) {
                publish_counts(n_lines, n_valid);
                next_chunk();   // the buffer is free: the next chunk streams in during the look-back
            }
            finish_pending();
            pend = true;
            pc = c;
            p_lines = n_lines;
            p_valid = n_valid;
            p_vpre = vpre;
            pres = res;
        } else {
            // very short lines: count every round, look back, then re-parse and write
            finish_pending();
            uint32_t n_valid = 0, rv;
            for (uint32_t r = 0; r < rounds; ++r) {
                block_scan(parse_round(r), s_w, &rv);
                n_valid += rv;
            }
            if (tid == 0) publish_counts(n_lines, n_valid);
            if (tid < 32) {
                uint64_t lb, vb;
                if (p.packed) {
                    const uint64_t x = finish_look_back(p.st_lines, c, ((uint64_t)n_lines << 31) | n_valid);
                    lb = x >> 31;
                    vb = x & kHalfMask;
                } else {
                    lb = finish_look_back(p.st_lines, c, n_lines);
                    vb = finish_look_back(p.st_valid, c, n_valid);
                }
                if (tid == 0) { s_base[0] = lb; s_base[1] = vb; }
            }
            __syncthreads();
            const uint64_t lb = s_base[0];
            uint64_t o = s_base[1];
            for (uint32_t r = 0; r < rounds; ++r) {
                const uint32_t vpre = block_scan(parse_round(r), s_w, &rv);
                write_line(res, lb + r * kLCap + tid, o + vpre);
                o += rv;
            }
            if (tid == 0) next_chunk();
        }
        __syncthreads();                               // s_next is set
        c = s_next;
    }
    finish_pending();
    __syncthreads();
    if (tid < 7 && s_stat[tid]) atomicAdd(reinterpret_cast<unsigned long long*>(p.result + 3 + tid),
                                          (unsigned long long)s_stat[tid]);
    if (tid == 0 && s_firstbad != ~0ull) atomicMin(reinterpret_cast<unsigned long long*>(p.result + 2),
                                                   (unsigned long long)s_firstbad);
}

}  // namespace

size_t parse_smem_bytes() { return kBufAlloc; }

cudaError_t launch_parse_text(const ParseParams& p, int sm_count, cudaStream_t st) {
    static bool init = false;
    if (!init) {
        cudaError_t e = cudaFuncSetAttribute(k_parse_text, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)parse_smem_bytes());
        if (e != cudaSuccess) return e;
        init = true;
    }
    int per_sm = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_parse_text, kPT, parse_smem_bytes());
    if (e != cudaSuccess) return e;
    const uint64_t grid = min((uint64_t)sm_count * (uint64_t)(per_sm > 0 ? per_sm : 1), p.n_chunks);
    if (grid == 0) return cudaSuccess;
    k_parse_text<<<(unsigned)grid, kPT, parse_smem_bytes(), st>>>(p);
    return cudaGetLastError();
}

}  // namespace sinet
