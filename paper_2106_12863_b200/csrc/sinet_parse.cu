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
// B200 design: one pass over the text in HBM.  Persistent CTAs take 48 KB chunks
// by ticket; each chunk (+ a 2 KB tail for the line that crosses its end) is
// staged into shared memory by a TMA bulk copy (cp.async.bulk, mbarrier
// completion), double buffered so the next chunk streams in while this one is
// parsed.  A chunk owns the lines that start right after one of its newlines
// (chunk 0 also the line at offset 0).  The CTA counts them (block scan), one
// thread parses one line from shared memory, and the chunk's (lines, valid)
// counts go through a decoupled look-back (two chained scans) that gives the
// line index and the output index of its first line, so valid records are
// compacted in line order without a second pass over the text.
#include <cstdint>
#include <cuda_runtime.h>

#include "sinet_parse.h"

namespace sinet {
namespace {

constexpr int kPT = 256;                       // threads per CTA
constexpr uint32_t kChunk = kParseChunk;       // bytes owned per chunk
constexpr uint32_t kTail = 2048;               // staged beyond the chunk: max line 2047 + '\n'
constexpr uint32_t kBuf = kChunk + kTail;      // staged bytes per buffer
constexpr uint32_t kBufAlloc = kBuf + 16;      // + slack: the word loop may read 3 bytes past the text
constexpr int kLPT = 2;                        // lines per thread per round
constexpr uint32_t kLCap = kPT * kLPT;         // lines per round
constexpr uint32_t kMaxLine = 2047;
constexpr uint32_t kNoLine = 0xFFu;
constexpr uint64_t kFlagAgg = 1ull << 62, kFlagInc = 2ull << 62, kValMask = (1ull << 62) - 1;
static_assert(kChunk % (16 * kPT) == 0, "each thread scans a whole number of 16-byte words");

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
__device__ __forceinline__ uint64_t ld_acquire_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
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

// Parse the line starting at buf[s] (chunk-local); lim = bytes of text staged from
// s on that belong to the text (<= kMaxLine + 1 is enough to decide).
__device__ LineOut parse_line(const uint8_t* buf, uint32_t s, uint32_t lim, int64_t tz_ms) {
    LineOut o;
    o.ts = 0; o.bytes = 0; o.src = 0; o.dst = 0;
    // scan for the end and the commas that bound fields 1, 5, 8 and 21 (0-based 0, 4, 7, 20)
    uint32_t nc = 0, c0 = 0, c3 = 0, c4 = 0, c6 = 0, c7 = 0, c19 = 0, c20 = 0;
    uint32_t e = 0xFFFFFFFFu;                         // offset of '\n' from s
    const uint32_t stop = min(lim, kMaxLine + 1u);
    uint32_t w0 = s & ~3u;                            // aligned word loop over [s, s + stop)
    for (uint32_t a = w0; a < s + stop && e == 0xFFFFFFFFu; a += 4u) {
        const uint32_t w = *reinterpret_cast<const uint32_t*>(buf + a);
        uint32_t valid = 0xFFFFFFFFu;
        if (a < s) valid <<= 8u * (s - a);            // bytes before the line start
        const uint32_t rem = s + stop - a;
        if (rem < 4u) valid &= (1u << (8u * rem)) - 1u;
        const uint32_t nl = __vcmpeq4(w, 0x0A0A0A0Au) & valid;
        uint32_t cm = __vcmpeq4(w, 0x2C2C2C2Cu) & valid;
        if (nl) {
            const uint32_t bpos = (__ffs(nl) - 1u) >> 3;
            e = a + bpos - s;
            cm &= (1u << (8u * bpos)) - 1u;            // commas before the newline only
        }
        while (cm) {
            const uint32_t bpos = (__ffs(cm) - 1u) >> 3;
            cm &= ~(0xFFu << (8u * bpos));
            const uint32_t q = a + bpos;
            if (nc == 0u) c0 = q;
            if (nc == 3u) c3 = q;
            if (nc == 4u) c4 = q;
            if (nc == 6u) c6 = q;
            if (nc == 7u) c7 = q;
            if (nc == 19u) c19 = q;
            if (nc == 20u) c20 = q;
            ++nc;
        }
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

// Decoupled look-back over one chained scan: publishes this chunk's aggregate, returns
// the exclusive prefix (sum of all earlier chunks) and publishes the inclusive value.
// Called by warp 0; lane k inspects predecessor chunk (c - 1 - k) of each window.
__device__ uint64_t look_back(unsigned long long* st, uint64_t c, uint64_t agg) {
    const uint32_t lane = threadIdx.x & 31u;
    if (c == 0) {
        if (lane == 0) st_release_u64(st, kFlagInc | agg);
        return 0;
    }
    if (lane == 0) st_release_u64(st + c, kFlagAgg | agg);
    uint64_t excl = 0;
    int64_t j = (int64_t)c - 1;
    for (;;) {
        const int64_t idx = j - (int64_t)lane;
        uint64_t w = idx >= 0 ? ld_acquire_u64(st + idx) : kFlagInc;
        // wait until every inspected predecessor has published something
        while (__any_sync(0xFFFFFFFFu, (w >> 62) == 0ull)) {
            if ((w >> 62) == 0ull) w = ld_acquire_u64(st + idx);
        }
        const uint32_t inc = __ballot_sync(0xFFFFFFFFu, (w >> 62) == 2ull);
        // lanes up to and including the nearest inclusive predecessor contribute
        const uint32_t upto = inc ? (__ffs(inc) - 1u) : 31u;
        uint64_t v = (lane <= upto) ? (w & kValMask) : 0ull;
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, d);
        excl += v;
        if (inc) break;
        j -= 32;
    }
    if (lane == 0) st_release_u64(st + c, kFlagInc | (excl + agg));
    return excl;
}

__global__ void __launch_bounds__(kPT, 2) k_parse_text(ParseParams p) {
    extern __shared__ __align__(128) uint8_t s_buf[];   // 2 x kBufAlloc
    __shared__ __align__(8) uint64_t s_bar[2];
    __shared__ uint16_t s_start[kLCap];
    __shared__ uint32_t s_w[kPT / 32];
    __shared__ uint64_t s_next, s_base[2];
    __shared__ uint32_t s_stat[8];
    __shared__ uint64_t s_firstbad;

    const uint32_t tid = threadIdx.x;
    if (tid == 0) {
        mbar_init(&s_bar[0], 1);
        mbar_init(&s_bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        const uint64_t c0 = atomicAdd(p.ticket, 1ull);
        s_next = c0;
        if (c0 < p.n_chunks) stage_chunk(p, c0 * kChunk, s_buf, &s_bar[0]);
    }
    if (tid < 8) s_stat[tid] = 0;
    if (tid == 0) s_firstbad = ~0ull;
    __syncthreads();
    uint64_t c = s_next;
    uint32_t stage = 0, phase[2] = {0u, 0u};

    while (c < p.n_chunks) {
        __syncthreads();                               // everyone has read s_next
        if (tid == 0) {                                // next ticket; its chunk streams in meanwhile
            const uint64_t cn = atomicAdd(p.ticket, 1ull);
            s_next = cn;
            if (cn < p.n_chunks) stage_chunk(p, cn * kChunk, s_buf + (stage ^ 1u) * kBufAlloc, &s_bar[stage ^ 1u]);
        }
        mbar_wait(&s_bar[stage], phase[stage]);
        phase[stage] ^= 1u;
        const uint8_t* buf = s_buf + stage * kBufAlloc;
        const uint64_t off = c * kChunk;
        const uint32_t cl = (uint32_t)min((uint64_t)kChunk, p.len - off);       // owned bytes
        const uint32_t staged = (uint32_t)min((uint64_t)kBuf, p.len - off);
        // newline at chunk-local x starts a line iff off + x < len - 1
        const uint32_t nl_lim = (uint32_t)min((uint64_t)cl, (uint64_t)(p.len - 1ull - off));
        const uint32_t head = (c == 0) ? 1u : 0u;      // the line at offset 0

        // ---- lines of this chunk: newlines per thread (16-byte words), block scan
        constexpr uint32_t kSeg = kChunk / kPT;
        const uint32_t a0 = tid * kSeg;
        auto nl_mask = [&](uint32_t a, uint4 v, int k) {
            const uint32_t w = k == 0 ? v.x : k == 1 ? v.y : k == 2 ? v.z : v.w;
            uint32_t m = __vcmpeq4(w, 0x0A0A0A0Au);
            const uint32_t base = a + 4u * k;
            if (base + 4u > nl_lim) m &= base >= nl_lim ? 0u : (1u << (8u * (nl_lim - base))) - 1u;
            return m;
        };
        uint32_t my_nl = 0;
        for (uint32_t a = a0; a < a0 + kSeg && a < nl_lim; a += 16u) {
            const uint4 v = *reinterpret_cast<const uint4*>(buf + a);
#pragma unroll
            for (int k = 0; k < 4; ++k) my_nl += __popc(nl_mask(a, v, k)) >> 3;
        }
        uint32_t n_lines;
        const uint32_t my_first = block_scan(my_nl, s_w, &n_lines) + head;
        n_lines += head;
        const int64_t tz_ms = (int64_t)p.tz_offset_min * 60000;

        // ---- parse in rounds of kLCap lines (thread t: lines t*kLPT .. t*kLPT+kLPT-1 of a round)
        const uint32_t rounds = (n_lines + kLCap - 1u) / kLCap;
        LineOut res[kLPT];
        auto parse_round = [&](uint32_t r) -> uint32_t {
            const uint32_t r0 = r * kLCap, r1 = min(r0 + kLCap, n_lines);
            if (head && r == 0 && tid == 0) s_start[0] = 0;
            uint32_t idx = my_first;
            for (uint32_t a = a0; a < a0 + kSeg && a < nl_lim && idx < r1; a += 16u) {
                const uint4 v = *reinterpret_cast<const uint4*>(buf + a);
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    uint32_t m = nl_mask(a, v, k);
                    while (m) {
                        const uint32_t bpos = (__ffs(m) - 1u) >> 3;
                        m &= ~(0xFFu << (8u * bpos));
                        if (idx >= r0 && idx < r1) s_start[idx - r0] = (uint16_t)(a + 4u * k + bpos + 1u);
                        ++idx;
                    }
                }
            }
            __syncthreads();
            uint32_t my_valid = 0;
#pragma unroll
            for (int u = 0; u < kLPT; ++u) {
                const uint32_t i = r0 + tid * kLPT + u;
                res[u].status = kNoLine;
                if (i < r1) {
                    const uint32_t st = s_start[i - r0];
                    res[u] = parse_line(buf, st, staged > st ? staged - st : 0u, tz_ms);
                    my_valid += res[u].status == kLineOk ? 1u : 0u;
                }
            }
            __syncthreads();                           // s_start is rewritten by the next round
            return my_valid;
        };
        auto write_round = [&](uint32_t r, uint64_t line_base, uint64_t o) {
            const uint32_t r0 = r * kLCap;
#pragma unroll
            for (int u = 0; u < kLPT; ++u) {
                if (res[u].status == kNoLine) continue;
                const uint64_t line = line_base + r0 + tid * kLPT + u;
                if (p.status && line < p.status_cap) p.status[line] = (uint8_t)res[u].status;
                atomicAdd(&s_stat[res[u].status], 1u);
                if (res[u].status == kLineOk) {
                    if (o < p.cap) {
                        p.ts[o] = res[u].ts;
                        p.src[o] = res[u].src;
                        p.dst[o] = res[u].dst;
                        p.bytes[o] = res[u].bytes;
                    }
                    ++o;
                } else {
                    atomicMin(reinterpret_cast<unsigned long long*>(&s_firstbad), (unsigned long long)line);
                }
            }
        };
        auto bases = [&](uint32_t n_valid) {    // decoupled look-back of both counts (warp 0)
            if (tid < 32) {
                const uint64_t lb = look_back(p.st_lines, c, n_lines);
                const uint64_t vb = look_back(p.st_valid, c, n_valid);
                if (tid == 0) { s_base[0] = lb; s_base[1] = vb; }
            }
            __syncthreads();
        };
        if (rounds <= 1u) {                    // the common case: parse once, keep results in registers
            const uint32_t my_valid = rounds ? parse_round(0) : 0u;
            uint32_t n_valid;
            const uint32_t vpre = block_scan(my_valid, s_w, &n_valid);
            bases(n_valid);
            if (rounds) write_round(0, s_base[0], s_base[1] + vpre);
        } else {                               // very short lines: count every round, then re-parse and write
            uint32_t n_valid = 0, rv;
            for (uint32_t r = 0; r < rounds; ++r) {
                block_scan(parse_round(r), s_w, &rv);
                n_valid += rv;
            }
            bases(n_valid);
            uint64_t o = s_base[1];
            for (uint32_t r = 0; r < rounds; ++r) {
                const uint32_t vpre = block_scan(parse_round(r), s_w, &rv);
                write_round(r, s_base[0], o + vpre);
                o += rv;
            }
        }
        __syncthreads();                               // buffer free for the next-but-one stage
        c = s_next;
        stage ^= 1u;
    }
    __syncthreads();
    if (tid < 7 && s_stat[tid]) atomicAdd(reinterpret_cast<unsigned long long*>(p.result + 3 + tid),
                                          (unsigned long long)s_stat[tid]);
    if (tid == 0 && s_firstbad != ~0ull) atomicMin(reinterpret_cast<unsigned long long*>(p.result + 2),
                                                   (unsigned long long)s_firstbad);
}

}  // namespace

size_t parse_smem_bytes() { return 2u * kBufAlloc; }

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
