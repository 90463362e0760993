/*
 * sinet_oracle.c -- the plain, slow, obviously-correct CPU ORACLE for the
 * SINET discrimination + millisecond-histogram hot path (arXiv 2106.12863).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or constant with the CUDA path under
 * paper_2106_12863_b200/ and include/ (it does not include them and they do
 * not include it).
 *
 * Citations: "P:Lnn" = line nn of the paper text; section numbers
 * follow the paper.  Readings where the paper is silent or ambiguous are the
 * A1..A23 list in DESIGN.md ("Readings").
 *
 * Everything is integer arithmetic; u64 sums wrap modulo 2^64 (reading A18).
 *
 * Pinned by tests/test_oracle_*.py against: the worked values of the paper's
 * operations (bitmask S:L196-198 / P:L160-161), brute-force 32-character
 * bit-string prefix comparison, Python's ipaddress module, collections.Counter
 * histograms, the hand-derived fixture tests/golden/f0.json, closed-form
 * invariants (conservation, permutation/chunk/shard invariance) and the
 * generator's construction-time ground truth.
 */
#include <stdint.h>
#include <stddef.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

/* ---------------------------------------------------------------------- */
/* Alg. 1 lines 6-7: SB = bitmask(X.X.X.X, Z), CB = bitmask(Y.Y.Y.Y, Z).
 * "translated to a 32-bit sequence": keep the Z leading bits of
 * the 32-bit address, clear the remaining 32-Z.  Z in [0,32] (reading A10);
 * Z == 0 is special-cased because a C shift by 32 is undefined.             */
uint32_t oracle_mask(uint32_t z)
{
    if (z == 0) return 0u;
    return 0xFFFFFFFFu << (32u - z);
}

uint32_t oracle_bitmask(uint32_t addr, uint32_t z)
{
    return addr & oracle_mask(z);
}

/* Alg. 1 lines 4-9 applied to one address against the whole
 * "CIDR list", match-any (reading A3), the block's Z masking both
 * sides (reading A4), and "Instead of matching S.D. to C.B., we use minus at
 * line 8": result = SB - CB in unsigned 32-bit arithmetic, a match
 * iff result == 0 (reading A5).  Linear scan, no precompiled table.         */
int oracle_member(uint32_t ip, const uint32_t* nets, const uint8_t* lens, uint32_t p)
{
    for (uint32_t i = 0; i < p; ++i) {
        uint32_t z = lens[i];
        uint32_t sb = oracle_bitmask(ip, z);        /* Alg.1 l.6 */
        uint32_t cb = oracle_bitmask(nets[i], z);   /* Alg.1 l.7 (normalises host bits, A9) */
        uint32_t result = sb - cb;                  /* Alg.1 l.8 */
        if (result == 0u) return 1;                 /* Alg.1 l.9 */
    }
    return 0;
}

/* Direction codes of the output: 0 = OUT (outgoing), 1 = IN (ingoing),
 * 2 = NEITHER (not binned, reading A20).  lut[s_in*2 + d_in] -> direction
 * (reading A1/A2; presets ALG1 {IN,IN,OUT,OUT}, SRC_PRIORITY {NEI,IN,OUT,OUT},
 * STRICT {NEI,IN,OUT,NEI}).                                                  */

/* Totals layout (12 x u64), reading A14 and the north_star invariants:
 *   [0..3]  m_count[s_in*2+d_in]   -- every record, mode independent
 *   [4..7]  m_bytes[s_in*2+d_in]
 *   [8..9]  oow_count[dir]         -- dir in {OUT, IN}, ts outside the window
 *   [10..11] oow_bytes[dir]                                                  */

/* One record through the method, in the paper's order: discriminate first
 * ("each workload (chunk) ... is discriminated and marked as ingoing/outgoing"
 * before the map-reduce phase), then Map to a
 * millisecond key and Reduce by addition (P:L202-204,
 * P:L213-214). */
static void oracle_one(uint64_t ts, uint32_t src, uint32_t dst, uint64_t bytes,
                       const uint32_t* nets, const uint8_t* lens, uint32_t p,
                       uint64_t start, uint64_t window, uint32_t width,
                       const uint8_t lut[4], uint64_t nbins,
                       uint64_t* out_count, uint64_t* out_bytes, uint64_t* totals)
{
    int s_in = oracle_member(src, nets, lens, p);
    int d_in = oracle_member(dst, nets, lens, p);
    int cell = s_in * 2 + d_in;
    totals[0 + cell] += 1u;
    totals[4 + cell] += bytes;
    int dir = lut[cell];
    if (dir != 0 && dir != 1) return;                     /* NEITHER: not binned */
    if (ts < start || ts - start >= window) {             /* reading A14 */
        totals[8 + dir] += 1u;
        totals[10 + dir] += bytes;
        return;
    }
    uint64_t key = (ts - start) / (uint64_t)width;        /* Map, half-open bins (A15) */
    out_count[(uint64_t)dir * nbins + key] += 1u;         /* <timestamp, count> */
    out_bytes[(uint64_t)dir * nbins + key] += bytes;      /* <timestamp, bytes> */
}

/* Accumulates (does not clear) into out_count[2][nbins], out_bytes[2][nbins]
 * and totals[12], nbins = window / width.  Records in any order.             */
void oracle_classify_histogram(const uint64_t* ts, const uint32_t* src, const uint32_t* dst,
                               const uint64_t* bytes, uint64_t n,
                               const uint32_t* nets, const uint8_t* lens, uint32_t p,
                               uint64_t start, uint64_t window, uint32_t width,
                               const uint8_t lut[4],
                               uint64_t* out_count, uint64_t* out_bytes, uint64_t* totals)
{
    uint64_t nbins = window / width;
    for (uint64_t r = 0; r < n; ++r)
        oracle_one(ts[r], src[r], dst[r], bytes[r], nets, lens, p, start, window, width,
                   lut, nbins, out_count, out_bytes, totals);
}

/* Per-record tag: s_in | d_in << 1 | (ts outside window) << 2. */
void oracle_tags(const uint64_t* ts, const uint32_t* src, const uint32_t* dst, uint64_t n,
                 const uint32_t* nets, const uint8_t* lens, uint32_t p,
                 uint64_t start, uint64_t window, uint8_t* tags)
{
    for (uint64_t r = 0; r < n; ++r) {
        int s_in = oracle_member(src[r], nets, lens, p);
        int d_in = oracle_member(dst[r], nets, lens, p);
        int oow = (ts[r] < start || ts[r] - start >= window) ? 1 : 0;
        tags[r] = (uint8_t)(s_in | (d_in << 1) | (oow << 2));
    }
}

/* ---------------------------------------------------------------------- */
/* The same definition evaluated by several host threads, only to make the
 * full-size configurations finish in seconds.  Each thread owns a contiguous
 * slab of bins and scans every record, handling exactly the records whose
 * bin lies in its slab; thread 0 also handles every record that is not binned
 * (NEITHER or out of window).  Every record is therefore processed exactly
 * once, by oracle_one(), and the result is identical to the serial loop
 * because integer addition is associative and commutative.         */
typedef struct {
    const uint64_t* ts; const uint32_t* src; const uint32_t* dst; const uint64_t* bytes;
    uint64_t n; const uint32_t* nets; const uint8_t* lens; uint32_t p;
    uint64_t start, window; uint32_t width; const uint8_t* lut;
    uint64_t* out_count; uint64_t* out_bytes;
    uint64_t slab_lo, slab_hi;   /* bins [slab_lo, slab_hi) */
    int take_unbinned;
    uint64_t totals[12];
} oracle_job;

static void* oracle_worker(void* arg)
{
    oracle_job* j = (oracle_job*)arg;
    uint64_t nbins = j->window / j->width;
    memset(j->totals, 0, sizeof j->totals);
    for (uint64_t r = 0; r < j->n; ++r) {
        uint64_t ts = j->ts[r];
        int in_window = !(ts < j->start || ts - j->start >= j->window);
        if (in_window) {
            uint64_t key = (ts - j->start) / (uint64_t)j->width;
            if (key < j->slab_lo || key >= j->slab_hi) continue;
            /* binned or NEITHER-in-window: this slab's thread owns it */
        } else if (!j->take_unbinned) {
            continue;
        }
        oracle_one(ts, j->src[r], j->dst[r], j->bytes[r], j->nets, j->lens, j->p,
                   j->start, j->window, j->width, j->lut, nbins,
                   j->out_count, j->out_bytes, j->totals);
    }
    return NULL;
}

int oracle_classify_histogram_mt(const uint64_t* ts, const uint32_t* src, const uint32_t* dst,
                                 const uint64_t* bytes, uint64_t n,
                                 const uint32_t* nets, const uint8_t* lens, uint32_t p,
                                 uint64_t start, uint64_t window, uint32_t width,
                                 const uint8_t lut[4],
                                 uint64_t* out_count, uint64_t* out_bytes, uint64_t* totals,
                                 int threads)
{
    if (threads < 1) threads = 1;
    uint64_t nbins = window / width;
    oracle_job* jobs = (oracle_job*)calloc((size_t)threads, sizeof(oracle_job));
    pthread_t* tid = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
    if (!jobs || !tid) { free(jobs); free(tid); return -1; }
    for (int t = 0; t < threads; ++t) {
        oracle_job* j = &jobs[t];
        j->ts = ts; j->src = src; j->dst = dst; j->bytes = bytes; j->n = n;
        j->nets = nets; j->lens = lens; j->p = p;
        j->start = start; j->window = window; j->width = width; j->lut = lut;
        j->out_count = out_count; j->out_bytes = out_bytes;
        j->slab_lo = nbins * (uint64_t)t / (uint64_t)threads;
        j->slab_hi = nbins * (uint64_t)(t + 1) / (uint64_t)threads;
        j->take_unbinned = (t == 0);
    }
    int rc = 0;
    for (int t = 1; t < threads; ++t)
        if (pthread_create(&tid[t], NULL, oracle_worker, &jobs[t]) != 0) { rc = -1; threads = t; break; }
    oracle_worker(&jobs[0]);
    for (int t = 1; t < threads; ++t) pthread_join(tid[t], NULL);
    if (rc == 0)
        for (int t = 0; t < threads; ++t)
            for (int k = 0; k < 12; ++k) totals[k] += jobs[t].totals[k];
    free(jobs); free(tid);
    return rc;
}

/* ---------------------------------------------------------------------- */
/* NEXT-1: re-binning and sparse export of one (dir, metric) plane.
 * "Session data is grouped into one-hour frame bins" and counts
 * "in 10 minutes": coarse bin k of a plane of fine bins is the sum
 * of fine bins [k*factor, (k+1)*factor) (the last coarse bin may be partial).
 * u64 sums wrap mod 2^64 (reading A18).                                     */
void oracle_rebin(const uint64_t* fine, uint64_t nfine, uint64_t factor, uint64_t* coarse)
{
    uint64_t ncoarse = (nfine + factor - 1) / factor;
    for (uint64_t k = 0; k < ncoarse; ++k) coarse[k] = 0;
    for (uint64_t b = 0; b < nfine; ++b) coarse[b / factor] += fine[b];
}

/* Sparse series of one direction (the paper's key/value namespaces
 * X1<timestamp>, X1<count>, X2<timestamp>, X2<bytes>):
 * every bin with a nonzero count, ascending, as (bin start in epoch ms,
 * count, bytes).  Returns the number of entries written (<= capacity).     */
uint64_t oracle_sparse(const uint64_t* count, const uint64_t* bytes, uint64_t nbins,
                       uint64_t start, uint32_t width,
                       uint64_t* out_ts, uint64_t* out_count, uint64_t* out_bytes, uint64_t capacity)
{
    uint64_t k = 0;
    for (uint64_t b = 0; b < nbins; ++b) {
        if (count[b] == 0) continue;
        if (k < capacity) {
            out_ts[k] = start + b * (uint64_t)width;
            out_count[k] = count[b];
            out_bytes[k] = bytes[b];
        }
        ++k;
    }
    return k;
}

/* ---------------------------------------------------------------------- */
/* NEXT-2: watchlist filter.  The paper's second workload histograms only the
 * sessions of listed hosts: "we randomly pick up 300 IP addresses by using
 * AbuseIP blacklist API" and "877 IP addresses from US-CERT
 * report", with ingoing and outgoing series for each list
 * (Figs 8-11).  A record is kept iff its source OR its destination equals a
 * listed address (exact match; reading A24 in DESIGN.md); kept records then go
 * through the unchanged discrimination + histogram (filter, then histogram).
 * Linear scan of the list, no precompiled set.                              */
int oracle_watched(uint32_t ip, const uint32_t* list, uint32_t nlist)
{
    for (uint32_t i = 0; i < nlist; ++i)
        if (list[i] == ip) return 1;
    return 0;
}

/* Writes the indices of kept records to keep[] and returns how many. */
uint64_t oracle_watch_filter(const uint32_t* src, const uint32_t* dst, uint64_t n,
                             const uint32_t* list, uint32_t nlist, uint64_t* keep)
{
    uint64_t k = 0;
    for (uint64_t r = 0; r < n; ++r)
        if (oracle_watched(src[r], list, nlist) || oracle_watched(dst[r], list, nlist))
            keep[k++] = r;
    return k;
}

/* ---------------------------------------------------------------------- */
/* NEXT-4, labelled longest-prefix match.  A table entry Y/Z carries a label
 * (1 = SINET inside, 0 = carved out); an address is inside iff the longest
 * entry whose Alg. 1 test matches it (l.6-9) is labelled inside,
 * outside if no entry matches (reading A26 in DESIGN.md).  With every label 1
 * this is oracle_member().  Equal (net, Z) entries: the last one wins.
 * Linear scan, literal mask-and-subtract.                                   */
int oracle_member_lpm(uint32_t ip, const uint32_t* nets, const uint8_t* lens, const uint8_t* labels,
                      uint32_t p)
{
    int best_len = -1, best_label = 0;
    for (uint32_t i = 0; i < p; ++i) {
        uint32_t z = lens[i];
        uint32_t sb = oracle_bitmask(ip, z);
        uint32_t cb = oracle_bitmask(nets[i], z);
        if (sb - cb == 0u && (int)z >= best_len) {
            best_len = (int)z;
            best_label = labels[i] ? 1 : 0;
        }
    }
    return best_label;
}

/* Per-address membership under a labelled table (for the histogram oracle the
 * labelled table is applied through oracle_lpm_to_members(): it lists the
 * member addresses' membership bits for a batch). */
void oracle_member_lpm_batch(const uint32_t* ips, uint64_t n, const uint32_t* nets, const uint8_t* lens,
                             const uint8_t* labels, uint32_t p, uint8_t* out)
{
    for (uint64_t r = 0; r < n; ++r) out[r] = (uint8_t)oracle_member_lpm(ips[r], nets, lens, labels, p);
}

/* The histogram of oracle_classify_histogram with the memberships given per
 * record (s_in[r], d_in[r] in {0,1}), e.g. from oracle_member_lpm(): the same
 * steps after discrimination (LUT, window test, Map, Reduce).               */
void oracle_histogram_members(const uint64_t* ts, const uint8_t* s_in, const uint8_t* d_in,
                              const uint64_t* bytes, uint64_t n, uint64_t start, uint64_t window,
                              uint32_t width, const uint8_t lut[4],
                              uint64_t* out_count, uint64_t* out_bytes, uint64_t* totals)
{
    uint64_t nbins = window / width;
    for (uint64_t r = 0; r < n; ++r) {
        int cell = (s_in[r] ? 2 : 0) + (d_in[r] ? 1 : 0);
        totals[0 + cell] += 1u;
        totals[4 + cell] += bytes[r];
        int dir = lut[cell];
        if (dir != 0 && dir != 1) continue;
        if (ts[r] < start || ts[r] - start >= window) {
            totals[8 + dir] += 1u;
            totals[10 + dir] += bytes[r];
            continue;
        }
        uint64_t key = (ts[r] - start) / (uint64_t)width;
        out_count[(uint64_t)dir * nbins + key] += 1u;
        out_bytes[(uint64_t)dir * nbins + key] += bytes[r];
    }
}

/* ---------------------------------------------------------------------- */
/* Alg. 1 l.4-9 for a long CIDR list, grouped by Z.  The list
 * test is an OR over the entries (match-any, reading A3), so it may be
 * evaluated in any order of the entries: for each distinct Z of the list,
 *     SB = bitmask(ip, Z)                      (l.6)
 *     match iff SB - CB == 0 for some entry of length Z, CB = bitmask(net, Z) (l.7-9),
 * i.e. iff SB is one of the sorted CB values of length Z (a binary search, a
 * library-style step).  The same result as oracle_member(), in O(33 log P)
 * instead of O(P) per address; used only where the linear scan is too slow at
 * full size (C5: 4096 entries x 800 M addresses) and pinned equal to
 * oracle_member() in tests/test_oracle_pins.py.                             */
typedef struct { uint32_t* cb[33]; uint32_t n[33]; } oracle_bylen;

static int oracle_u32_cmp(const void* a, const void* b)
{
    uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    return (x > y) - (x < y);
}

static int oracle_bylen_member(const oracle_bylen* t, uint32_t ip)
{
    for (uint32_t z = 0; z <= 32; ++z) {
        if (!t->n[z]) continue;
        uint32_t sb = oracle_bitmask(ip, z);
        uint32_t lo = 0, hi = t->n[z];              /* first CB >= SB */
        while (lo < hi) {
            uint32_t mid = lo + (hi - lo) / 2;
            if (t->cb[z][mid] < sb) lo = mid + 1; else hi = mid;
        }
        if (lo < t->n[z] && t->cb[z][lo] - sb == 0u) return 1;
    }
    return 0;
}

typedef struct { const oracle_bylen* t; const uint32_t* ips; uint8_t* out; uint64_t lo, hi; } oracle_bylen_job;

static void* oracle_bylen_worker(void* arg)
{
    oracle_bylen_job* j = (oracle_bylen_job*)arg;
    for (uint64_t r = j->lo; r < j->hi; ++r) j->out[r] = (uint8_t)oracle_bylen_member(j->t, j->ips[r]);
    return NULL;
}

/* out[r] = membership of ips[r] in the list (0/1); threads share the batch. */
int oracle_member_bylen_batch(const uint32_t* ips, uint64_t n, const uint32_t* nets, const uint8_t* lens,
                              uint32_t p, uint8_t* out, int threads)
{
    oracle_bylen t;
    memset(&t, 0, sizeof t);
    for (uint32_t i = 0; i < p; ++i) if (lens[i] <= 32) t.n[lens[i]]++;
    int rc = 0;
    for (uint32_t z = 0; z <= 32; ++z) {
        if (t.n[z] && !(t.cb[z] = (uint32_t*)malloc(sizeof(uint32_t) * t.n[z]))) rc = -1;
        t.n[z] = 0;
    }
    if (rc == 0) {
        for (uint32_t i = 0; i < p; ++i) {
            uint32_t z = lens[i];
            if (z > 32) continue;
            t.cb[z][t.n[z]++] = oracle_bitmask(nets[i], z);   /* CB (l.7, normalises host bits) */
        }
        for (uint32_t z = 0; z <= 32; ++z) if (t.n[z]) qsort(t.cb[z], t.n[z], sizeof(uint32_t), oracle_u32_cmp);
        if (threads < 1) threads = 1;
        oracle_bylen_job* jobs = (oracle_bylen_job*)calloc((size_t)threads, sizeof(oracle_bylen_job));
        pthread_t* tid = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
        if (!jobs || !tid) rc = -1;
        else {
            for (int k = 0; k < threads; ++k) {
                jobs[k].t = &t; jobs[k].ips = ips; jobs[k].out = out;
                jobs[k].lo = n * (uint64_t)k / (uint64_t)threads;
                jobs[k].hi = n * (uint64_t)(k + 1) / (uint64_t)threads;
            }
            int started = threads;
            for (int k = 1; k < threads; ++k)
                if (pthread_create(&tid[k], NULL, oracle_bylen_worker, &jobs[k]) != 0) { rc = -1; started = k; break; }
            oracle_bylen_worker(&jobs[0]);
            for (int k = 1; k < started; ++k) pthread_join(tid[k], NULL);
        }
        free(jobs); free(tid);
    }
    for (uint32_t z = 0; z <= 32; ++z) free(t.cb[z]);
    return rc;
}

/* ---------------------------------------------------------------------- */
/* NEXT-3: session-log text -> the four columns the path reads.
 *
 * Table 1 ("PA-7080 data description") lists the 24 items of a
 * session record in order; the path needs No. 1 capture_time,
 * No. 5 source_ip, No. 8 destination_ip and No. 21 bytes
 * (P:L254).  The paper prints no file syntax; readings A27-A31
 * fix it: one record per line, '\n' separated (an optional '\r' before it is
 * dropped), 24 comma-separated fields in Table 1 order, capture_time as
 * "YYYY/MM/DD HH:MM:SS.mmm" (Table 1's sample value) in local time at
 * tz_offset_min minutes east of UTC, dotted-quad IPv4 addresses
 * ("translated to a 32-bit sequence"; first octet most
 * significant), bytes a decimal u64.  Other fields are opaque.
 *
 * Status per line (first failing check wins, in this order):
 *   0 OK, 1 LONG (content > 2047 bytes), 2 COLUMNS (not 24 fields),
 *   3 TIME, 4 SRC, 5 DST, 6 BYTES.
 * Valid lines are written to the output columns in line order (skip policy);
 * every line, valid or not, gets a status and a line number.
 *
 * Written as plain string handling: find the line, split it on every comma,
 * then parse the four fields character by character.                       */

#define ORACLE_PARSE_MAX_LINE 2047u

static int oracle_is_leap(uint32_t y)
{
    return (y % 4u == 0u && y % 100u != 0u) || y % 400u == 0u;
}

static uint32_t oracle_month_days(uint32_t y, uint32_t m)
{
    static const uint32_t days[12] = {31, 28, 31, 30, 31, 30, 31, 31, 30, 31, 30, 31};
    return (m == 2u && oracle_is_leap(y)) ? 29u : days[m - 1u];
}

/* Reads exactly k decimal digits at s into *v; 0 if any is not a digit. */
static int oracle_digits(const char* s, uint32_t k, uint32_t* v)
{
    uint32_t x = 0;
    for (uint32_t i = 0; i < k; ++i) {
        if (s[i] < '0' || s[i] > '9') return 0;
        x = x * 10u + (uint32_t)(s[i] - '0');
    }
    *v = x;
    return 1;
}

/* capture_time "YYYY/MM/DD HH:MM:SS.mmm" -> epoch ms (UTC) of that local time.
 * Days since 1970-01-01 are counted year by year and month by month (the
 * Gregorian calendar; Unix time has no leap seconds, reading A11).         */
int oracle_parse_time(const char* f, uint64_t len, int32_t tz_offset_min, uint64_t* out)
{
    uint32_t Y, M, D, h, mi, s, ms;
    if (len != 23u) return 0;
    if (f[4] != '/' || f[7] != '/' || f[10] != ' ' || f[13] != ':' || f[16] != ':' || f[19] != '.')
        return 0;
    if (!oracle_digits(f + 0, 4, &Y) || !oracle_digits(f + 5, 2, &M) || !oracle_digits(f + 8, 2, &D) ||
        !oracle_digits(f + 11, 2, &h) || !oracle_digits(f + 14, 2, &mi) ||
        !oracle_digits(f + 17, 2, &s) || !oracle_digits(f + 20, 3, &ms))
        return 0;
    if (Y < 1970u || M < 1u || M > 12u || D < 1u || D > oracle_month_days(Y, M)) return 0;
    if (h > 23u || mi > 59u || s > 59u) return 0;
    uint64_t days = 0;
    for (uint32_t y = 1970u; y < Y; ++y) days += oracle_is_leap(y) ? 366u : 365u;
    for (uint32_t m = 1u; m < M; ++m) days += oracle_month_days(Y, m);
    days += D - 1u;
    int64_t local_ms = (int64_t)((((days * 24u + h) * 60u + mi) * 60u + s) * 1000u + ms);
    int64_t utc_ms = local_ms - (int64_t)tz_offset_min * 60000;
    if (utc_ms < 0) return 0;
    *out = (uint64_t)utc_ms;
    return 1;
}

/* Dotted quad: four octets of 1-3 decimal digits, no leading zero unless the
 * octet is "0", each <= 255 (the strictness of Python's ipaddress module). */
int oracle_parse_ipv4(const char* f, uint64_t len, uint32_t* out)
{
    uint32_t value = 0, octets = 0;
    uint64_t i = 0;
    while (octets < 4u) {
        uint64_t b = i;
        uint32_t x = 0;
        while (i < len && f[i] >= '0' && f[i] <= '9') {
            x = x * 10u + (uint32_t)(f[i] - '0');
            ++i;
            if (i - b > 3u) return 0;
        }
        uint64_t nd = i - b;
        if (nd == 0u || x > 255u || (nd > 1u && f[b] == '0')) return 0;
        value = (value << 8) | x;
        ++octets;
        if (octets < 4u) {
            if (i >= len || f[i] != '.') return 0;
            ++i;
        }
    }
    if (i != len) return 0;
    *out = value;
    return 1;
}

/* bytes: 1 to 20 decimal digits, value < 2^64 ("NA" is an error, reading A30). */
int oracle_parse_u64(const char* f, uint64_t len, uint64_t* out)
{
    if (len == 0u || len > 20u) return 0;
    uint64_t x = 0;
    for (uint64_t i = 0; i < len; ++i) {
        if (f[i] < '0' || f[i] > '9') return 0;
        uint64_t d = (uint64_t)(f[i] - '0');
        if (x > (UINT64_MAX - d) / 10u) return 0;   /* x*10 + d would exceed 2^64 - 1 */
        x = x * 10u + d;
    }
    *out = x;
    return 1;
}

/* One line (content without its '\n'): status code, and on OK the four values. */
int oracle_parse_line(const char* line, uint64_t len, int32_t tz_offset_min,
                      uint64_t* ts, uint32_t* src, uint32_t* dst, uint64_t* bytes)
{
    if (len > ORACLE_PARSE_MAX_LINE) return 1;
    if (len > 0u && line[len - 1u] == '\r') --len;
    uint64_t fb[24], fe[24];           /* field i = line[fb[i], fe[i]) */
    uint32_t nf = 0;
    uint64_t b = 0;
    for (uint64_t i = 0; i <= len; ++i) {
        if (i == len || line[i] == ',') {
            if (nf == 24u) return 2;    /* a 25th field */
            fb[nf] = b;
            fe[nf] = i;
            ++nf;
            b = i + 1u;
        }
    }
    if (nf != 24u) return 2;
    /* Table 1 numbering is 1-based: No. 1, 5, 8, 21 are fields 0, 4, 7, 20. */
    if (!oracle_parse_time(line + fb[0], fe[0] - fb[0], tz_offset_min, ts)) return 3;
    if (!oracle_parse_ipv4(line + fb[4], fe[4] - fb[4], src)) return 4;
    if (!oracle_parse_ipv4(line + fb[7], fe[7] - fb[7], dst)) return 5;
    if (!oracle_parse_u64(line + fb[20], fe[20] - fb[20], bytes)) return 6;
    return 0;
}

/* The whole text: a line starts at offset 0 and after every '\n' that is not
 * the last byte (so "" has no line and a final '\n' ends the last line).
 * status may be NULL; out[0] = lines, out[1] = valid lines.                 */
void oracle_parse_text(const char* text, uint64_t len, int32_t tz_offset_min,
                       uint64_t* ts, uint32_t* src, uint32_t* dst, uint64_t* bytes,
                       uint8_t* status, uint64_t* out)
{
    uint64_t lines = 0, valid = 0, start = 0;
    while (start < len) {
        uint64_t end = start;
        while (end < len && text[end] != '\n') ++end;
        uint64_t t = 0, b = 0;
        uint32_t s = 0, d = 0;
        int st = oracle_parse_line(text + start, end - start, tz_offset_min, &t, &s, &d, &b);
        if (status) status[lines] = (uint8_t)st;
        if (st == 0) {
            ts[valid] = t;
            src[valid] = s;
            dst[valid] = d;
            bytes[valid] = b;
            ++valid;
        }
        ++lines;
        start = end + 1u;
    }
    out[0] = lines;
    out[1] = valid;
}
