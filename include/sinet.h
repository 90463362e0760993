/*
 * sinet.h -- C ABI of the B200-native SINET session discrimination + millisecond
 * histogram library (libsinet.so), after arXiv 2106.12863.
 *
 * What the library computes (the paper's two procedures):
 *   "Discrimination is dividing session data into ingoing/outgoing with subnet
 *    mask calculation and network address matching.  Histogramming is grouping
 *    ingoing/outgoing session data into bins with map-reduce."
 * For every session record r (Table 1 fields capture_time, source_ip,
 * destination_ip, bytes):
 *   s_in = OR over CIDR entries (Y/Z): bitmask(r.src, Z) - bitmask(Y, Z) == 0
 *   d_in = the same for r.dst                              (Alg. 1 l.4-9)
 *   dir  = dir_lut[s_in*2 + d_in]  (OUT / IN / NEITHER; readings A1, A2)
 *   bin  = (r.ts - window_start) / bin_width, if window_start <= r.ts < window_start + window
 *                                                          (Map; 1 ms bins P:L49)
 *   bins[bin][dir] += (1, r.bytes)   (mod 2^64)            (Reduce)
 * plus side totals (membership matrix, out-of-window), and across GPUs the
 * merge of partial histograms (merge-scatter) as a reduce-scatter
 * over bin ranges.
 *
 * Conventions
 *  - Every function returns SINET_OK (0) or a negative SINET_E_* code; a
 *    detail string is then available from sinet_last_error(ctx).
 *  - Device memory is owned by the CALLER (records, bins, workspace, tags,
 *    staging).  The library never allocates device memory.  It keeps no
 *    pointer to caller host memory after a call returns.
 *  - Every call enqueues work on cfg.stream (a cudaStream_t passed as void*),
 *    in call order.  Calls that return host data synchronise that stream.
 *  - A ctx is not thread-safe; distinct ctxs on distinct devices are independent.
 *  - Addresses are IPv4 as u32 with the first octet most significant (the
 *    numeric value, not network byte order in memory).
 */
#ifndef SINET_H
#define SINET_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SINET_ABI_VERSION 3

/* error codes */
#define SINET_OK        0
#define SINET_E_INVAL  -1   /* invalid argument (see each call) */
#define SINET_E_ALIGN  -2   /* device columns misaligned (see sinet_records) */
#define SINET_E_RANGE  -3   /* bin range outside [0,B) or outside this rank's owned range after reduce */
#define SINET_E_CUDA   -4   /* CUDA runtime error (asynchronous errors surface at the next synchronising call) */
#define SINET_E_NCCL   -5   /* NCCL unavailable or failed */
#define SINET_E_STATE  -6   /* call not allowed in the current state (e.g. classify after reduce without reset) */

/* directions (values of dir_lut and of the `dir` argument) */
#define SINET_DIR_OUT      0
#define SINET_DIR_IN       1
#define SINET_DIR_NEITHER  2

/* metrics (the paper's <timestamp,count> and <timestamp,bytes>) */
#define SINET_METRIC_COUNT 0
#define SINET_METRIC_BYTES 1

/* accumulation strategy */
#define SINET_ORDER_AUTO      0   /* library probes the input's time locality */
#define SINET_ORDER_STREAM    1   /* records approximately time ordered: tile-claim, write-once bins */
#define SINET_ORDER_SHUFFLED  2   /* arbitrary order: prefill bins, then L2 atomics */

typedef struct sinet_ctx sinet_ctx;
typedef struct sinet_hub sinet_hub;   /* in-process rendezvous of the ranks of one merge (see sinet_hub_create) */

/* One batch ("chunk") of session records, columnar.
 * Device pointers for sinet_classify_histogram: naturally aligned, and all four
 * columns starting at the same record offset within a 16-byte group (true for
 * any slice [i, j) of 16-byte aligned columns); host pointers for
 * sinet_classify_histogram_host.  n may be 0.                              */
typedef struct {
    const uint64_t* ts_ms;   /* capture_time, epoch milliseconds (Table 1 no. 1) */
    const uint32_t* src;     /* source_ip (no. 5) */
    const uint32_t* dst;     /* destination_ip (no. 8) */
    const uint64_t* bytes;   /* bytes (no. 21) */
    uint64_t n;
} sinet_records;

typedef struct {
    uint64_t window_start_ms;  /* first millisecond of the window (reading A13: explicit, no tz logic) */
    uint64_t window_ms;        /* W; 86,400,000 for one day; 1 <= W < 2^32 */
    uint32_t bin_width_ms;     /* w >= 1, W % w == 0; B = W / w bins per direction */
    uint8_t  dir_lut[4];       /* [s_in*2+d_in] -> SINET_DIR_*; presets below */
    int32_t  device;           /* CUDA device ordinal the ctx lives on */
    int32_t  rank;             /* this process's rank in [0, world) */
    int32_t  world;            /* number of ranks (GPUs) sharing one histogram, >= 1 */
    void*    stream;           /* cudaStream_t all work is enqueued on (NULL = legacy default) */
    uint32_t order_hint;       /* SINET_ORDER_* */
    uint32_t reserved[7];      /* must be zero */
} sinet_config;

/* direction-LUT presets (A1/A2) */
#define SINET_LUT_SRC_PRIORITY {SINET_DIR_NEITHER, SINET_DIR_IN, SINET_DIR_OUT, SINET_DIR_OUT}
#define SINET_LUT_ALG1         {SINET_DIR_IN, SINET_DIR_IN, SINET_DIR_OUT, SINET_DIR_OUT}
#define SINET_LUT_STRICT       {SINET_DIR_NEITHER, SINET_DIR_IN, SINET_DIR_OUT, SINET_DIR_NEITHER}

/* Side totals, all u64 modulo 2^64. */
typedef struct {
    uint64_t m_count[4];   /* membership matrix over every record, index s_in*2+d_in */
    uint64_t m_bytes[4];
    uint64_t oow_count[2]; /* per dir OUT/IN: records outside the window (counted, not binned, A14) */
    uint64_t oow_bytes[2];
} sinet_totals;

/* ---------------------------------------------------------------- sizing */
/* Device bytes the bins buffer needs: 32 * B_pad, B_pad = B rounded up to a
 * multiple of world * SINET_TILE_BINS.  Layout: u64 bins[B_pad][2 dir][2 metric]
 * (count, bytes) -- one 32-byte DRAM sector per millisecond bin.  0 if cfg invalid. */
size_t sinet_bins_bytes(const sinet_config* cfg);

/* Device bytes of workspace for a table of n_prefixes entries (compiled
 * prefix table, per-tile state flags, totals).  0 if cfg invalid. */
size_t sinet_workspace_bytes(const sinet_config* cfg, uint32_t n_prefixes);

/* Device staging bytes sinet_classify_histogram_host needs to stream host
 * records in chunks of chunk_records (double buffered). */
size_t sinet_staging_bytes(uint64_t chunk_records);

/* ---------------------------------------------------------------- lifecycle */
/* Create a ctx.  Copies and compiles the CIDR list ("CIDR list", Alg. 1 l.1,
 * P:L155; Y.Y.Y.Y/Z, l.4): host bits of prefix_net are cleared (Alg. 1 l.7,
 * reading A9), duplicates dropped, the union compiled to a lookup table in the
 * workspace.  The histogram starts empty (all bins and totals zero).
 * d_bins / d_ws: device buffers of at least sinet_bins_bytes / sinet_workspace_bytes,
 * 256-byte aligned.  Synchronises cfg.stream before returning.
 * Errors: E_INVAL (n_prefixes == 0, a prefix_len > 32, bin_width 0, W % w != 0,
 * W == 0 or W >= 2^32, window_start + W overflows, world < 1, rank outside
 * [0,world), dir_lut entry > 2, reserved != 0, buffer too small or misaligned),
 * E_CUDA.  At most 16383 entries. */
int sinet_open(sinet_ctx** out, const sinet_config* cfg,
               const uint32_t* prefix_net, const uint8_t* prefix_len, uint32_t n_prefixes,
               void* d_bins, size_t bins_bytes, void* d_ws, size_t ws_bytes);

/* NEXT-4, labelled longest-prefix match: as sinet_open, but entry i carries
 * prefix_label[i] (1 = SINET inside, 0 = carved out) and an address is inside iff
 * the longest entry matching it (Alg. 1 l.6-9 per entry) is labelled inside;
 * unmatched addresses are outside; of equal (Y/Z) entries the last one wins.
 * prefix_label == NULL is sinet_open (every entry inside: match-any).  The
 * labelled table is compiled to the same member intervals, so every kernel is
 * unchanged.  At most 16383 entries.  Errors: as sinet_open. */
int sinet_open_labelled(sinet_ctx** out, const sinet_config* cfg,
                        const uint32_t* prefix_net, const uint8_t* prefix_len, const uint8_t* prefix_label,
                        uint32_t n_prefixes, void* d_bins, size_t bins_bytes, void* d_ws, size_t ws_bytes);

/* Destroy a ctx (does not free caller memory).  NULL is a no-op. */
void sinet_close(sinet_ctx* ctx);

/* Start a new, empty histogram (all bins and totals zero) without touching
 * the bins buffer (O(1): bins become "virtually zero" by epoch, DESIGN.md
 * "Tile states").  Clears the reduced state. */
int sinet_reset(sinet_ctx* ctx);

/* ---------------------------------------------------------------- the hot path */
/* Discriminate every record of `recs` (device pointers) and ACCUMULATE its
 * count and bytes into its (bin, dir).  Calling it on k batches
 * equals calling it once on their concatenation (work queue chunks).
 * d_tags (nullable, device, n bytes): per-record tag s_in | d_in<<1 | oow<<2.
 * Errors: E_INVAL (NULL column with n > 0), E_ALIGN (see sinet_records), E_STATE (after reduce
 * without reset), E_CUDA (launch failure). */
int sinet_classify_histogram(sinet_ctx* ctx, const sinet_records* recs, uint8_t* d_tags);

/* The same, with HOST record columns: the library streams them through the
 * caller's device staging buffer (sinet_staging_bytes(chunk_records) bytes)
 * in chunks, overlapping host->device copies with the kernel.  Pinned host
 * memory makes the copies asynchronous.  Synchronises cfg.stream. */
int sinet_classify_histogram_host(sinet_ctx* ctx, const sinet_records* host_recs,
                                  void* d_staging, size_t staging_bytes, uint64_t chunk_records);

/* NEXT-4 comparator -- the paper's own histogram design on this GPU:
 * discriminate, emit <key = bin*2+dir, bytes> pairs, sort by key and
 * reduce_by_key ("pairwise reduction"), then add each run into
 * its bin.  Same semantics and result as sinet_classify_histogram (no tags);
 * needs caller scratch of sinet_sortreduce_scratch_bytes(cfg, n) device bytes
 * (~40 B/record).  n < 2^31 and 2B < 2^32.  Errors: as classify, E_INVAL. */
size_t sinet_sortreduce_scratch_bytes(const sinet_config* cfg, uint64_t n);
int sinet_classify_histogram_sortreduce(sinet_ctx* ctx, const sinet_records* recs,
                                        void* d_scratch, size_t scratch_bytes);

/* Unordered input, partition then bin (SURVEY §8(d) strategy S4; the paper's tiling of a
 * problem that "does not fit in the cache", §4): with a caller scratch buffer
 * registered here, batches the order probe finds unordered (or cfg.order_hint SHUFFLED) are
 * radix-partitioned by time into buckets of 8192 ms bins and every bucket is reduced in
 * shared memory and written once, in sub-batches of as many records as the scratch holds
 * (24 B/record + ~0.3 MB).  Without scratch such batches take the L2-atomic kernel.  Same
 * result either way.  Windows of at most 2^27 bins.  sinet_partition_scratch_bytes(cfg, m)
 * = bytes for sub-batches of m >= 2^16 records (0 if unsupported).  set_scratch: 256-byte
 * aligned device buffer the library may use until it is replaced or removed (NULL / 0
 * removes it); it must not be used by anything else meanwhile.  Errors: E_INVAL, E_ALIGN. */
size_t sinet_partition_scratch_bytes(const sinet_config* cfg, uint64_t max_records);
int sinet_set_scratch(sinet_ctx* ctx, void* d_scratch, size_t bytes);

/* NEXT-2, watchlist filter (Figs 8-11: 300 AbuseIPDB addresses P:L345-350, 877
 * GRIZZLY STEPPE addresses P:L366-370): from now on only records whose source OR
 * destination equals a listed address are counted (totals and bins; tags still
 * describe every record) -- filter, then the unchanged histogram.  The list (set
 * semantics: duplicates collapse) is copied into the caller's device buffer of
 * sinet_watchlist_bytes(n) bytes (16-byte aligned), which must stay valid while
 * the filter is active.  n == 0 removes the filter.  Synchronises the stream.
 * Errors: E_INVAL, E_CUDA. */
size_t sinet_watchlist_bytes(uint32_t n);
int sinet_set_watchlist(sinet_ctx* ctx, const uint32_t* ips, uint32_t n, void* d_buf, size_t buf_bytes);

/* Materialise every bin (zero-fill tiles no record touched).  Idempotent;
 * called implicitly by sinet_reduce and sinet_read_bins. */
int sinet_finalize(sinet_ctx* ctx);

/* ---------------------------------------------------------------- multi-GPU */
/* Build this rank's NCCL communicator from a 128-byte ncclUniqueId created by
 * rank 0 and shared by the caller (e.g. through torch.distributed).  NCCL is
 * loaded at run time (the libnccl.so.2 already in the process, else by name).
 * Optional with world == 1 (sinet_reduce then runs the same NCCL calls on a
 * one-rank communicator).  Errors: E_NCCL, E_INVAL, E_STATE (already initialised). */
int sinet_comm_init(sinet_ctx* ctx, const void* nccl_unique_id);

/* Create a fresh 128-byte ncclUniqueId (rank 0), to be shared with the other
 * ranks before sinet_comm_init.  Errors: E_NCCL, E_INVAL (NULL out). */
int sinet_nccl_unique_id(void* out128);

/* In-process merge, the paper's own layout ("we assign one thread for each GPU"):
 * `world` ctxs in ONE process -- on distinct GPUs, or several on one GPU -- join a hub
 * instead of NCCL; each rank then calls sinet_reduce from its own host thread (the calls
 * rendezvous on a host barrier; device order is kept with CUDA events).  Data moves by
 * peer copies over UVA, and the dense reduce-scatter is one kernel per owner reading its
 * slice from every rank's bins directly (NVLink P2P loads between GPUs; peer access is
 * enabled on first use).  Results are identical to the NCCL path.  The hub is reference
 * counted: sinet_hub_destroy drops the creator's reference and the memory is freed when the
 * last attached ctx closes (in any order); a ctx attaches once (sinet_close detaches it).
 * Errors: E_INVAL (world < 1 or > 64, NULL out / hub, hub world != cfg.world, rank already
 * attached), E_STATE (ctx already has a communicator). */
int sinet_hub_create(sinet_hub** out, int32_t world);
void sinet_hub_destroy(sinet_hub* hub);
int sinet_comm_init_hub(sinet_ctx* ctx, sinet_hub* hub);

/* Merge the per-GPU partial histograms (merge-scatter): finalize,
 * then an in-place reduce-scatter (u64 sum) leaves rank g the global sums of
 * bins [g*B_pad/world, (g+1)*B_pad/world); totals are all-reduced so every
 * rank holds the global totals.  world == 1 without a communicator: finalize only.
 * With contiguous time shards each rank's partial histogram is zero outside the
 * bins it touched, so by default (exchange mode 0) the ranks all-gather their
 * touched ranges and, when that moves at most half the data of the dense
 * reduce-scatter, only the overlaps travel (grouped ncclSend/ncclRecv into the
 * workspace's staging, then added to the owned bins) -- same result.
 * Synchronises the stream in that case (the plan is made on the host).
 * Errors: E_STATE (already reduced), E_NCCL (no comm / NCCL failure). */
int sinet_reduce(sinet_ctx* ctx);

/* Merge strategy for sinet_reduce: 0 automatic, 1 dense reduce-scatter,
 * 2 sparse touched-range exchange (falls back to dense if staging is too small).
 * sinet_last_exchange reports what the last reduce did (1 dense, 2 sparse, 0 none). */
int sinet_set_exchange(sinet_ctx* ctx, int mode);
int sinet_last_exchange(const sinet_ctx* ctx);
/* Smallest / largest bin written since the last reset (min > max: none); synchronises. */
int sinet_touched_range(sinet_ctx* ctx, uint32_t* min_bin, uint32_t* max_bin);
/* Host-side plan of the sparse exchange (no GPU): touched[2*r], touched[2*r+1] =
 * min / max bin rank r wrote (min > max: none).  Fills send[2*o] = first bin,
 * send[2*o+1] = count this rank sends to owner o, and recv[2*r], recv[2*r+1] what
 * it receives from rank r.  Errors: E_INVAL. */
int sinet_exchange_plan(int32_t world, int32_t rank, uint64_t nbins, uint64_t nbins_pad, const uint32_t* touched,
                        uint64_t* send, uint64_t* recv);

/* Owned bin range: [0, B) before reduce or with world == 1, else this rank's
 * slice clipped to [0, B). */
int sinet_owned_range(sinet_ctx* ctx, uint64_t* first_bin, uint64_t* n_bins);

/* ---------------------------------------------------------------- read-out */
/* Copy bins [first_bin, first_bin + n_bins) of one (dir, metric) plane into
 * dst (u64[n_bins]; device if dst_is_device else host, host copies
 * synchronise the stream).  Errors: E_INVAL (dir not OUT/IN, metric not
 * COUNT/BYTES, NULL dst), E_RANGE (outside the owned range), E_CUDA. */
int sinet_read_bins(sinet_ctx* ctx, int dir, int metric, uint64_t first_bin, uint64_t n_bins,
                    uint64_t* dst, int dst_is_device);

/* Copy bins [first_bin, first_bin + n_bins) in the native layout, u64
 * dst[n_bins][2 dir][2 metric] (32 bytes per bin: the paper's <timestamp,count>
 * and <timestamp,bytes> of both directions), with ONE contiguous copy into
 * dst (device if dst_is_device else host; page-locked host memory makes it an
 * async DMA at full link rate; host copies synchronise the stream).  Errors:
 * E_INVAL (NULL dst), E_RANGE (outside the owned range), E_CUDA. */
int sinet_read_bins_raw(sinet_ctx* ctx, uint64_t first_bin, uint64_t n_bins, uint64_t* dst, int dst_is_device);

/* NEXT-1, coarser frames: "Session data is grouped into one-hour frame bins"
 * (P:L323); "about 40,000 in 10 minutes".  Frame F = bins
 * [F*factor, (F+1)*factor) of the window (frames aligned to window_start).  The
 * owned range [lo, lo+n) meets frames first_frame = floor(lo/factor) ..
 * ceil((lo+n)/factor) - 1 (sinet_rebin_frames); sinet_rebin writes, for each, the sum
 * of its OWNED bins into d_out u64[n_frames][2 dir][2 metric] (device, 8-byte
 * aligned), d_out[k] = frame first_frame + k.  A frame that straddles two ranks'
 * owned ranges is the sum of their two entries for it.  n_out must equal
 * n_frames.  u64 sums wrap mod 2^64.  Errors: E_INVAL, E_CUDA. */
int sinet_rebin_frames(sinet_ctx* ctx, uint64_t factor, uint64_t* first_frame, uint64_t* n_frames);
int sinet_rebin(sinet_ctx* ctx, uint64_t factor, uint64_t* d_out, uint64_t n_out);

/* NEXT-1, sparse series: the key/value namespaces X1<timestamp>, X1<count>,
 * X2<timestamp>, X2<bytes>.  Writes, in ascending bin order,
 * (bin start in epoch ms, count, bytes) of every bin of direction `dir` in the
 * owned range whose count is nonzero, at most `capacity` entries, into device
 * arrays u64[capacity]; *n_nonzero (host) receives the total number of such
 * bins (may exceed capacity).  Synchronises the stream.  Errors: E_INVAL, E_CUDA. */
int sinet_export_sparse(sinet_ctx* ctx, int dir, uint64_t* d_ts_ms, uint64_t* d_count, uint64_t* d_bytes,
                        uint64_t capacity, uint64_t* n_nonzero);

/* Copy the totals to host (synchronises the stream). */
int sinet_read_totals(sinet_ctx* ctx, sinet_totals* out);

/* ---------------------------------------------------------------- NEXT-3: session-log text
 * The step before the path: PA-7080 session-log text (Table 1) into
 * the four device columns sinet_classify_histogram reads.  The paper prints the
 * 24 items and sample values but no file syntax; readings A27-A31 fix it:
 *   - one record per line, lines separated by '\n' (a '\r' before it is allowed);
 *     a line starts at offset 0 and after every '\n' that is not the last byte;
 *   - 24 comma-separated fields in Table 1 order; the parser reads No. 1
 *     capture_time "YYYY/MM/DD HH:MM:SS.mmm" (local time at tz_offset_min minutes
 *     east of UTC, Gregorian calendar, no leap seconds; result epoch ms UTC >= 0),
 *     No. 5 source_ip and No. 8 destination_ip (dotted quad: four 1-3 digit octets
 *     <= 255, no leading zeros), No. 21 bytes (1-20 decimal digits, < 2^64);
 *     every other field is opaque;
 *   - line status, the first failing check in this order: LONG (content, '\r'
 *     included, longer than SINET_PARSE_MAX_LINE bytes), COLUMNS (not 24 fields),
 *     TIME, SRC, DST, BYTES; else OK.
 * Valid lines are written, in line order, to out (skip policy); the per-line
 * status array and the counts let the caller apply any other policy. */
#define SINET_PARSE_MAX_LINE 2047
#define SINET_LINE_OK       0
#define SINET_LINE_LONG     1
#define SINET_LINE_COLUMNS  2
#define SINET_LINE_TIME     3
#define SINET_LINE_SRC      4
#define SINET_LINE_DST      5
#define SINET_LINE_BYTES    6

/* Output columns of the parser (device pointers, naturally aligned; capacity records). */
typedef struct {
    uint64_t* ts_ms;
    uint32_t* src;
    uint32_t* dst;
    uint64_t* bytes;
    uint64_t capacity;
} sinet_columns;

typedef struct {
    uint64_t lines;            /* lines in the text */
    uint64_t valid;            /* lines with status OK (records produced; see E_RANGE) */
    uint64_t first_bad_line;   /* 0-based index of the first non-OK line, UINT64_MAX if none */
    uint64_t by_status[7];     /* lines per SINET_LINE_* code */
} sinet_parse_result;

/* Device workspace of sinet_parse_text for text_bytes of text (256-byte aligned). */
size_t sinet_parse_workspace_bytes(uint64_t text_bytes);
/* Parse d_text[0, text_bytes) (device, 16-byte aligned; not modified) into out;
 * if d_status != NULL, d_status[i] = status of line i for i < status_capacity.
 * Enqueued on `stream` (a cudaStream_t, NULL = legacy default); synchronises it
 * to fill *result (host).  tz_offset_min in [-1440, 1440] (JST logs: 540).
 * Errors: E_INVAL (NULL result, bad tz, workspace too small, NULL columns with
 * capacity > 0); E_ALIGN (text or columns misaligned); E_RANGE (more valid lines
 * than out.capacity: the first capacity records are written, result is complete);
 * E_CUDA.  Detail string: sinet_parse_last_error() (per thread). */
int sinet_parse_text(const uint8_t* d_text, uint64_t text_bytes, int32_t tz_offset_min,
                     const sinet_columns* out, uint8_t* d_status, uint64_t status_capacity,
                     void* d_ws, size_t ws_bytes, void* stream, sinet_parse_result* result);
const char* sinet_parse_last_error(void);

/* ---------------------------------------------------------------- introspection */
const char* sinet_last_error(const sinet_ctx* ctx);
/* Number of kernels this ctx has launched since open (all kinds). */
uint64_t sinet_launch_count(const sinet_ctx* ctx);
/* Enable (1) / disable (0) CUDA-event timing of the main classify kernel on
 * cfg.stream; sinet_kernel_time reads back the summed duration (ms) and the
 * number of timed launches since enabling (synchronises the stream). */
int sinet_set_kernel_timing(sinet_ctx* ctx, int on);
int sinet_kernel_time(sinet_ctx* ctx, double* total_ms, uint64_t* launches);
/* Which accumulation strategy the last classify call used (SINET_ORDER_STREAM/SHUFFLED, 3 = sort-reduce). */
int sinet_last_strategy(const sinet_ctx* ctx);
/* Host-side check of the prefix compiler (no GPU needed): compiles the CIDR
 * list exactly as sinet_open does and evaluates the lookups the kernels use
 * (packed /16 classes + /24 level 2 + boundary search; the same without level
 * 2; the byte /16 + /24 tables of the stream kernel) on the host, for
 * ips[0..n): out[i] = member (0/1).
 * Errors: E_INVAL as sinet_open's table checks, or if the encodings disagree. */
int sinet_table_member_host(const uint32_t* prefix_net, const uint8_t* prefix_len, uint32_t n_prefixes,
                            const uint32_t* ips, uint64_t n, uint8_t* out);
/* The same for a labelled table (sinet_open_labelled semantics). */
int sinet_table_member_host_labelled(const uint32_t* prefix_net, const uint8_t* prefix_len,
                                     const uint8_t* prefix_label, uint32_t n_prefixes,
                                     const uint32_t* ips, uint64_t n, uint8_t* out);
/* Performance knobs of the STREAM kernel (results are identical for every setting):
 * stream_groups 0 = automatic, 1 = one 8192-bin ring per CTA, 2 = two independent
 * 4096-bin rings per CTA; warp_aggregation 1/0 = on/off, -1 = unchanged.  Errors: E_INVAL. */
int sinet_set_tuning(sinet_ctx* ctx, int stream_groups, int warp_aggregation);
/* Named performance knobs (results are identical for every setting; they exist for A/B
 * measurements and tests): "stream_groups" 0..2, "warp_aggregation" 0/1,
 * "ranges_per_group" 0..64 (0 = default: ranges of ~300 k records), "table_mode" -1..3
 * (as sinet_set_table_mode), "exchange" 0..2 (as sinet_set_exchange), "stream_kernel" 0..2
 * (0 automatic, 1 the group-barrier kernel k_hist_stream, 2 the warp-specialised k_hist_ws),
 * "shuffled_kernel" 0..1 (0 partition-then-bin when scratch is registered, 1 L2 atomics).
 * Errors: E_INVAL (unknown name or value out of range). */
int sinet_set_knob(sinet_ctx* ctx, const char* name, int64_t value);
/* Name of the dominant kernel the last classify call launched ("k_hist_ws",
 * "k_hist_stream", "k_hist_atomic"; "" before the first call or for a NULL ctx). */
const char* sinet_last_kernel(const sinet_ctx* ctx);
/* Lookup-table encoding of the STREAM kernel (Alg. 1 l.6-9 compiled by sinet_open;
 * results are identical for every setting): -1 = automatic (the fastest that fits
 * in shared memory), 0 = byte /16 + /24 classes, 1 = packed 2-bit classes with
 * level 2, 2 = packed without level 2, 3 = packed with level 2 and boundaries
 * read from global memory.  A forced encoding that does not exist or fit falls
 * back to the automatic choice.  Errors: E_INVAL (mode < -1 or > 3). */
int sinet_set_table_mode(sinet_ctx* ctx, int mode);
/* The encoding the next STREAM launch will use (0..3), or E_INVAL for a NULL ctx. */
int sinet_table_mode(const sinet_ctx* ctx);
/* Compile-time constants of this build. */
uint32_t sinet_tile_bins(void);
uint32_t sinet_parse_chunk_bytes(void);   /* text bytes one CTA of sinet_parse_text owns per ticket */
/* Process-wide performance/test knob of sinet_parse_text (results identical for every value):
 * "unpacked_look_back" 1 forces the two-word look-back used for >= 2 GiB of text.  E_INVAL
 * for an unknown name or value. */
int sinet_parse_set_knob(const char* name, int64_t value);
int sinet_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SINET_H */
