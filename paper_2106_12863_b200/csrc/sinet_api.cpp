// libsinet C ABI (include/sinet.h): context lifecycle, validation, launch
// planning, NCCL merge and read-out.  All device memory is the caller's.
#include "sinet.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "prefix_compile.h"
#include "sinet_comm.h"
#include "sinet_kernels.h"
#include "sinet_parse.h"

using namespace sinet;

namespace {

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

struct Geometry {
    uint64_t B = 0, B_pad = 0, n_tiles = 0;
};

bool check_cfg(const sinet_config* c, std::string* err, Geometry* g) {
    if (!c) { *err = "NULL config"; return false; }
    if (c->window_ms == 0 || c->window_ms >= (1ull << 32)) { *err = "window_ms must be in [1, 2^32)"; return false; }
    if (c->bin_width_ms == 0) { *err = "bin_width_ms must be >= 1"; return false; }
    if (c->window_ms % c->bin_width_ms != 0) { *err = "window_ms must be a multiple of bin_width_ms"; return false; }
    if (c->window_start_ms > ~0ull - c->window_ms) { *err = "window_start_ms + window_ms overflows u64"; return false; }
    if (c->world < 1 || c->world > 4096) { *err = "world must be in [1, 4096]"; return false; }
    if (c->rank < 0 || c->rank >= c->world) { *err = "rank must be in [0, world)"; return false; }
    for (int k = 0; k < 4; ++k)
        if (c->dir_lut[k] > SINET_DIR_NEITHER) { *err = "dir_lut entries must be 0 (OUT), 1 (IN) or 2 (NEITHER)"; return false; }
    if (c->order_hint > SINET_ORDER_SHUFFLED) { *err = "order_hint must be SINET_ORDER_*"; return false; }
    for (int k = 0; k < 7; ++k)
        if (c->reserved[k]) { *err = "reserved fields must be zero"; return false; }
    g->B = c->window_ms / c->bin_width_ms;
    uint64_t unit = (uint64_t)c->world * kTileBins;
    g->B_pad = (g->B + unit - 1) / unit * unit;
    g->n_tiles = g->B_pad / kTileBins;
    return true;
}

struct WsLayout {
    size_t totals, cls2, bnd, rank, mentry, l2, b16, b24, flags, sparse, counters, probe, xranges, xtotals, staging,
        staging_bytes, total;
};

// Device staging for the sparse multi-GPU exchange: a quarter of the owned slice, capped.
size_t exchange_staging_bytes(uint64_t n_tiles, int world) {
    if (world <= 1) return 0;
    const uint64_t per = n_tiles * kTileBins / (uint64_t)world;
    uint64_t b = per * 32u / 4u;
    const uint64_t cap = 256ull << 20;
    return (size_t)(b < cap ? b : cap);
}

WsLayout ws_layout(uint64_t n_tiles, uint32_t n_prefixes, int world) {
    WsLayout L{};
    size_t off = 0;
    L.totals = off; off = align_up(off + 16 * 8, 256);
    L.cls2 = off;   off = align_up(off + (size_t)kClsWords * 4, 256);
    L.bnd = off;    off = align_up(off + ((size_t)4 * n_prefixes + 2) * 4, 256);
    L.rank = off;   off = align_up(off + (size_t)kRankWords * 4, 256);
    L.mentry = off; off = align_up(off + (size_t)(4u * n_prefixes + 2u) * 4, 256);
    L.l2 = off;     off = align_up(off + (size_t)(4u * n_prefixes + 2u) * 64, 256);
    L.b16 = off;    off = align_up(off + 65536, 256);
    L.b24 = off;    off = align_up(off + (size_t)kMaxByteMixed * 256 + 16, 256);   // + the 16 B the staging over-reads
    L.flags = off;  off = align_up(off + (size_t)n_tiles * 4, 256);
    L.sparse = off; off = align_up(off + 16 + (size_t)sparse_blocks(n_tiles * kTileBins) * 4, 256);
    L.counters = off; off = align_up(off + 64, 256);   // [0] range counter, [4..5] touched min/max
    L.probe = off;  off = align_up(off + (size_t)kProbeRuns * kProbeRun * 8, 256);   // AUTO order probe
    L.xranges = off; off = align_up(off + (size_t)world * 8, 256);
    L.xtotals = off; off = align_up(off + (size_t)(world > 1 ? world : 0) * 12 * 8, 256);   // in-process all-reduce
    L.staging_bytes = exchange_staging_bytes(n_tiles, world);
    L.staging = off; off = align_up(off + L.staging_bytes, 256);
    L.total = off;
    return L;
}

}  // namespace

struct sinet_ctx {
    sinet_config cfg{};
    Geometry geo;
    WsLayout ws{};
    cudaStream_t stream = nullptr;
    int device = 0;
    int sm_count = 0;
    int atomic_grid = 0;
    int materialize_grid = 0;
    unsigned long long* bins = nullptr;
    unsigned char* d_ws = nullptr;
    uint32_t nbnd = 0;
    uint32_t lut = 0;
    uint32_t magic = 0;
    uint32_t epoch = 1;
    bool reduced = false;
    bool materialized = false;
    int last_strategy = 0;
    const char* last_kernel = "";   // dominant kernel of the last classify call
    int auto_choice = 0;          // strategy AUTO resolved by the first probe
    const uint64_t* probe_ts = nullptr;   // the last probed batch (column address, size) and its verdict
    uint64_t probe_n = 0;
    int probe_choice = 0;
    bool agg = false;             // warp aggregation of equal keys in the stream kernel (measured slower on C4)
    uint32_t stream_groups = 0;   // 0 auto, 1 or 2
    uint32_t stream_kernel = 0;   // 0 auto, 1 k_hist_stream (group barriers), 2 k_hist_ws (warp-specialised)
    uint32_t debug = 0;           // knob "debug_counters"
    uint32_t shuffled_kernel = 0; // 0 auto (partition-then-bin when scratch is set), 1 L2 atomics only
    void* scratch = nullptr;      // caller scratch for the partitioned path (sinet_set_scratch)
    size_t scratch_bytes = 0;
    uint64_t scratch_cap = 0;     // records per partitioned sub-batch
    uint32_t ranges_per_group = 0;
    int tab_mode = -1;            // stream kernel lookup-table encoding: -1 automatic, 0..3 forced
    int exchange = 0;             // multi-GPU merge: 0 auto (sparse when cheaper), 1 dense, 2 sparse
    int last_exchange = 0;        // 1 dense reduce-scatter, 2 sparse touched-range exchange
    // NEXT-2 watchlist (caller-owned device buffer)
    const uint32_t* wbits = nullptr;
    const uint32_t* wlist = nullptr;
    uint32_t wn = 0;
    uint64_t launches = 0;
    std::unique_ptr<Transport> comm;   // cross-GPU merge: NCCL or the in-process hub (sinet_comm.h)
    // host-streaming pipeline
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t copy_done[2] = {nullptr, nullptr};
    cudaEvent_t kern_done[2] = {nullptr, nullptr};
    // optional kernel timing
    bool timing = false;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> tev;
    std::string err;
    CompiledTable table;
};

namespace {

struct DeviceGuard {
    int prev = -1;
    bool ok = true;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != dev) ok = cudaSetDevice(dev) == cudaSuccess;
    }
    ~DeviceGuard() {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

int fail(sinet_ctx* c, int code, const std::string& msg) {
    if (c) c->err = msg;
    return code;
}

int cuda_fail(sinet_ctx* c, cudaError_t e, const char* where) {
    return fail(c, SINET_E_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define SINET_CUDA(ctx, expr)                                    \
    do {                                                         \
        cudaError_t e_ = (expr);                                 \
        if (e_ != cudaSuccess) return cuda_fail(ctx, e_, #expr); \
    } while (0)

uint32_t* ws_u32(sinet_ctx* c, size_t off) { return reinterpret_cast<uint32_t*>(c->d_ws + off); }

KernelParams base_params(sinet_ctx* c) {
    KernelParams p{};
    p.bins = c->bins;
    p.totals = reinterpret_cast<unsigned long long*>(c->d_ws + c->ws.totals);
    p.tile_flags = ws_u32(c, c->ws.flags);
    p.cls2 = ws_u32(c, c->ws.cls2);
    p.bnd = ws_u32(c, c->ws.bnd);
    p.rank = ws_u32(c, c->ws.rank);
    p.mentry = ws_u32(c, c->ws.mentry);
    p.l2 = ws_u32(c, c->ws.l2);
    p.b16 = c->d_ws + c->ws.b16;
    p.b24 = c->d_ws + c->ws.b24;
    p.has_bytes = c->table.b16.empty() ? 0u : 1u;
    p.tab_mode = c->tab_mode;
    p.n_mixed = c->table.n_mixed;
    p.nbnd = c->nbnd;
    p.small = table_small(c->nbnd, c->table.n_mixed) ? 1u : 0u;
    p.stream_groups = c->stream_groups;
    p.stream_kernel = c->stream_kernel;
    p.debug = c->debug;
    p.ranges_per_group = c->ranges_per_group;
    p.range_counter = ws_u32(c, c->ws.counters);
    p.touched = ws_u32(c, c->ws.counters) + 4;
    p.wbits = c->wbits;
    p.wlist = c->wlist;
    p.wn = c->wn;
    p.lut = c->lut;
    p.start = c->cfg.window_start_ms;
    p.window = (uint32_t)c->cfg.window_ms;
    p.width = c->cfg.bin_width_ms;
    p.magic = c->magic;
    p.nbins = (uint32_t)c->geo.B;
    p.epoch = c->epoch;
    p.n_tiles = (uint32_t)c->geo.n_tiles;
    return p;
}

uint32_t init_word(const sinet_ctx* c) { return (c->epoch << 2) | kTileInit; }

int do_materialize(sinet_ctx* c) {
    if (c->materialized) return SINET_OK;
    SINET_CUDA(c, launch_materialize(c->bins, ws_u32(c, c->ws.flags), (uint32_t)c->geo.n_tiles,
                                     init_word(c), c->materialize_grid, c->stream));
    c->launches++;
    c->materialized = true;
    return SINET_OK;
}

// Strategy AUTO: look at 64 evenly spaced runs of 32 consecutive capture times.
// Time-ordered logs (day files processed chunk by chunk) have runs that
// span about the capture disorder; shuffled input spans the whole window.
int probe_order(sinet_ctx* c, const sinet_records* r, int* out) {
    constexpr int kRuns = (int)kProbeRuns, kRun = (int)kProbeRun;
    // too small to judge: the stream kernel (exact for any order), decision not kept
    if (r->n < (uint64_t)kRuns * kRun) { *out = SINET_ORDER_STREAM; return SINET_OK; }
    // the same batch again (same columns, same size: e.g. a day re-run after sinet_reset) keeps
    // its verdict -- the choice affects speed only, both kernels are exact for any order
    if (c->probe_ts == r->ts_ms && c->probe_n == r->n && c->probe_choice) { *out = c->probe_choice; return SINET_OK; }
    // one gather kernel into workspace, one 16 KB copy to host
    uint64_t* d_runs = reinterpret_cast<uint64_t*>(c->d_ws + c->ws.probe);
    std::vector<uint64_t> h((size_t)kRuns * kRun);
    SINET_CUDA(c, launch_probe_gather(r->ts_ms, r->n, d_runs, c->stream));
    SINET_CUDA(c, cudaMemcpyAsync(h.data(), d_runs, h.size() * 8, cudaMemcpyDeviceToHost, c->stream));
    SINET_CUDA(c, cudaStreamSynchronize(c->stream));
    std::vector<uint64_t> span(kRuns);
    for (int k = 0; k < kRuns; ++k) {
        uint64_t lo = ~0ull, hi = 0;
        for (int i = 0; i < kRun; ++i) { uint64_t v = h[(size_t)k * kRun + i]; lo = v < lo ? v : lo; hi = v > hi ? v : hi; }
        span[k] = hi - lo;
    }
    std::nth_element(span.begin(), span.begin() + kRuns / 2, span.end());
    const uint64_t limit = (uint64_t)kStreamWindowBins * c->cfg.bin_width_ms;
    *out = (span[kRuns / 2] <= limit || c->geo.B <= kStreamWindowBins) ? SINET_ORDER_STREAM : SINET_ORDER_SHUFFLED;
    c->probe_ts = r->ts_ms;
    c->probe_n = r->n;
    c->probe_choice = *out;
    return SINET_OK;
}

int prepare_params(sinet_ctx* c, const sinet_records* r, uint8_t* d_tags, KernelParams* out) {
    if (c->reduced) return fail(c, SINET_E_STATE, "classify after reduce: call sinet_reset first");
    if (!r) return fail(c, SINET_E_INVAL, "NULL records");
    if (r->n > (1ull << 38)) return fail(c, SINET_E_INVAL, "batch larger than 2^38 records: split it");
    if (r->n && (!r->ts_ms || !r->src || !r->dst || !r->bytes)) return fail(c, SINET_E_INVAL, "NULL record column");
    // Columns may start mid-way into a 16-byte group (e.g. a batch sliced at any
    // record index) as long as all four are offset by the same number of records.
    const uintptr_t a_ts = reinterpret_cast<uintptr_t>(r->ts_ms), a_src = reinterpret_cast<uintptr_t>(r->src),
                    a_dst = reinterpret_cast<uintptr_t>(r->dst), a_by = reinterpret_cast<uintptr_t>(r->bytes);
    const uint32_t head = (uint32_t)((a_src & 15u) >> 2);
    if (r->n && ((a_ts & 7u) || (a_by & 7u) || (a_src & 3u) || (a_dst & 3u) || ((a_dst & 15u) >> 2) != head ||
                 ((a_ts - 8u * head) & 15u) || ((a_by - 8u * head) & 15u)))
        return fail(c, SINET_E_ALIGN, "record columns must be naturally aligned and start at the same "
                                      "record offset within a 16-byte group (16-byte aligned bases)");
    KernelParams p = base_params(c);
    p.ts = r->ts_ms; p.src = r->src; p.dst = r->dst; p.bytes = r->bytes; p.n = r->n; p.tags = d_tags;
    p.head = head;
    p.nv = r->n + head;
    p.tags_vec = d_tags && (((reinterpret_cast<uintptr_t>(d_tags) - head) & 3u) == 0) ? 1u : 0u;
    *out = p;
    return SINET_OK;
}

constexpr uint64_t kPartMinCap = 1u << 16;   // records: smaller scratch is not worth the passes
constexpr bool kWsAuto = false;   // k_hist_ws opt-in (knob stream_kernel=2) until measured on the GPU

int classify_device(sinet_ctx* c, const sinet_records* r, uint8_t* d_tags) {
    KernelParams p;
    int prc = prepare_params(c, r, d_tags, &p);
    if (prc) return prc;
    if (r->n == 0) return SINET_OK;
    int strategy = (int)c->cfg.order_hint;
    if (strategy == SINET_ORDER_AUTO) {
        // probed once per histogram (sinet_reset forgets it) on the first batch large enough
        // to judge; smaller batches take the stream kernel without deciding
        if (!c->auto_choice) {
            int choice = SINET_ORDER_STREAM;
            int rc = probe_order(c, r, &choice);
            if (rc) return rc;
            if (r->n >= 2048) c->auto_choice = choice;
            strategy = choice;
        } else {
            strategy = c->auto_choice;
        }
    }
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    const bool partitioned = strategy == SINET_ORDER_SHUFFLED && c->scratch_cap >= kPartMinCap &&
                             c->shuffled_kernel == 0u && partition_supported((uint32_t)c->geo.B);
    if (strategy == SINET_ORDER_SHUFFLED && !partitioned) {
        // materialise every tile, then L2 atomics (any order)
        int rc = do_materialize(c);
        if (rc) return rc;
    }
    if (c->timing) {
        SINET_CUDA(c, cudaEventCreate(&e0));
        SINET_CUDA(c, cudaEventCreate(&e1));
        SINET_CUDA(c, cudaEventRecord(e0, c->stream));
    }
    uint64_t n_launched = 1;
    if (partitioned) {
        n_launched = 0;
        // sub-batches of scratch_cap records (a multiple of 4: every sub-batch keeps the batch's
        // 16-byte phase); tiles are claimed per sub-batch, so later ones add onto earlier ones
        const PartLayout L = part_layout(c->scratch_cap, (uint32_t)c->geo.B);
        for (uint64_t o = 0; o < r->n; o += c->scratch_cap) {
            const uint64_t m = (r->n - o < c->scratch_cap) ? r->n - o : c->scratch_cap;
            sinet_records sub{r->ts_ms + o, r->src + o, r->dst + o, r->bytes + o, m};
            KernelParams q;
            int prc2 = prepare_params(c, &sub, d_tags ? d_tags + o : nullptr, &q);
            if (prc2) return prc2;
            int k = 0;
            SINET_CUDA(c, launch_partitioned(q, c->scratch, L, c->sm_count, c->stream, &k));
            n_launched += (uint64_t)k;
        }
        c->materialized = false;
        c->last_kernel = "k_part (count, scatter, fine, bin)";
    } else if (strategy == SINET_ORDER_SHUFFLED) {
        SINET_CUDA(c, launch_hist_atomic(p, c->atomic_grid, c->stream));
        c->last_kernel = "k_hist_atomic";
    } else {
        // time-window privatisation, write-once bins; untouched tiles stay virtual
        // k_hist_ws for dense input (>= 1 record per bin: its 15 workers' in-flight chunks stay
        // inside the ring), k_hist_stream (8192-bin ring per 512 threads) for sparse input
        const int tab = stream_table_mode(p.has_bytes != 0u, p.nbnd, p.n_mixed, p.tab_mode);
        const bool ws = p.stream_kernel == 2u ||
                        (kWsAuto && p.stream_kernel == 0u && p.n >= (uint64_t)p.nbins && hist_ws_fits(tab, p.nbnd, p.n_mixed));
        if (ws && hist_ws_fits(tab, p.nbnd, p.n_mixed)) {
            SINET_CUDA(c, launch_hist_ws(p, c->sm_count, c->stream));
            c->last_kernel = "k_hist_ws";
        } else {
            SINET_CUDA(c, launch_hist_stream(p, c->sm_count, c->agg, c->stream));
            c->last_kernel = "k_hist_stream";
        }
        c->materialized = false;
    }
    c->launches += n_launched;
    c->last_strategy = strategy;
    if (c->timing) {
        SINET_CUDA(c, cudaEventRecord(e1, c->stream));
        c->tev.emplace_back(e0, e1);
    }
    return SINET_OK;
}

}  // namespace

// Sparse exchange plan: rank r's partial histogram is zero outside its touched range
// T_r = [min_r, max_r]; owner o needs T_r ∩ Own(o) from every r != o.
struct Seg { uint64_t first, n; };
void plan_exchange(int world, int rank, uint64_t B, uint64_t B_pad, const uint32_t* tr,
                   std::vector<Seg>* send, std::vector<Seg>* recv) {
    const uint64_t per = B_pad / (uint64_t)world;
    auto own = [&](int o, uint64_t* lo, uint64_t* hi) {
        *lo = per * (uint64_t)o; *hi = *lo + per;
        if (*lo > B) *lo = B;
        if (*hi > B) *hi = B;
    };
    auto inter = [&](int r, int o) -> Seg {
        const uint64_t tmin = tr[2 * r], tmax = tr[2 * r + 1];
        if (r == o || tmin > tmax) return Seg{0, 0};
        uint64_t lo, hi;
        own(o, &lo, &hi);
        const uint64_t a = tmin > lo ? tmin : lo, b = (tmax + 1 < hi) ? tmax + 1 : hi;
        return (a < b) ? Seg{a, b - a} : Seg{0, 0};
    };
    send->assign(world, Seg{0, 0});
    recv->assign(world, Seg{0, 0});
    for (int o = 0; o < world; ++o) (*send)[o] = inter(rank, o);
    for (int r = 0; r < world; ++r) (*recv)[r] = inter(r, rank);
}

namespace {
std::atomic<bool> g_parse_unpacked{false};   // sinet_parse_set_knob("unpacked_look_back")
}  // namespace

extern "C" {

int sinet_exchange_plan(int32_t world, int32_t rank, uint64_t nbins, uint64_t nbins_pad, const uint32_t* touched,
                        uint64_t* send, uint64_t* recv) {
    if (world < 1 || rank < 0 || rank >= world || !touched || !send || !recv || nbins_pad % (uint64_t)world)
        return SINET_E_INVAL;
    std::vector<Seg> sd, rv;
    plan_exchange(world, rank, nbins, nbins_pad, touched, &sd, &rv);
    for (int k = 0; k < world; ++k) {
        send[2 * k] = sd[k].first; send[2 * k + 1] = sd[k].n;
        recv[2 * k] = rv[k].first; recv[2 * k + 1] = rv[k].n;
    }
    return SINET_OK;
}

int sinet_abi_version(void) { return SINET_ABI_VERSION; }

const char* sinet_last_kernel(const sinet_ctx* c) { return c ? c->last_kernel : ""; }
uint32_t sinet_tile_bins(void) { return kTileBins; }
uint32_t sinet_parse_chunk_bytes(void) { return kParseChunk; }

size_t sinet_bins_bytes(const sinet_config* cfg) {
    std::string err;
    Geometry g;
    if (!check_cfg(cfg, &err, &g)) return 0;
    return (size_t)g.B_pad * 32u;
}

size_t sinet_workspace_bytes(const sinet_config* cfg, uint32_t n_prefixes) {
    std::string err;
    Geometry g;
    if (!check_cfg(cfg, &err, &g) || n_prefixes == 0 || n_prefixes > kMaxPrefixes) return 0;
    return ws_layout(g.n_tiles, n_prefixes, cfg->world).total;
}

size_t sinet_staging_bytes(uint64_t chunk_records) {
    if (chunk_records == 0) return 0;
    size_t per = align_up(chunk_records * 8, 256) * 2 + align_up(chunk_records * 4, 256) * 2;
    return per * 2;
}

int sinet_open(sinet_ctx** out, const sinet_config* cfg, const uint32_t* prefix_net,
               const uint8_t* prefix_len, uint32_t n_prefixes, void* d_bins, size_t bins_bytes,
               void* d_ws, size_t ws_bytes) {
    return sinet_open_labelled(out, cfg, prefix_net, prefix_len, nullptr, n_prefixes, d_bins, bins_bytes, d_ws, ws_bytes);
}

int sinet_open_labelled(sinet_ctx** out, const sinet_config* cfg, const uint32_t* prefix_net,
                        const uint8_t* prefix_len, const uint8_t* prefix_label, uint32_t n_prefixes,
                        void* d_bins, size_t bins_bytes, void* d_ws, size_t ws_bytes) {
    if (!out) return SINET_E_INVAL;
    *out = nullptr;
    sinet_ctx* c = new (std::nothrow) sinet_ctx();
    if (!c) return SINET_E_INVAL;
    auto bail = [&](int code) { delete c; return code; };
    Geometry g;
    if (!check_cfg(cfg, &c->err, &g)) { std::fprintf(stderr, "sinet_open: %s\n", c->err.c_str()); return bail(SINET_E_INVAL); }
    if (!compile_prefixes_labelled(prefix_net, prefix_len, prefix_label, n_prefixes, &c->table, &c->err)) {
        std::fprintf(stderr, "sinet_open: %s\n", c->err.c_str());
        return bail(SINET_E_INVAL);
    }
    c->cfg = *cfg;
    c->geo = g;
    c->ws = ws_layout(g.n_tiles, n_prefixes, cfg->world);
    if (!d_bins || !d_ws || bins_bytes < (size_t)g.B_pad * 32u || ws_bytes < c->ws.total ||
        (reinterpret_cast<uintptr_t>(d_bins) & 255u) || (reinterpret_cast<uintptr_t>(d_ws) & 255u)) {
        std::fprintf(stderr, "sinet_open: bins/workspace buffer missing, too small or not 256-byte aligned\n");
        return bail(SINET_E_INVAL);
    }
    c->bins = static_cast<unsigned long long*>(d_bins);
    c->d_ws = static_cast<unsigned char*>(d_ws);
    c->stream = static_cast<cudaStream_t>(cfg->stream);
    c->device = cfg->device;
    c->nbnd = (uint32_t)c->table.bnd.size();
    for (int k = 0; k < 4; ++k) c->lut |= (uint32_t)cfg->dir_lut[k] << (2 * k);
    c->magic = (cfg->bin_width_ms >= 2) ? (uint32_t)((1ull << 32) / cfg->bin_width_ms) : 0u;

    DeviceGuard dg(c->device);
    if (!dg.ok) { std::fprintf(stderr, "sinet_open: cannot select device %d\n", c->device); return bail(SINET_E_CUDA); }
    cudaError_t e;
#define OPEN_CUDA(expr) \
    if ((e = (expr)) != cudaSuccess) { std::fprintf(stderr, "sinet_open: %s: %s\n", #expr, cudaGetErrorString(e)); return bail(SINET_E_CUDA); }
    OPEN_CUDA(cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, c->device));
    OPEN_CUDA(setup_hist_atomic());
    OPEN_CUDA(setup_hist_stream());
    OPEN_CUDA(setup_hist_ws());
    OPEN_CUDA(setup_partition());
    c->atomic_grid = c->sm_count * hist_atomic_blocks_per_sm(base_params(c));
    c->materialize_grid = c->sm_count * 8;
    // upload the compiled table; zero totals and tile states
    OPEN_CUDA(cudaMemsetAsync(c->d_ws + c->ws.totals, 0, 16 * 8, c->stream));
    OPEN_CUDA(cudaMemcpyAsync(c->d_ws + c->ws.cls2, c->table.cls2.data(), (size_t)kClsWords * 4, cudaMemcpyHostToDevice, c->stream));
    if (c->nbnd)
        OPEN_CUDA(cudaMemcpyAsync(c->d_ws + c->ws.bnd, c->table.bnd.data(), (size_t)c->nbnd * 4, cudaMemcpyHostToDevice, c->stream));
    OPEN_CUDA(cudaMemcpyAsync(c->d_ws + c->ws.rank, c->table.rank.data(), (size_t)kRankWords * 4, cudaMemcpyHostToDevice, c->stream));
    if (!c->table.mentry.empty())
        OPEN_CUDA(cudaMemcpyAsync(c->d_ws + c->ws.mentry, c->table.mentry.data(), c->table.mentry.size() * 4, cudaMemcpyHostToDevice, c->stream));
    if (!c->table.l2.empty())
        OPEN_CUDA(cudaMemcpyAsync(c->d_ws + c->ws.l2, c->table.l2.data(), c->table.l2.size() * 4, cudaMemcpyHostToDevice, c->stream));
    if (!c->table.b16.empty())
        OPEN_CUDA(cudaMemcpyAsync(c->d_ws + c->ws.b16, c->table.b16.data(), 65536, cudaMemcpyHostToDevice, c->stream));
    // the stream kernel stages b24 in whole 16-byte words plus one (b24[0] is always read):
    // zero the bytes past the table so that every staged byte is initialised
    OPEN_CUDA(cudaMemsetAsync(c->d_ws + c->ws.b24 + c->table.b24.size(), 0, 16, c->stream));
    if (!c->table.b24.empty())
        OPEN_CUDA(cudaMemcpyAsync(c->d_ws + c->ws.b24, c->table.b24.data(), c->table.b24.size(), cudaMemcpyHostToDevice, c->stream));
    OPEN_CUDA(cudaMemsetAsync(c->d_ws + c->ws.flags, 0, (size_t)g.n_tiles * 4, c->stream));
    OPEN_CUDA(cudaMemsetAsync(c->d_ws + c->ws.counters, 0, 64, c->stream));
    OPEN_CUDA(cudaMemsetAsync(c->d_ws + c->ws.counters + 16, 0xFF, 4, c->stream));   // touched min = ~0
    OPEN_CUDA(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
    for (int k = 0; k < 2; ++k) {
        OPEN_CUDA(cudaEventCreateWithFlags(&c->copy_done[k], cudaEventDisableTiming));
        OPEN_CUDA(cudaEventCreateWithFlags(&c->kern_done[k], cudaEventDisableTiming));
    }
    OPEN_CUDA(cudaStreamSynchronize(c->stream));
#undef OPEN_CUDA
    *out = c;
    return SINET_OK;
}

void sinet_close(sinet_ctx* c) {
    if (!c) return;
    {
        DeviceGuard dg(c->device);
        if (c->stream) cudaStreamSynchronize(c->stream);
        for (auto& pr : c->tev) { cudaEventDestroy(pr.first); cudaEventDestroy(pr.second); }
        for (int k = 0; k < 2; ++k) {
            if (c->copy_done[k]) cudaEventDestroy(c->copy_done[k]);
            if (c->kern_done[k]) cudaEventDestroy(c->kern_done[k]);
        }
        if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
        c->comm.reset();
    }
    delete c;
}

int sinet_reset(sinet_ctx* c) {
    if (!c) return SINET_E_INVAL;
    DeviceGuard dg(c->device);
    SINET_CUDA(c, cudaMemsetAsync(c->d_ws + c->ws.totals, 0, 16 * 8, c->stream));
    SINET_CUDA(c, cudaMemsetAsync(c->d_ws + c->ws.counters + 16, 0xFF, 4, c->stream));   // touched min
    SINET_CUDA(c, cudaMemsetAsync(c->d_ws + c->ws.counters + 20, 0, 4, c->stream));      // touched max
    c->epoch++;
    if (c->epoch >= (1u << 30)) {   // epoch space exhausted: re-zero the state words
        SINET_CUDA(c, cudaMemsetAsync(c->d_ws + c->ws.flags, 0, (size_t)c->geo.n_tiles * 4, c->stream));
        c->epoch = 1;
    }
    c->reduced = false;
    c->materialized = false;
    c->auto_choice = 0;
    return SINET_OK;
}

int sinet_classify_histogram(sinet_ctx* c, const sinet_records* r, uint8_t* d_tags) {
    if (!c) return SINET_E_INVAL;
    DeviceGuard dg(c->device);
    return classify_device(c, r, d_tags);
}

int sinet_classify_histogram_host(sinet_ctx* c, const sinet_records* h, void* d_staging,
                                  size_t staging_bytes, uint64_t chunk) {
    if (!c) return SINET_E_INVAL;
    if (!h) return fail(c, SINET_E_INVAL, "NULL records");
    if (c->reduced) return fail(c, SINET_E_STATE, "classify after reduce: call sinet_reset first");
    if (h->n == 0) return SINET_OK;
    if (!h->ts_ms || !h->src || !h->dst || !h->bytes) return fail(c, SINET_E_INVAL, "NULL record column");
    if (chunk == 0 || !d_staging || staging_bytes < sinet_staging_bytes(chunk) ||
        (reinterpret_cast<uintptr_t>(d_staging) & 255u))
        return fail(c, SINET_E_INVAL, "staging buffer missing, too small or not 256-byte aligned");
    DeviceGuard dg(c->device);
    const size_t o_ts = 0, o_src = align_up(chunk * 8, 256), o_dst = o_src + align_up(chunk * 4, 256),
                 o_by = o_dst + align_up(chunk * 4, 256), per = o_by + align_up(chunk * 8, 256);
    unsigned char* stage = static_cast<unsigned char*>(d_staging);
    uint64_t k = 0;
    for (uint64_t lo = 0; lo < h->n; lo += chunk, ++k) {
        const uint64_t m = (h->n - lo < chunk) ? h->n - lo : chunk;
        const int b = (int)(k & 1);
        unsigned char* buf = stage + per * b;
        if (k >= 2) SINET_CUDA(c, cudaStreamWaitEvent(c->copy_stream, c->kern_done[b], 0));
        SINET_CUDA(c, cudaMemcpyAsync(buf + o_ts, h->ts_ms + lo, m * 8, cudaMemcpyHostToDevice, c->copy_stream));
        SINET_CUDA(c, cudaMemcpyAsync(buf + o_src, h->src + lo, m * 4, cudaMemcpyHostToDevice, c->copy_stream));
        SINET_CUDA(c, cudaMemcpyAsync(buf + o_dst, h->dst + lo, m * 4, cudaMemcpyHostToDevice, c->copy_stream));
        SINET_CUDA(c, cudaMemcpyAsync(buf + o_by, h->bytes + lo, m * 8, cudaMemcpyHostToDevice, c->copy_stream));
        SINET_CUDA(c, cudaEventRecord(c->copy_done[b], c->copy_stream));
        SINET_CUDA(c, cudaStreamWaitEvent(c->stream, c->copy_done[b], 0));
        sinet_records dr{reinterpret_cast<const uint64_t*>(buf + o_ts), reinterpret_cast<const uint32_t*>(buf + o_src),
                         reinterpret_cast<const uint32_t*>(buf + o_dst), reinterpret_cast<const uint64_t*>(buf + o_by), m};
        int rc = classify_device(c, &dr, nullptr);
        if (rc) return rc;
        SINET_CUDA(c, cudaEventRecord(c->kern_done[b], c->stream));
    }
    SINET_CUDA(c, cudaStreamSynchronize(c->stream));
    return SINET_OK;
}

size_t sinet_partition_scratch_bytes(const sinet_config* cfg, uint64_t max_records) {
    std::string err;
    Geometry g;
    if (!check_cfg(cfg, &err, &g) || !partition_supported((uint32_t)g.B) || max_records < kPartMinCap) return 0;
    return part_layout((max_records + 3) & ~3ull, (uint32_t)g.B).total;
}

int sinet_set_scratch(sinet_ctx* c, void* d_scratch, size_t bytes) {
    if (!c) return SINET_E_INVAL;
    if (!d_scratch || bytes == 0) { c->scratch = nullptr; c->scratch_bytes = 0; c->scratch_cap = 0; return SINET_OK; }
    if (reinterpret_cast<uintptr_t>(d_scratch) & 255u) return fail(c, SINET_E_ALIGN, "scratch must be 256-byte aligned");
    if (!partition_supported((uint32_t)c->geo.B)) return fail(c, SINET_E_INVAL, "partitioned path: window of more than 2^27 bins");
    // the largest multiple of 4 records (< 2^31: u32 offsets) whose layout fits
    uint64_t lo = 0, hi = (bytes / 24u + 4u) & ~3ull;
    if (hi >= (1ull << 31)) hi = (1ull << 31) - 4u;
    while (lo < hi) {
        const uint64_t mid = ((lo + hi) / 2 + 4u) & ~3ull;
        if (mid > hi) break;
        if (part_layout(mid, (uint32_t)c->geo.B).total <= bytes) lo = mid; else hi = mid - 4u;
    }
    if (lo < kPartMinCap) return fail(c, SINET_E_INVAL, "scratch smaller than sinet_partition_scratch_bytes(cfg, 2^16)");
    c->scratch = d_scratch;
    c->scratch_bytes = bytes;
    c->scratch_cap = lo;
    return SINET_OK;
}

size_t sinet_sortreduce_scratch_bytes(const sinet_config* cfg, uint64_t n) {
    std::string err;
    Geometry g;
    if (!check_cfg(cfg, &err, &g) || n >= (1ull << 31) || g.B * 2 >= (1ull << 32)) return 0;
    return sortreduce_scratch_bytes(n, g.B);
}

int sinet_classify_histogram_sortreduce(sinet_ctx* c, const sinet_records* r, void* d_scratch, size_t scratch_bytes) {
    if (!c) return SINET_E_INVAL;
    KernelParams p;
    int prc = prepare_params(c, r, nullptr, &p);
    if (prc) return prc;
    if (r->n == 0) return SINET_OK;
    if (r->n >= (1ull << 31) || c->geo.B * 2 >= (1ull << 32))
        return fail(c, SINET_E_INVAL, "sort-reduce comparator: n < 2^31 and 2B < 2^32 required");
    if (!d_scratch || scratch_bytes < sortreduce_scratch_bytes(r->n, c->geo.B))
        return fail(c, SINET_E_INVAL, "sort-reduce comparator: scratch buffer too small");
    DeviceGuard dg(c->device);
    int rc = do_materialize(c);
    if (rc) return rc;
    int k = 0;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (c->timing) {
        SINET_CUDA(c, cudaEventCreate(&e0));
        SINET_CUDA(c, cudaEventCreate(&e1));
        SINET_CUDA(c, cudaEventRecord(e0, c->stream));
    }
    SINET_CUDA(c, launch_sortreduce(p, d_scratch, scratch_bytes, c->sm_count, c->stream, &k));
    if (c->timing) {
        SINET_CUDA(c, cudaEventRecord(e1, c->stream));
        c->tev.emplace_back(e0, e1);
    }
    c->launches += (uint64_t)k;
    c->last_strategy = 3;
    return SINET_OK;
}

size_t sinet_watchlist_bytes(uint32_t n) { return (size_t)2048 * 4 + align_up((size_t)n * 4, 256); }

int sinet_set_watchlist(sinet_ctx* c, const uint32_t* ips, uint32_t n, void* d_buf, size_t buf_bytes) {
    if (!c) return SINET_E_INVAL;
    if (n == 0) { c->wn = 0; c->wbits = c->wlist = nullptr; return SINET_OK; }
    if (!ips || !d_buf || buf_bytes < sinet_watchlist_bytes(n) || (reinterpret_cast<uintptr_t>(d_buf) & 15u))
        return fail(c, SINET_E_INVAL, "watchlist: NULL list or device buffer too small / misaligned");
    std::vector<uint32_t> list(ips, ips + n);
    std::sort(list.begin(), list.end());
    list.erase(std::unique(list.begin(), list.end()), list.end());   // set semantics
    std::vector<uint32_t> bits(2048, 0u);
    for (uint32_t a : list) bits[a >> 21] |= 1u << ((a >> 16) & 31u);
    DeviceGuard dg(c->device);
    unsigned char* b = static_cast<unsigned char*>(d_buf);
    SINET_CUDA(c, cudaMemcpyAsync(b, bits.data(), 2048 * 4, cudaMemcpyHostToDevice, c->stream));
    SINET_CUDA(c, cudaMemcpyAsync(b + 2048 * 4, list.data(), list.size() * 4, cudaMemcpyHostToDevice, c->stream));
    SINET_CUDA(c, cudaStreamSynchronize(c->stream));
    c->wbits = reinterpret_cast<const uint32_t*>(b);
    c->wlist = reinterpret_cast<const uint32_t*>(b + 2048 * 4);
    c->wn = (uint32_t)list.size();
    return SINET_OK;
}

int sinet_finalize(sinet_ctx* c) {
    if (!c) return SINET_E_INVAL;
    if (c->reduced) return SINET_OK;
    DeviceGuard dg(c->device);
    return do_materialize(c);
}

int sinet_nccl_unique_id(void* out) {
    if (!out) return SINET_E_INVAL;
    std::string err;
    int rc = nccl_unique_id(out, &err);
    if (rc) std::fprintf(stderr, "sinet_nccl_unique_id: %s\n", err.c_str());
    return rc;
}

int sinet_comm_init(sinet_ctx* c, const void* uid) {
    if (!c) return SINET_E_INVAL;
    if (!uid) return fail(c, SINET_E_INVAL, "NULL unique id");
    if (c->comm) return fail(c, SINET_E_STATE, "communicator already initialised");
    DeviceGuard dg(c->device);
    c->comm = make_nccl_transport(c->cfg.world, c->cfg.rank, uid, &c->err);
    return c->comm ? SINET_OK : SINET_E_NCCL;
}

int sinet_comm_init_hub(sinet_ctx* c, sinet_hub* hub) {
    if (!c) return SINET_E_INVAL;
    if (!hub) return fail(c, SINET_E_INVAL, "NULL hub");
    if (c->comm) return fail(c, SINET_E_STATE, "communicator already initialised");
    if (hub_world(hub) != c->cfg.world) return fail(c, SINET_E_INVAL, "hub world differs from cfg.world");
    DeviceGuard dg(c->device);
    c->comm = make_hub_transport(hub, c->cfg.rank, c->device, &c->err);
    return c->comm ? SINET_OK : SINET_E_INVAL;
}

// Merge-scatter through the ctx's transport.  The same code runs over NCCL
// (one process per GPU) and over the in-process hub (one thread per GPU).
int sinet_reduce(sinet_ctx* c) {
    if (!c) return SINET_E_INVAL;
    if (c->reduced) return fail(c, SINET_E_STATE, "already reduced: call sinet_reset first");
    DeviceGuard dg(c->device);
    const int world = c->cfg.world, rank = c->cfg.rank;
    const bool may_sparse = world > 1 && c->comm && c->exchange != 1 && c->ws.staging_bytes;
    if (!may_sparse) {
        int rc = do_materialize(c);
        if (rc) return rc;
    }
    if (world > 1 || c->comm) {
        if (!c->comm) return fail(c, SINET_E_NCCL, "no communicator: call sinet_comm_init or sinet_comm_init_hub");
        Transport* T = c->comm.get();
        const int tcode = std::strcmp(T->name(), "nccl") == 0 ? SINET_E_NCCL : SINET_E_CUDA;
        const size_t slice = (size_t)(c->geo.B_pad / (uint64_t)world) * 4u;   // u64 per rank
        unsigned long long* tot = reinterpret_cast<unsigned long long*>(c->d_ws + c->ws.totals);
        unsigned long long* xtot = reinterpret_cast<unsigned long long*>(c->d_ws + c->ws.xtotals);
        bool sparse = false;
        std::vector<Seg> sd, rv;
        int rc = SINET_OK;
        if (may_sparse) {
            // every rank's touched range, then the same plan (and decision) on every rank
            uint32_t* xr = ws_u32(c, c->ws.xranges);
            rc = T->all_gather_u32(ws_u32(c, c->ws.counters) + 4, xr, 2, c->stream, &c->err);
            if (rc) return fail(c, rc == SINET_E_NCCL ? SINET_E_NCCL : tcode, "touched-range all-gather: " + c->err);
            std::vector<uint32_t> h((size_t)world * 2);
            SINET_CUDA(c, cudaMemcpyAsync(h.data(), xr, h.size() * 4, cudaMemcpyDeviceToHost, c->stream));
            SINET_CUDA(c, cudaStreamSynchronize(c->stream));
            uint64_t worst_recv = 0, total_moved = 0;
            for (int o = 0; o < world; ++o) {
                std::vector<Seg> s_o, r_o;
                plan_exchange(world, o, c->geo.B, c->geo.B_pad, h.data(), &s_o, &r_o);
                uint64_t rb = 0;
                for (auto& g : r_o) rb += g.n;
                total_moved += rb;
                if (rb > worst_recv) worst_recv = rb;
            }
            const uint64_t dense_moved = (uint64_t)(world - 1) * (c->geo.B_pad / (uint64_t)world) * (uint64_t)world;
            sparse = (c->exchange == 2 || total_moved * 2 <= dense_moved) &&
                     worst_recv * 32u <= (uint64_t)c->ws.staging_bytes;
            if (sparse) {
                plan_exchange(world, rank, c->geo.B, c->geo.B_pad, h.data(), &sd, &rv);
                // materialise only the owned slice and the slices sent (others stay virtual)
                const uint64_t per = c->geo.B_pad / (uint64_t)world;
                auto mat = [&](uint64_t b_lo, uint64_t b_n) -> int {
                    if (!b_n) return SINET_OK;
                    const uint32_t t0 = (uint32_t)(b_lo / kTileBins);
                    const uint32_t t1 = (uint32_t)((b_lo + b_n + kTileBins - 1) / kTileBins);
                    SINET_CUDA(c, launch_materialize_range(c->bins, ws_u32(c, c->ws.flags), t0, t1, init_word(c),
                                                           c->materialize_grid, c->stream));
                    c->launches++;
                    return SINET_OK;
                };
                int mrc = mat(per * (uint64_t)rank, per);
                for (int o = 0; o < world && !mrc; ++o) mrc = mat(sd[o].first, sd[o].n);
                if (mrc) return mrc;
            } else {
                int mrc = do_materialize(c);
                if (mrc) return mrc;
            }
        }
        rc = T->group_start(&c->err);
        if (!rc && sparse) {
            // only the touched overlaps travel: send my partial bins inside each owner's range,
            // receive the other ranks' partial bins of my owned range into staging
            unsigned long long* stage = reinterpret_cast<unsigned long long*>(c->d_ws + c->ws.staging);
            size_t off = 0;
            for (int o = 0; o < world && !rc; ++o)
                if (sd[o].n) rc = T->send_u64(c->bins + sd[o].first * 4u, sd[o].n * 4u, o, c->stream, &c->err);
            for (int q = 0; q < world && !rc; ++q)
                if (rv[q].n) { rc = T->recv_u64(stage + off, rv[q].n * 4u, q, c->stream, &c->err); off += rv[q].n * 4u; }
        } else if (!rc) {
            rc = T->reduce_scatter_u64(c->bins, c->bins + slice * (size_t)rank, slice, c->stream, &c->err);
            if (!rc && std::strcmp(T->name(), "hub") == 0) c->launches++;   // k_sum_peers
        }
        if (!rc) {
            rc = T->all_reduce_u64(tot, tot, 12, xtot, c->stream, &c->err);
            if (!rc && std::strcmp(T->name(), "hub") == 0) c->launches++;
        }
        const int rc2 = T->group_end(c->stream, rc ? &c->err : &c->err);
        if (!rc) rc = rc2;
        if (rc) return fail(c, rc, std::string("merge (") + T->name() + "): " + c->err);
        if (sparse) {
            const unsigned long long* stage = reinterpret_cast<const unsigned long long*>(c->d_ws + c->ws.staging);
            size_t off = 0;
            for (int q = 0; q < world; ++q)
                if (rv[q].n) {
                    SINET_CUDA(c, launch_add_bins(c->bins, stage + off, rv[q].first, rv[q].n, c->sm_count, c->stream));
                    c->launches++;
                    off += rv[q].n * 4u;
                }
        }
        c->last_exchange = sparse ? 2 : 1;
    }
    c->reduced = true;
    return SINET_OK;
}

int sinet_last_exchange(const sinet_ctx* c) { return c ? c->last_exchange : 0; }

int sinet_touched_range(sinet_ctx* c, uint32_t* min_bin, uint32_t* max_bin) {
    if (!c || !min_bin || !max_bin) return SINET_E_INVAL;
    DeviceGuard dg(c->device);
    uint32_t h[2];
    SINET_CUDA(c, cudaMemcpyAsync(h, c->d_ws + c->ws.counters + 16, 8, cudaMemcpyDeviceToHost, c->stream));
    SINET_CUDA(c, cudaStreamSynchronize(c->stream));
    *min_bin = h[0];
    *max_bin = h[1];
    return SINET_OK;
}

int sinet_set_exchange(sinet_ctx* c, int mode) {
    if (!c || mode < 0 || mode > 2) return c ? fail(c, SINET_E_INVAL, "exchange mode must be 0, 1 or 2") : SINET_E_INVAL;
    c->exchange = mode;
    return SINET_OK;
}

int sinet_owned_range(sinet_ctx* c, uint64_t* first, uint64_t* n) {
    if (!c || !first || !n) return SINET_E_INVAL;
    if (!c->reduced || c->cfg.world == 1) { *first = 0; *n = c->geo.B; return SINET_OK; }
    uint64_t per = c->geo.B_pad / (uint64_t)c->cfg.world;
    uint64_t lo = per * (uint64_t)c->cfg.rank, hi = lo + per;
    if (lo > c->geo.B) lo = c->geo.B;
    if (hi > c->geo.B) hi = c->geo.B;
    *first = lo;
    *n = hi - lo;
    return SINET_OK;
}

int sinet_read_bins(sinet_ctx* c, int dir, int metric, uint64_t first, uint64_t n, uint64_t* dst, int dst_is_device) {
    if (!c) return SINET_E_INVAL;
    if (dir != SINET_DIR_OUT && dir != SINET_DIR_IN) return fail(c, SINET_E_INVAL, "dir must be SINET_DIR_OUT or SINET_DIR_IN");
    if (metric != SINET_METRIC_COUNT && metric != SINET_METRIC_BYTES) return fail(c, SINET_E_INVAL, "metric must be COUNT or BYTES");
    uint64_t lo, cnt;
    sinet_owned_range(c, &lo, &cnt);
    if (first < lo || first > lo + cnt || n > lo + cnt - first) return fail(c, SINET_E_RANGE, "bin range outside the owned range");
    if (n == 0) return SINET_OK;
    if (!dst) return fail(c, SINET_E_INVAL, "NULL destination");
    DeviceGuard dg(c->device);
    int rc = c->reduced ? SINET_OK : do_materialize(c);
    if (rc) return rc;
    const unsigned long long* srcp = c->bins + (first * 4u + (uint64_t)dir * 2u + (uint64_t)metric);
    SINET_CUDA(c, cudaMemcpy2DAsync(dst, 8, srcp, 32, 8, n, dst_is_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, c->stream));
    if (!dst_is_device) SINET_CUDA(c, cudaStreamSynchronize(c->stream));
    return SINET_OK;
}

int sinet_read_bins_raw(sinet_ctx* c, uint64_t first, uint64_t n, uint64_t* dst, int dst_is_device) {
    if (!c) return SINET_E_INVAL;
    uint64_t lo, cnt;
    sinet_owned_range(c, &lo, &cnt);
    if (first < lo || first > lo + cnt || n > lo + cnt - first) return fail(c, SINET_E_RANGE, "bin range outside the owned range");
    if (n == 0) return SINET_OK;
    if (!dst) return fail(c, SINET_E_INVAL, "NULL destination");
    DeviceGuard dg(c->device);
    int rc = c->reduced ? SINET_OK : do_materialize(c);
    if (rc) return rc;
    SINET_CUDA(c, cudaMemcpyAsync(dst, c->bins + first * 4u, n * 32u,
                                  dst_is_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, c->stream));
    if (!dst_is_device) SINET_CUDA(c, cudaStreamSynchronize(c->stream));
    return SINET_OK;
}

int sinet_rebin_frames(sinet_ctx* c, uint64_t factor, uint64_t* first_frame, uint64_t* n_frames) {
    if (!c || factor == 0 || !first_frame || !n_frames) return c ? fail(c, SINET_E_INVAL, "rebin_frames: bad argument") : SINET_E_INVAL;
    uint64_t lo, cnt;
    sinet_owned_range(c, &lo, &cnt);
    // frame k = absolute bins [k*factor, (k+1)*factor): the owned range meets frames
    // floor(lo/f) .. ceil((lo+cnt)/f) - 1
    *first_frame = lo / factor;
    *n_frames = cnt ? (lo + cnt + factor - 1) / factor - lo / factor : 0;
    return SINET_OK;
}

int sinet_rebin(sinet_ctx* c, uint64_t factor, uint64_t* d_out, uint64_t n_out) {
    if (!c) return SINET_E_INVAL;
    if (factor == 0 || !d_out || (reinterpret_cast<uintptr_t>(d_out) & 7u))
        return fail(c, SINET_E_INVAL, "rebin: factor must be >= 1 and d_out an 8-byte aligned device buffer");
    uint64_t lo, cnt, f0, nf;
    sinet_owned_range(c, &lo, &cnt);
    sinet_rebin_frames(c, factor, &f0, &nf);
    if (n_out != nf) return fail(c, SINET_E_INVAL, "rebin: n_out must be the frame count of sinet_rebin_frames");
    DeviceGuard dg(c->device);
    int rc = c->reduced ? SINET_OK : do_materialize(c);
    if (rc) return rc;
    SINET_CUDA(c, launch_rebin(c->bins, lo, lo + cnt, factor, reinterpret_cast<unsigned long long*>(d_out), n_out,
                               c->sm_count, c->stream));
    c->launches += (cnt ? 1 : 0);
    return SINET_OK;
}

int sinet_export_sparse(sinet_ctx* c, int dir, uint64_t* d_ts, uint64_t* d_count, uint64_t* d_bytes,
                        uint64_t capacity, uint64_t* n_nonzero) {
    if (!c) return SINET_E_INVAL;
    if (dir != SINET_DIR_OUT && dir != SINET_DIR_IN) return fail(c, SINET_E_INVAL, "dir must be SINET_DIR_OUT or SINET_DIR_IN");
    if (!n_nonzero || (capacity && (!d_ts || !d_count || !d_bytes)))
        return fail(c, SINET_E_INVAL, "export_sparse: NULL output");
    uint64_t lo, cnt;
    sinet_owned_range(c, &lo, &cnt);
    DeviceGuard dg(c->device);
    int rc = c->reduced ? SINET_OK : do_materialize(c);
    if (rc) return rc;
    unsigned long long* d_total = reinterpret_cast<unsigned long long*>(c->d_ws + c->ws.sparse);
    uint32_t* scratch = reinterpret_cast<uint32_t*>(c->d_ws + c->ws.sparse + 16);
    SINET_CUDA(c, launch_sparse(c->bins, lo, lo + cnt, (uint32_t)dir, scratch, d_total, c->cfg.window_start_ms,
                                c->cfg.bin_width_ms, reinterpret_cast<unsigned long long*>(d_ts),
                                reinterpret_cast<unsigned long long*>(d_count),
                                reinterpret_cast<unsigned long long*>(d_bytes), capacity, c->stream));
    c->launches += cnt ? (capacity ? 3 : 2) : 0;
    unsigned long long h = 0;
    SINET_CUDA(c, cudaMemcpyAsync(&h, d_total, 8, cudaMemcpyDeviceToHost, c->stream));
    SINET_CUDA(c, cudaStreamSynchronize(c->stream));
    *n_nonzero = h;
    return SINET_OK;
}

int sinet_read_totals(sinet_ctx* c, sinet_totals* out) {
    if (!c || !out) return c ? fail(c, SINET_E_INVAL, "NULL output") : SINET_E_INVAL;
    DeviceGuard dg(c->device);
    unsigned long long h[12];
    SINET_CUDA(c, cudaMemcpyAsync(h, c->d_ws + c->ws.totals, sizeof h, cudaMemcpyDeviceToHost, c->stream));
    SINET_CUDA(c, cudaStreamSynchronize(c->stream));
    for (int k = 0; k < 4; ++k) { out->m_count[k] = h[k]; out->m_bytes[k] = h[4 + k]; }
    out->oow_count[0] = h[8]; out->oow_count[1] = h[9];
    out->oow_bytes[0] = h[10]; out->oow_bytes[1] = h[11];
    return SINET_OK;
}

int sinet_table_member_host(const uint32_t* net, const uint8_t* len, uint32_t np,
                            const uint32_t* ips, uint64_t n, uint8_t* out) {
    return sinet_table_member_host_labelled(net, len, nullptr, np, ips, n, out);
}

int sinet_table_member_host_labelled(const uint32_t* net, const uint8_t* len, const uint8_t* label, uint32_t np,
                                     const uint32_t* ips, uint64_t n, uint8_t* out) {
    CompiledTable t;
    std::string err;
    if (!compile_prefixes_labelled(net, len, label, np, &t, &err)) return SINET_E_INVAL;
    if (n && (!ips || !out)) return SINET_E_INVAL;
    auto search = [&](uint32_t e, uint32_t ip) {   // #boundaries <= ip, from a block's entry
        uint32_t cnt = e & 0xFFFFu, m = e >> 16;
        const uint32_t* b = t.bnd.data() + cnt;
        while (m) {
            uint32_t half = m >> 1;
            if (b[half] <= ip) { b += half + 1; cnt += half + 1; m -= half + 1; }
            else m = half;
        }
        return cnt & 1u;
    };
    const bool have_bytes = !t.b16.empty();
    for (uint64_t i = 0; i < n; ++i) {
        // the kernels' lookups (sinet_device.cuh member() / member_batch(), all three table
        // encodings), evaluated on the host; an encoding that disagrees is a compiler bug
        uint32_t ip = ips[i], x = ip >> 16;
        uint32_t c = (t.cls2[x >> 4] >> ((x & 15u) * 2u)) & 3u;
        uint32_t r_packed = c, r_nol2 = c, r_byte = c;
        if (c == 2u) {
            // mixed block: rank + level-2 /24 classes + per-block entry
            const uint32_t w = t.cls2[x >> 4], sh = (x & 15u) * 2u;
            const uint32_t mixed = (w >> 1) & ~w & 0x55555555u;
            const uint16_t* rk = reinterpret_cast<const uint16_t*>(t.rank.data());
            const uint32_t mi = rk[x >> 4] + (uint32_t)__builtin_popcount(mixed & ((1u << sh) - 1u));
            if (mi >= t.n_mixed || t.mentry[mi] != t.entry[x]) return SINET_E_INVAL;
            const uint32_t y = (ip >> 8) & 0xFFu;
            const uint32_t c2 = (t.l2[(size_t)mi * 16u + (y >> 4)] >> ((y & 15u) * 2u)) & 3u;
            r_packed = (c2 < 2u) ? c2 : search(t.mentry[mi], ip);
            // packed encoding without level 2: the block's inline entries as stage_stream_table
            // builds them (<= 7 boundaries as u16 low half - 1), else the search
            const uint32_t me = t.mentry[mi], lo = me & 0xFFFFu, nb = me >> 16;
            if (nb <= 7u) {
                uint32_t cnt = 0;
                for (uint32_t j = 0; j < 7u; ++j) {
                    const uint32_t v = (j < nb) ? ((t.bnd[lo + j] & 0xFFFFu) - 1u) : 0xFFFFu;
                    cnt += v < (ip & 0xFFFFu) ? 1u : 0u;
                }
                r_nol2 = (cnt ^ lo) & 1u;
            } else {
                r_nol2 = search(me, ip);
            }
        }
        if (have_bytes) {   // byte encoding: b16, then b24 of the mixed block, then its search
            const uint32_t b = t.b16[x];
            if (b < 2u) r_byte = b;
            else {
                const uint32_t m = b - 2u, b2 = t.b24[(size_t)m * 256u + ((ip >> 8) & 0xFFu)];
                r_byte = (b2 < 2u) ? b2 : search(t.mentry[m], ip);
            }
        } else {
            r_byte = r_packed;
        }
        if (r_nol2 != r_packed || r_byte != r_packed) return SINET_E_INVAL;
        out[i] = (uint8_t)r_packed;
    }
    return SINET_OK;
}

const char* sinet_last_error(const sinet_ctx* c) { return c ? c->err.c_str() : "NULL ctx"; }
uint64_t sinet_launch_count(const sinet_ctx* c) { return c ? c->launches : 0; }
int sinet_last_strategy(const sinet_ctx* c) { return c ? c->last_strategy : 0; }

int sinet_set_tuning(sinet_ctx* c, int stream_groups, int warp_aggregation) {
    if (!c) return SINET_E_INVAL;
    if (stream_groups < 0 || stream_groups > 2 || warp_aggregation < -1 || warp_aggregation > 1)
        return fail(c, SINET_E_INVAL, "stream_groups must be 0, 1 or 2; warp_aggregation -1, 0 or 1");
    c->stream_groups = (uint32_t)stream_groups;
    if (warp_aggregation >= 0) c->agg = warp_aggregation != 0;
    return SINET_OK;
}

int sinet_set_knob(sinet_ctx* c, const char* name, int64_t value) {
    if (!c) return SINET_E_INVAL;
    if (!name) return fail(c, SINET_E_INVAL, "NULL knob name");
    const std::string k(name);
    auto range = [&](int64_t lo, int64_t hi) { return value >= lo && value <= hi; };
    if (k == "stream_groups" && range(0, 2)) c->stream_groups = (uint32_t)value;
    else if (k == "warp_aggregation" && range(0, 1)) c->agg = value != 0;
    else if (k == "stream_kernel" && range(0, 2)) c->stream_kernel = (uint32_t)value;
    else if (k == "shuffled_kernel" && range(0, 1)) c->shuffled_kernel = (uint32_t)value;
    else if (k == "debug_counters" && range(0, 1)) c->debug = (uint32_t)value;
    else if (k == "ranges_per_group" && range(0, 64)) c->ranges_per_group = (uint32_t)value;
    else if (k == "table_mode" && range(-1, 3)) c->tab_mode = (int)value;
    else if (k == "exchange" && range(0, 2)) c->exchange = (int)value;
    else return fail(c, SINET_E_INVAL, "unknown knob or value out of range: " + k);
    return SINET_OK;
}

int sinet_set_table_mode(sinet_ctx* c, int mode) {
    if (!c) return SINET_E_INVAL;
    if (mode < -1 || mode > 3) return fail(c, SINET_E_INVAL, "table mode must be -1 (automatic) or 0..3");
    c->tab_mode = mode;
    return SINET_OK;
}

int sinet_table_mode(const sinet_ctx* c) {
    if (!c) return SINET_E_INVAL;
    return stream_table_mode(!c->table.b16.empty(), c->nbnd, c->table.n_mixed, c->tab_mode);
}

int sinet_set_kernel_timing(sinet_ctx* c, int on) {
    if (!c) return SINET_E_INVAL;
    DeviceGuard dg(c->device);
    SINET_CUDA(c, cudaStreamSynchronize(c->stream));
    for (auto& pr : c->tev) { cudaEventDestroy(pr.first); cudaEventDestroy(pr.second); }
    c->tev.clear();
    c->timing = on != 0;
    return SINET_OK;
}

int sinet_kernel_time(sinet_ctx* c, double* total_ms, uint64_t* launches) {
    if (!c || !total_ms || !launches) return SINET_E_INVAL;
    DeviceGuard dg(c->device);
    SINET_CUDA(c, cudaStreamSynchronize(c->stream));
    double t = 0;
    for (auto& pr : c->tev) {
        float ms = 0;
        SINET_CUDA(c, cudaEventElapsedTime(&ms, pr.first, pr.second));
        t += ms;
    }
    *total_ms = t;
    *launches = c->tev.size();
    return SINET_OK;
}

}  // extern "C"

// ------------------------------------------------------------------ NEXT-3: text parser
namespace {
thread_local std::string g_parse_err;
int parse_fail(int code, const std::string& msg) {
    g_parse_err = msg;
    return code;
}
int parse_sm_count() {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms > 0 ? sms : 1;
}
// workspace: ticket (8) + result (10 x 8) padded to 256, then two look-back arrays
uint64_t parse_chunks(uint64_t text_bytes) { return (text_bytes + kParseChunk - 1) / kParseChunk; }
}  // namespace

extern "C" size_t sinet_parse_workspace_bytes(uint64_t text_bytes) {
    return 256u + 16u * (size_t)parse_chunks(text_bytes);
}

extern "C" const char* sinet_parse_last_error(void) { return g_parse_err.c_str(); }

extern "C" int sinet_parse_set_knob(const char* name, int64_t value) {
    if (!name) return SINET_E_INVAL;
    if (std::string(name) == "unpacked_look_back" && (value == 0 || value == 1)) {
        g_parse_unpacked.store(value != 0, std::memory_order_relaxed);
        return SINET_OK;
    }
    return SINET_E_INVAL;
}

int sinet_parse_text(const uint8_t* d_text, uint64_t text_bytes, int32_t tz_offset_min,
                                const sinet_columns* out, uint8_t* d_status, uint64_t status_capacity,
                                void* d_ws, size_t ws_bytes, void* stream, sinet_parse_result* result) {
    g_parse_err.clear();
    if (!result || !out) return parse_fail(SINET_E_INVAL, "parse_text: NULL result or columns");
    if (tz_offset_min < -1440 || tz_offset_min > 1440)
        return parse_fail(SINET_E_INVAL, "parse_text: tz_offset_min outside [-1440, 1440]");
    if (out->capacity && (!out->ts_ms || !out->src || !out->dst || !out->bytes))
        return parse_fail(SINET_E_INVAL, "parse_text: NULL output column with capacity > 0");
    if (text_bytes && !d_text) return parse_fail(SINET_E_INVAL, "parse_text: NULL text");
    if (!d_ws || ws_bytes < sinet_parse_workspace_bytes(text_bytes) || (reinterpret_cast<uintptr_t>(d_ws) & 255u))
        return parse_fail(SINET_E_INVAL, "parse_text: workspace missing, too small or not 256-byte aligned");
    if ((reinterpret_cast<uintptr_t>(d_text) & 15u) || (reinterpret_cast<uintptr_t>(out->ts_ms) & 7u) ||
        (reinterpret_cast<uintptr_t>(out->bytes) & 7u) || (reinterpret_cast<uintptr_t>(out->src) & 3u) ||
        (reinterpret_cast<uintptr_t>(out->dst) & 3u))
        return parse_fail(SINET_E_ALIGN, "parse_text: text must be 16-byte aligned, columns naturally aligned");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const uint64_t nch = parse_chunks(text_bytes);
    uint8_t* ws = reinterpret_cast<uint8_t*>(d_ws);
    cudaError_t e = cudaMemsetAsync(ws, 0, 256u + 16u * (size_t)nch, st);
    unsigned long long* res = reinterpret_cast<unsigned long long*>(ws + 8);
    if (e == cudaSuccess) e = cudaMemsetAsync(res + 2, 0xFF, 8, st);   // first bad line: none
    ParseParams p{};
    p.text = d_text;
    p.len = text_bytes;
    p.tz_offset_min = tz_offset_min;
    p.ts = out->ts_ms;
    p.src = out->src;
    p.dst = out->dst;
    p.bytes = out->bytes;
    p.cap = out->capacity;
    p.status = d_status;
    p.status_cap = d_status ? status_capacity : 0;
    p.ticket = reinterpret_cast<unsigned long long*>(ws);
    p.result = res;
    p.st_lines = reinterpret_cast<unsigned long long*>(ws + 256);
    p.st_valid = p.st_lines + nch;
    p.n_chunks = nch;
    p.packed = text_bytes < (1ull << 31) ? 1u : 0u;
    if (g_parse_unpacked.load(std::memory_order_relaxed)) p.packed = 0u;   // knob "unpacked_look_back"
    if (e == cudaSuccess && nch) e = launch_parse_text(p, parse_sm_count(), st);
    unsigned long long h[10] = {0};
    unsigned long long last[2] = {0, 0};
    if (e == cudaSuccess) e = cudaMemcpyAsync(h, res, sizeof(h), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess && nch) e = cudaMemcpyAsync(&last[0], p.st_lines + nch - 1, 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess && nch && !p.packed)
        e = cudaMemcpyAsync(&last[1], p.st_valid + nch - 1, 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return parse_fail(SINET_E_CUDA, std::string("parse_text: ") + cudaGetErrorString(e));
    const unsigned long long mask = (1ull << 62) - 1;
    if (p.packed) {                         // the last chunk's inclusive prefix: lines << 31 | valid
        result->lines = (last[0] & mask) >> 31;
        result->valid = last[0] & ((1ull << 31) - 1);
    } else {
        result->lines = last[0] & mask;
        result->valid = last[1] & mask;
    }
    result->first_bad_line = h[2];
    for (int k = 0; k < 7; ++k) result->by_status[k] = h[3 + k];
    if (result->valid > out->capacity)
        return parse_fail(SINET_E_RANGE, "parse_text: more valid lines than out.capacity");
    return SINET_OK;
}
