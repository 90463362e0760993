// Host-visible launchers of the sinet kernels.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "sinet_params.h"

namespace sinet {

cudaError_t launch_materialize(unsigned long long* bins, uint32_t* flags, uint32_t n_tiles,
                               uint32_t init_word, int grid, cudaStream_t st);
cudaError_t launch_materialize_range(unsigned long long* bins, uint32_t* flags, uint32_t t_lo, uint32_t t_hi,
                                     uint32_t init_word, int grid, cudaStream_t st);

// AUTO order probe: kProbeRuns evenly spaced runs of kProbeRun consecutive capture times
constexpr uint32_t kProbeRuns = 64, kProbeRun = 32;
cudaError_t launch_probe_gather(const uint64_t* ts, uint64_t n, uint64_t* out, cudaStream_t st);

cudaError_t setup_hist_atomic();
int hist_atomic_blocks_per_sm(const KernelParams& p);
cudaError_t launch_hist_atomic(const KernelParams& p, int grid, cudaStream_t st);

cudaError_t setup_hist_stream();
cudaError_t setup_hist_ws();
cudaError_t launch_hist_ws(const KernelParams& p, int sm_count, cudaStream_t st);
bool hist_ws_fits(int tab, uint32_t nbnd, uint32_t n_mixed);
cudaError_t launch_hist_stream(const KernelParams& p, int sm_count, bool agg, cudaStream_t st);
constexpr uint32_t kStreamWindowBins = 4096;   // smallest ring of the stream kernel (AUTO probe threshold)

cudaError_t launch_rebin(const unsigned long long* bins, uint64_t lo, uint64_t hi, uint64_t factor,
                         unsigned long long* out, uint64_t n_out, int sm_count, cudaStream_t st);
uint32_t sparse_blocks(uint64_t nbins);
cudaError_t launch_sparse(const unsigned long long* bins, uint64_t lo, uint64_t hi, uint32_t dir, uint32_t* scratch,
                          unsigned long long* d_total, uint64_t start, uint32_t width, unsigned long long* o_ts,
                          unsigned long long* o_cnt, unsigned long long* o_bytes, uint64_t capacity,
                          cudaStream_t st);

// unordered input: partition by time, then bin (sinet_partition.cu)
constexpr uint32_t kMaxFine = 16384;     // fine buckets of 8192 bins: windows of up to 2^27 bins
constexpr uint32_t kMaxCoarse = 128;
struct PartLayout {
    uint64_t cap;                        // records per sub-batch
    uint32_t nf, nc;                     // fine / coarse buckets of the window
    size_t by_a, by_b, key_a, key_b, fine_cnt, fine_base, fine_cur, unit_base, coarse_base, coarse_cur,
        cunit_base, counters, total;     // byte offsets in the scratch buffer, total size
};
PartLayout part_layout(uint64_t cap, uint32_t nbins);
bool partition_supported(uint32_t nbins);
cudaError_t setup_partition();
cudaError_t launch_partitioned(const KernelParams& p, void* scratch, const PartLayout& L, int sm_count,
                               cudaStream_t st, int* launches);

size_t sortreduce_scratch_bytes(uint64_t n, uint64_t nbins);
cudaError_t launch_sortreduce(const KernelParams& p, void* scratch, size_t scratch_bytes, int sm_count,
                              cudaStream_t st, int* launches);

}  // namespace sinet
