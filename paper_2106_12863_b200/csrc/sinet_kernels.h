// Host-visible launchers of the sinet kernels.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "sinet_params.h"

namespace sinet {

cudaError_t launch_materialize(unsigned long long* bins, uint32_t* flags, uint32_t n_tiles,
                               uint32_t init_word, int grid, cudaStream_t st);

size_t hist_atomic_smem(uint32_t nbnd);
cudaError_t setup_hist_atomic();
int hist_atomic_blocks_per_sm(uint32_t nbnd);
cudaError_t launch_hist_atomic(const KernelParams& p, int grid, cudaStream_t st);

cudaError_t setup_hist_stream();
cudaError_t launch_hist_stream(const KernelParams& p, int sm_count, bool agg, cudaStream_t st);
constexpr uint32_t kStreamWindowBins = 8192;

}  // namespace sinet
