// Micro-benchmarks that decide the accumulation design of the histogram
// kernel on B200: shared-memory atomics vs L2 reductions vs plain streams.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench tools/microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t hsh(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

template <int MODE>   // 0: ATOMS no-return, 1: ATOMS with return, 2: plain LDS+STS RMW, 3: ATOMS 64 (CAS loop)
__global__ void k_smem(uint32_t iters, uint32_t* sink) {
    extern __shared__ uint32_t s[];
    const uint32_t S = 24 * 1024;   // 96 KB of u32 slots
    for (uint32_t i = threadIdx.x; i < S; i += blockDim.x) s[i] = 0;
    __syncthreads();
    uint32_t acc = 0, x = hsh(blockIdx.x * 977 + threadIdx.x);
    for (uint32_t it = 0; it < iters; ++it) {
        x = x * 1664525u + 1013904223u;
        uint32_t idx = (x >> 8) % S;
        if (MODE == 0) atomicAdd(&s[idx], 1u);
        else if (MODE == 1) acc += atomicAdd(&s[idx], x);
        else if (MODE == 2) s[idx] += 1u;
        else atomicAdd(reinterpret_cast<unsigned long long*>(s) + (idx >> 1), 1ull);
    }
    __syncthreads();
    if (threadIdx.x == 0) sink[blockIdx.x] = s[blockIdx.x % S] + acc;
    if (MODE == 1 && acc == 0xFFFFFFFF) sink[0] = acc;
}

template <bool RET>
__global__ void k_redg(unsigned long long* g, uint64_t mask_elems, uint32_t iters, unsigned long long* sink) {
    uint32_t x = hsh(blockIdx.x * 1024 + threadIdx.x);
    unsigned long long acc = 0;
    for (uint32_t it = 0; it < iters; ++it) {
        x = x * 1664525u + 1013904223u;
        uint64_t idx = ((uint64_t)hsh(x) * 4u) & mask_elems;   // sector-strided like [bin][4]
        if (RET) acc += atomicAdd(g + idx, 1ull);
        else atomicAdd(g + idx, 1ull);
    }
    if (RET && acc == 7) sink[0] = acc;
}

// two REDG per "record" to adjacent words (count + bytes), stream-ordered addresses (local window)
__global__ void k_redg_local(unsigned long long* g, uint64_t n_bins, uint32_t iters) {
    uint64_t gt = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (uint64_t)gridDim.x * blockDim.x;
    uint32_t x = hsh((uint32_t)gt);
    for (uint32_t it = 0; it < iters; ++it) {
        uint64_t rec = gt + (uint64_t)it * nt;             // record index, time ordered
        x = x * 1664525u + 1013904223u;
        uint64_t bin = (rec * 864ull / 1000ull + (x >> 21)) % n_bins;   // ~1.16 records/bin + 2 s disorder
        atomicAdd(g + bin * 4, 1ull);
        atomicAdd(g + bin * 4 + 1, (unsigned long long)(x & 0xFFFF));
    }
}

__global__ void k_read(const ulonglong2* a, uint64_t n, unsigned long long* sink) {
    unsigned long long acc = 0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        ulonglong2 v = __ldcs(a + i);
        acc += v.x ^ v.y;
    }
    if (acc == 12345) sink[0] = acc;
}

__global__ void k_write(ulonglong2* a, uint64_t n) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        a[i] = make_ulonglong2(i, 0);
}

int main() {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    int clk = 0;
    CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
    printf("SMs %d, clock %d MHz\n", sms, clk / 1000);
    uint32_t* sink;
    CK(cudaMalloc(&sink, 1 << 20));
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    float ms;
    const int threads = 512, blocks = sms * 2;
    const uint32_t it = 4096;
    const double lane_ops = (double)blocks * threads * it;
#define SMEM(MODE, name)                                                                          \
    CK(cudaFuncSetAttribute(k_smem<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024)); \
    k_smem<MODE><<<blocks, threads, 96 * 1024>>>(16, sink);                                       \
    cudaEventRecord(a); k_smem<MODE><<<blocks, threads, 96 * 1024>>>(it, sink); cudaEventRecord(b); \
    CK(cudaEventSynchronize(b)); cudaEventElapsedTime(&ms, a, b);                                  \
    printf("%-28s %8.3f ms  %7.1f G lane-ops/s  %.3f lane-ops/clk/SM\n", name, ms, lane_ops / ms / 1e6, \
           lane_ops / (ms * 1e-3) / sms / (clk * 1e3));
    SMEM(0, "smem ATOMS.ADD no-ret");
    SMEM(1, "smem ATOMS.ADD with ret");
    SMEM(2, "smem LDS+STS (racy RMW)");
    SMEM(3, "smem atomicAdd u64 (CAS)");

    unsigned long long* g;
    const uint64_t big = 2764800000ull;   // ~2.76 GB like the day of bins
    CK(cudaMalloc(&g, big));
    CK(cudaMemset(g, 0, big));
    for (int ret = 0; ret < 2; ++ret) {
        for (uint64_t bytes : {64ull << 20, 2048ull << 20}) {
            uint64_t elems = bytes / 8, mask = elems - 1;
            const int rb = sms * 8, rt = 256;
            const uint32_t rit = 256;
            if (ret) k_redg<true><<<rb, rt>>>(g, mask, 8, (unsigned long long*)sink);
            else k_redg<false><<<rb, rt>>>(g, mask, 8, (unsigned long long*)sink);
            cudaEventRecord(a);
            if (ret) k_redg<true><<<rb, rt>>>(g, mask, rit, (unsigned long long*)sink);
            else k_redg<false><<<rb, rt>>>(g, mask, rit, (unsigned long long*)sink);
            cudaEventRecord(b);
            CK(cudaEventSynchronize(b));
            cudaEventElapsedTime(&ms, a, b);
            double ops = (double)rb * rt * rit;
            printf("REDG u64 %s random over %5llu MB  %8.3f ms  %7.2f G atom/s\n", ret ? "ATOMG" : "RED  ",
                   (unsigned long long)(bytes >> 20), ms, ops / ms / 1e6);
        }
    }
    {
        uint64_t n_bins = big / 32;
        const int rb = sms * 8, rt = 256;
        const uint32_t rit = 100000000ull / (rb * rt) + 1;
        cudaEventRecord(a);
        k_redg_local<<<rb, rt>>>(g, n_bins, rit);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        cudaEventElapsedTime(&ms, a, b);
        double recs = (double)rb * rt * rit;
        printf("REDG x2 stream-local 100M recs %8.3f ms  %7.2f G rec/s\n", ms, recs / ms / 1e6);
    }
    {
        uint64_t n = big / 16;
        k_read<<<sms * 8, 512>>>((ulonglong2*)g, n, (unsigned long long*)sink);
        cudaEventRecord(a);
        k_read<<<sms * 8, 512>>>((ulonglong2*)g, n, (unsigned long long*)sink);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        cudaEventElapsedTime(&ms, a, b);
        printf("stream read 2.76 GB        %8.3f ms  %7.1f GB/s\n", ms, big / ms / 1e6);
        cudaEventRecord(a);
        k_write<<<sms * 8, 512>>>((ulonglong2*)g, n);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        cudaEventElapsedTime(&ms, a, b);
        printf("stream write 2.76 GB       %8.3f ms  %7.1f GB/s\n", ms, big / ms / 1e6);
        cudaEventRecord(a);
        CK(cudaMemsetAsync(g, 0, big));
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        cudaEventElapsedTime(&ms, a, b);
        printf("cudaMemset 2.76 GB         %8.3f ms  %7.1f GB/s\n", ms, big / ms / 1e6);
    }
    return 0;
}
