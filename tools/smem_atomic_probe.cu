// Shared-memory OR-update throughput (random addresses within a CTA's slab):
// decides whether region-partitioned inserts (smem-resident sub-filters) pay.
#include <cuda_runtime.h>
#include <cstdio>
typedef unsigned long long u64;

__device__ __forceinline__ u64 mix(u64 z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

template <int MODE>
__global__ void __launch_bounds__(256) smem_or(int iters, unsigned *sink) {
    extern __shared__ unsigned slab[];  // 32768 u32 = 128 KB
    for (int i = threadIdx.x; i < 32768; i += 256) slab[i] = 0;
    __syncthreads();
    u64 st = mix(blockIdx.x * 256 + threadIdx.x);
    for (int it = 0; it < iters; ++it) {
        st = st * 6364136223846793005ull + 1442695040888963407ull;
        const unsigned r = (unsigned)(st >> 32);
        if (MODE == 0) {
            atomicOr(&slab[r & 32767], 1u << (r >> 27));
        } else if (MODE == 1) {
            atomicOr((unsigned long long *)&slab[(r & 16383) * 2], 1ull << (r >> 26));
        } else {  // plain RMW (racy): LDS + OR + STS
            unsigned *p = &slab[r & 32767];
            *p |= 1u << (r >> 27);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) sink[blockIdx.x] = slab[blockIdx.x & 32767];
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned *sink;
    cudaMalloc(&sink, 4096 * 4);
    const int iters = 4096;
    for (int mode = 0; mode < 3; ++mode) {
        auto k = mode == 0 ? smem_or<0> : mode == 1 ? smem_or<1> : smem_or<2>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
        k<<<sms, 256, 131072>>>(iters, sink);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        k<<<sms, 256, 131072>>>(iters, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        double ops = (double)sms * 256 * iters;
        printf("mode %d (%s): %.3f ms, %.2f lane-ops/clk/SM at 1.965 GHz, %.1f G ops/s\n", mode,
               mode == 0 ? "atomicOr u32" : mode == 1 ? "atomicOr u64" : "LDS+OR+STS racy", ms,
               ops / sms / (ms * 1e-3 * 1.965e9), ops / ms / 1e6);
    }
    printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
}
