// DRAM locality probe: how fast are random 64-byte block gathers from an
// 8 GiB array when the accesses in flight at any moment are confined to a
// small region of the array (what bucketing a lookup batch by filter region
// would give), against the fully random pattern of the lookup kernel?
//
// Lookup i reads block  region(i) * R + h(i) % R,  region(i) = (i / P) % NR,
// where R = blocks per region and P = lookups per region visit; with a
// grid-stride loop in index order the GPU's in-flight lookups then span one
// or two regions.  R = all blocks is the fully random pattern.  Four lanes
// per block (LDG.128 each, .L2::64B), one key read and one byte written per
// lookup, as in tools/gather_probe.cu.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o locality_probe tools/locality_probe.cu
//   ./locality_probe [filter GiB] [lookups log2]
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

typedef unsigned long long u64;

__device__ __forceinline__ u64 mix(u64 z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ uint4 ld64(const uint4 *p) {
    uint4 r;
    asm volatile("ld.global.cg.L2::64B.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

// R, NR, P powers of two (masks and shifts: no runtime 64-bit division, which
// would make the probe instruction-bound)
template <int UNR>
__global__ void __launch_bounds__(256) gather(const uint4 *__restrict__ blocks, u64 R, u64 NR,
                                              int lgP, const u64 *__restrict__ keys, u64 n,
                                              unsigned char *__restrict__ out) {
    const int s = threadIdx.x & 3;
    const u64 g0 = (blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 2;
    const u64 groups = ((u64)gridDim.x * blockDim.x) >> 2;
    for (u64 base = g0; base < n; base += groups * UNR) {
        uint4 w[UNR];
        u64 x[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const u64 i = base + u * groups;
            x[u] = i < n ? __ldcs(keys + i) : 0;
            const u64 region = (i >> lgP) & (NR - 1);
            const u64 b = region * R + (mix(i ^ x[u]) & (R - 1));
            w[u] = i < n ? ld64(blocks + b * 4 + s) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const u64 i = base + u * groups;
            unsigned v = w[u].x ^ w[u].y ^ w[u].z ^ w[u].w;
            v ^= __shfl_xor_sync(0xffffffffu, v, 1);
            v ^= __shfl_xor_sync(0xffffffffu, v, 2);
            if (s == 0 && i < n) out[i] = (unsigned char)(v & 1);
        }
    }
}

int main(int argc, char **argv) {
    const u64 gib = argc > 1 ? strtoull(argv[1], nullptr, 10) : 8;
    const int lg = argc > 2 ? atoi(argv[2]) : 28;
    const u64 bytes = gib << 30, nblocks = bytes / 64, n = 1ull << lg;
    uint4 *blocks;
    u64 *keys;
    unsigned char *out;
    cudaMalloc(&blocks, bytes);
    cudaMalloc(&keys, n * 8);
    cudaMalloc(&out, n);
    cudaMemset(blocks, 0x5a, bytes);
    cudaMemset(keys, 0x33, n * 8);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, gather<4>, 256, 0);
    const unsigned grid = per * sms;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    printf("array %llu GiB, %llu lookups, grid %u x 256\n", gib, n, grid);
    printf("%12s %12s %10s %12s\n", "region", "P", "ms", "G access/s");
    const u64 regions_bytes[] = {64ull << 10, 256ull << 10, 1ull << 20, 2ull << 20, 8ull << 20,
                                 32ull << 20, 128ull << 20, 1ull << 30, bytes};
    const int lgPs[] = {12, 15, 18};
    for (u64 rb : regions_bytes) {
        for (int lgP : lgPs) {
            const u64 R = rb / 64, NR = nblocks / R, P = 1ull << lgP;
            gather<4><<<grid, 256>>>(blocks, R, NR, lgP, keys, n, out);
            cudaEventRecord(e0);
            for (int it = 0; it < 3; ++it)
                gather<4><<<grid, 256>>>(blocks, R, NR, lgP, keys, n, out);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            ms /= 3;
            printf("%10llu KB %12llu %10.3f %12.2f\n", rb >> 10, P, ms, n / (ms * 1e-3) / 1e9);
            if (rb == bytes) break;
        }
    }
    cudaError_t err = cudaGetLastError();
    printf("status: %s\n", cudaGetErrorString(err));
    return 0;
}
