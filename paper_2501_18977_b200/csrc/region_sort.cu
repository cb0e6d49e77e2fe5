// Region-ordered relaxed inserts for multi-choice filters (c >= 2).
//
// A relaxed insert (atomic OR, bounded keys in flight) reads the c candidate
// blocks of every key and ORs its mask into one of them.  With the keys in
// stream order every one of those accesses is a random DRAM access, and the
// DRAM rate of random 64-byte accesses (~33 G/s on B200, activation-bound,
// tools/gather_probe.cu) bounds the insert.
//
// Relaxed mode does not promise stream order, so the keys of a batch are
// first bucketed by the region (kRegionBlocks consecutive blocks) of their
// first candidate.  Processed in that order, the first-candidate reads and the
// write-backs of blocks chosen there are served by L2 while a region is being
// worked on; only the remaining candidates stay random.  One counting-sort
// pass (count, scan, scatter with shared-memory staging so every bucket run
// is written contiguously) costs ~24 B of streaming traffic per key.
#include <algorithm>

#include "blocks.cuh"

namespace bc {

constexpr int kSortThreads = 512;
constexpr int kSortPerThread = 8;
constexpr int kSortChunk = kSortThreads * kSortPerThread;  // keys per CTA pass
constexpr int kMaxBuckets = 1024;

__device__ __forceinline__ u32 bucket_of(const KParams &p, u64 x, u32 shift) {
    return (u32)(block_index(p, x, 0) >> shift);
}

__global__ void __launch_bounds__(kSortThreads) bucket_count_kernel(
    const __grid_constant__ KParams p, const u64 *__restrict__ keys, u64 n, u32 shift, u32 nb,
    unsigned long long *__restrict__ counts) {
    __shared__ u32 hist[kMaxBuckets];
    for (u32 b = threadIdx.x; b < nb; b += kSortThreads) hist[b] = 0;
    __syncthreads();
    const u64 stride = (u64)gridDim.x * kSortThreads;
    for (u64 i = blockIdx.x * (u64)kSortThreads + threadIdx.x; i < n; i += stride)
        atomicAdd(&hist[bucket_of(p, ld_stream(keys + i), shift)], 1u);
    __syncthreads();
    for (u32 b = threadIdx.x; b < nb; b += kSortThreads)
        if (hist[b]) atomicAdd(counts + b, (unsigned long long)hist[b]);
}

// Each CTA pass: counting sort of kSortChunk keys in shared memory, then one
// global atomic per non-empty bucket reserves the chunk's run in the output.
__global__ void __launch_bounds__(kSortThreads) bucket_scatter_kernel(
    const __grid_constant__ KParams p, const u64 *__restrict__ keys, u64 n, u32 shift, u32 nb,
    unsigned long long *__restrict__ cursor, u64 *__restrict__ out) {
    extern __shared__ u64 stage[];  // kSortChunk keys
    __shared__ u32 hist[kMaxBuckets], loff[kMaxBuckets], warp_tot[kSortThreads / 32];
    __shared__ unsigned long long gbase[kMaxBuckets];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const u64 nchunks = (n + kSortChunk - 1) / kSortChunk;
    for (u64 ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
        for (u32 b = tid; b < nb; b += kSortThreads) hist[b] = 0;
        __syncthreads();
        const u64 base = ch * kSortChunk;
        const u32 cnt = (u32)min((u64)kSortChunk, n - base);
        u64 x[kSortPerThread];
        u32 bk[kSortPerThread], rk[kSortPerThread];
#pragma unroll
        for (int j = 0; j < kSortPerThread; ++j) {
            const u32 i = (u32)j * kSortThreads + tid;
            if (i < cnt) {
                x[j] = ld_stream(keys + base + i);
                bk[j] = bucket_of(p, x[j], shift);
                rk[j] = atomicAdd(&hist[bk[j]], 1u);
            } else {
                bk[j] = 0xffffffffu;
            }
        }
        __syncthreads();
        // exclusive scan of hist[0..nb) -> loff (nb <= 1024 = 2 per thread)
        const u32 b0 = 2 * tid, b1 = 2 * tid + 1;
        const u32 h0 = b0 < nb ? hist[b0] : 0u, h1 = b1 < nb ? hist[b1] : 0u;
        u32 incl = h0 + h1;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const u32 t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        if (lane == 31) warp_tot[warp] = incl;
        __syncthreads();
        u32 before = 0;
        for (int w = 0; w < warp; ++w) before += warp_tot[w];
        const u32 ex = before + incl - h0 - h1;
        if (b0 < nb) loff[b0] = ex;
        if (b1 < nb) loff[b1] = ex + h0;
        // reserve each bucket's run in the global output
        if (b0 < nb && h0) gbase[b0] = atomicAdd(cursor + b0, (unsigned long long)h0);
        if (b1 < nb && h1) gbase[b1] = atomicAdd(cursor + b1, (unsigned long long)h1);
        __syncthreads();
#pragma unroll
        for (int j = 0; j < kSortPerThread; ++j)
            if (bk[j] != 0xffffffffu) stage[loff[bk[j]] + rk[j]] = x[j];
        __syncthreads();
        // bucket runs are contiguous in stage[] and in out[]
        for (u32 i = tid; i < cnt; i += kSortThreads) {
            const u64 v = stage[i];
            const u32 b = bucket_of(p, v, shift);
            out[gbase[b] + (i - loff[b])] = v;
        }
        __syncthreads();
    }
}

u32 region_sort_buckets(const KParams &p, u32 shift) {
    return (u32)((p.num_blocks + (1ull << shift) - 1) >> shift);
}

// keys -> out (same n), bucketed by region of the first candidate.
// scratch: 2 * nb u64 counters
cudaError_t launch_region_sort(const KParams &p, const u64 *keys, u64 n, u32 shift, u64 *out,
                               unsigned long long *scratch, cudaStream_t s) {
    const u32 nb = region_sort_buckets(p, shift);
    if (nb > kMaxBuckets) return cudaErrorInvalidValue;
    unsigned long long *counts = scratch, *cursor = scratch + nb;
    cudaError_t e = cudaMemsetAsync(counts, 0, sizeof(u64) * nb, s);
    if (e != cudaSuccess) return e;
    const unsigned g0 = grid_for((const void *)bucket_count_kernel, kSortThreads, 0,
                                 (n + kSortChunk - 1) / kSortChunk);
    bucket_count_kernel<<<g0, kSortThreads, 0, s>>>(p, keys, n, shift, nb, counts);
    e = launch_scan(reinterpret_cast<u64 *>(counts), nb, nullptr, s);
    if (e != cudaSuccess) return e;
    e = cudaMemcpyAsync(cursor, counts, sizeof(u64) * nb, cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return e;
    const size_t smem = sizeof(u64) * kSortChunk;
    cudaFuncSetAttribute(bucket_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    const unsigned g1 = grid_for((const void *)bucket_scatter_kernel, kSortThreads, smem,
                                 (n + kSortChunk - 1) / kSortChunk);
    bucket_scatter_kernel<<<g1, kSortThreads, smem, s>>>(p, keys, n, shift, nb, cursor, out);
    count_launch(2);
    return cudaGetLastError();
}

}  // namespace bc
