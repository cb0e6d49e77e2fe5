// Region-partitioned insert for single-choice blocked filters (c == 1,
// 512-bit blocks, random strategy).
//
// Direct inserts OR each key's mask into its block with ~6.5 RED.64 into a
// random 64-byte block; past ~64 MiB the dirty lines do not stay in L2 and the
// scatter runs at the random-RED ceiling (tools/gather_probe.cu scatter:
// 37.6 G updates/s at 96 MiB).  Because OR commutes, the keys can be applied
// in any order -- so they are first bucketed by filter region (1024
// consecutive blocks = 64 KiB), and each region is then updated inside one
// CTA's shared memory (32-bit ATOMS.OR, ~6 lane-ops/clk/SM measured by
// tools/smem_atomic_probe.cu) and written back once with full-line stores.
// The result is bit-identical to the reference's stream-order build
// (_kernels.py:142-147: c == 1 is a plain OR).
//
//   region_count_kernel   CTA c histograms its contiguous key range into
//                         counts[r][c] (no global atomics)
//   region_prefix_kernel  per region: prefix over CTAs + region total
//   launch_scan           bucket starts = exclusive scan of the totals
//   region_scatter_kernel CTA c re-reads its range; a shared cursor per region
//                         (start + prefix) hands out bucket slots
//   region_apply_kernel   one CTA per region: load 64 KiB, OR every key's bits
//                         with shared-memory atomics, store 64 KiB
#include <algorithm>

#include "blocks.cuh"

namespace bc {

constexpr int kRegionShift = 10;                    // 1024 blocks per region
constexpr int kRegionBlocks = 1 << kRegionShift;
constexpr int kRegionWords32 = kRegionBlocks * 16;  // 64 KiB of u32
constexpr int kMaxRegions = 8192;                   // shared histogram bound
constexpr int kPartThreads = 512;

__device__ __forceinline__ u32 region_of(const KParams &p, u64 x) {
    return (u32)(block_index(p, x, 0) >> kRegionShift);
}

__device__ __forceinline__ void range_of(u64 n, u32 G, u32 c, u64 &lo, u64 &hi) {
    const u64 per = (n + G - 1) / G;
    lo = min(n, (u64)c * per);
    hi = min(n, lo + per);
}

__global__ void __launch_bounds__(kPartThreads) region_count_kernel(
    const __grid_constant__ KParams p, const u64 *__restrict__ keys, u64 n, u32 nreg,
    u32 *__restrict__ counts) {
    __shared__ u32 hist[kMaxRegions];
    for (u32 r = threadIdx.x; r < nreg; r += kPartThreads) hist[r] = 0;
    __syncthreads();
    u64 lo, hi;
    range_of(n, gridDim.x, blockIdx.x, lo, hi);
    for (u64 i = lo + threadIdx.x; i < hi; i += kPartThreads)
        atomicAdd(&hist[region_of(p, ld_stream(keys + i))], 1u);
    __syncthreads();
    for (u32 r = threadIdx.x; r < nreg; r += kPartThreads)
        counts[(u64)r * gridDim.x + blockIdx.x] = hist[r];
}

// counts[r][c] -> exclusive prefix over c in place; totals[r] = row sum
__global__ void __launch_bounds__(256) region_prefix_kernel(u32 *__restrict__ counts, u32 G,
                                                            u32 nreg,
                                                            u64 *__restrict__ totals) {
    const u32 r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= nreg) return;
    u32 *row = counts + (u64)r * G;
    u32 run = 0;
    for (u32 c = 0; c < G; ++c) {
        const u32 v = row[c];
        row[c] = run;
        run += v;
    }
    totals[r] = run;
}

__global__ void __launch_bounds__(kPartThreads) region_scatter_kernel(
    const __grid_constant__ KParams p, const u64 *__restrict__ keys, u64 n, u32 nreg,
    const u32 *__restrict__ prefix, const u64 *__restrict__ starts, u64 *__restrict__ buckets) {
    __shared__ u32 cur[kMaxRegions];
    for (u32 r = threadIdx.x; r < nreg; r += kPartThreads)
        cur[r] = (u32)starts[r] + prefix[(u64)r * gridDim.x + blockIdx.x];
    __syncthreads();
    u64 lo, hi;
    range_of(n, gridDim.x, blockIdx.x, lo, hi);
    for (u64 i = lo + threadIdx.x; i < hi; i += kPartThreads) {
        const u64 x = ld_stream(keys + i);
        buckets[atomicAdd(&cur[region_of(p, x)], 1u)] = x;
    }
}

__global__ void __launch_bounds__(kPartThreads) region_apply_kernel(
    const __grid_constant__ KParams p, u64 *__restrict__ words,
    const u64 *__restrict__ buckets, const u64 *__restrict__ starts, u32 nreg, u64 n) {
    extern __shared__ uint4 slab4[];
    u32 *slab = reinterpret_cast<u32 *>(slab4);
    for (u32 r = blockIdx.x; r < nreg; r += gridDim.x) {
        const u64 blk0 = (u64)r << kRegionShift;
        const u32 nblk = (u32)min((u64)kRegionBlocks, p.num_blocks - blk0);
        uint4 *g4 = reinterpret_cast<uint4 *>(words) + blk0 * 4;
        for (u32 i = threadIdx.x; i < nblk * 4; i += kPartThreads) slab4[i] = ld_block_cg(g4 + i);
        __syncthreads();
        const u64 lo = starts[r], hi = r + 1 < nreg ? starts[r + 1] : n;
        for (u64 i = lo + threadIdx.x; i < hi; i += kPartThreads) {
            const u64 x = __ldcs(buckets + i);
            u32 *blk = slab + (u32)(block_index(p, x, 0) - blk0) * 16;
            const u32 xlo = (u32)x, xhi = (u32)(x >> 32);
#pragma unroll 4
            for (u32 b = 0; b < p.k; ++b) {
                const u32 h = bit512(p.bit_a_lo[b], p.bit_a_hi[b], xlo, xhi);
                atomicOr(blk + (h >> 5), 1u << (h & 31));
            }
        }
        __syncthreads();
        for (u32 i = threadIdx.x; i < nblk * 4; i += kPartThreads) g4[i] = slab4[i];
        __syncthreads();
    }
}

u32 partition_regions(const KParams &p) {
    return (u32)((p.num_blocks + kRegionBlocks - 1) >> kRegionShift);
}

bool partition_supported(const KParams &p) {
    return p.c == 1 && p.wpb == 8 && p.fast_random && partition_regions(p) <= kMaxRegions;
}

static u32 partition_ctas(u64 n) {
    // enough CTAs to fill the GPU, each with a contiguous range of >= 4096 keys
    const unsigned cap = grid_for((const void *)region_scatter_kernel, kPartThreads, 0, 1u << 30);
    const u64 want = (n + 4095) / 4096;
    return (u32)std::max<u64>(1, std::min<u64>(cap, want));
}

size_t partition_scratch_bytes(const KParams &p, u64 n) {
    const u64 nreg = partition_regions(p);
    return sizeof(u64) * (n + 2 * nreg) + sizeof(u32) * nreg * partition_ctas(n);
}

// scratch layout: buckets[n] u64 | totals[nreg] u64 | spare[nreg] u64 | counts[nreg][G] u32
cudaError_t launch_partitioned_insert(const KParams &p, u64 *words, const u64 *keys, u64 n,
                                      void *scratch, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const u32 nreg = partition_regions(p);
    const u32 G = partition_ctas(n);
    u64 *buckets = reinterpret_cast<u64 *>(scratch);
    u64 *starts = buckets + n;
    u32 *counts = reinterpret_cast<u32 *>(starts + 2 * (u64)nreg);
    region_count_kernel<<<G, kPartThreads, 0, s>>>(p, keys, n, nreg, counts);
    region_prefix_kernel<<<(nreg + 255) / 256, 256, 0, s>>>(counts, G, nreg, starts);
    cudaError_t e = launch_scan(starts, nreg, nullptr, s);
    if (e != cudaSuccess) return e;
    region_scatter_kernel<<<G, kPartThreads, 0, s>>>(p, keys, n, nreg, counts, starts, buckets);
    const size_t smem = sizeof(u32) * kRegionWords32;
    cudaFuncSetAttribute(region_apply_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    const unsigned g2 = grid_for((const void *)region_apply_kernel, kPartThreads, smem, nreg);
    region_apply_kernel<<<g2, kPartThreads, smem, s>>>(p, words, buckets, starts, nreg, n);
    count_launch(4);
    return cudaGetLastError();
}

}  // namespace bc
