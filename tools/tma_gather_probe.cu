// Block staging for the lookup kernels: cp.async (LDGSTS, four lanes x 16 B
// per 64-byte block, what lookup.cuh does) against Blackwell's TMA gather
// (cp.async.bulk.tensor.2d ... tile::gather4: one elected lane stages four
// random 64-byte rows of a [M x 64 B] tensor map per instruction, completion
// on an mbarrier).  Each warp stages the blocks of 32 lookups per step into
// its shared-memory slice and every lane then reads its key's block (16
// words, XOR-folded into one output byte) -- the lookup kernel's memory
// pattern without its hashing.  Two stages per warp: step t+1's copies are in
// flight while step t is read.
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tma_gather_probe tools/tma_gather_probe.cu
//   ./tma_gather_probe <filter MiB> <lookups log2>      (PROBE_PERSIST=1: L2-persisting filter)
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

typedef unsigned long long u64;
typedef unsigned u32;

constexpr int kWarps = 8;

__device__ __forceinline__ u64 mix(u64 z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

struct __align__(128) Stage {
    uint4 rows[32][4];  // 32 blocks of 64 B
};

__device__ __forceinline__ u32 fold(const Stage &st, int lane) {
    u32 v = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const uint4 w = st.rows[lane][q];
        v ^= w.x ^ w.y ^ w.z ^ w.w;
    }
    return v;
}

// ---- variant 0: cp.async (LDGSTS), four lanes per block ---------------------------
__global__ void __launch_bounds__(256) stage_ldgsts(const uint4 *__restrict__ blocks, u64 nblocks,
                                                    const u64 *__restrict__ keys, u64 n,
                                                    unsigned char *__restrict__ out) {
    __shared__ Stage st[kWarps][2];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int g = lane >> 2, s = lane & 3;
    const u64 warp = blockIdx.x * (u64)kWarps + w, nwarps = (u64)gridDim.x * kWarps;
    auto issue = [&](u64 t, int buf) {
        const u64 i = t * 32 + lane;
        const u64 b = i < n ? __umul64hi(mix(__ldcs(keys + i)), nblocks) : 0;
#pragma unroll
        for (int pp = 0; pp < 4; ++pp) {
            const int kk = 4 * g + pp;
            const u64 bk = __shfl_sync(0xffffffffu, b, kk);
            const u32 dst = (u32)__cvta_generic_to_shared(&st[w][buf].rows[kk][s]);
            asm volatile("cp.async.cg.shared.global.L2::64B [%0], [%1], 16;" ::"r"(dst),
                         "l"(blocks + bk * 4 + s));
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    const u64 ntiles = (n + 31) / 32;
    u64 t = warp;
    int buf = 0;
    if (t < ntiles) issue(t, 0);
    for (; t < ntiles; t += nwarps) {
        if (t + nwarps < ntiles) {
            issue(t + nwarps, buf ^ 1);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncwarp();
        const u64 i = t * 32 + lane;
        const u32 v = fold(st[w][buf], lane);
        if (i < n) out[i] = (unsigned char)v;
        __syncwarp();
        buf ^= 1;
    }
}

// ---- variant 1: TMA gather4, one lane issues 8 instructions per 32 blocks ---------------
__device__ __forceinline__ void mbar_init(u64 *bar, u32 count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((u32)__cvta_generic_to_shared(bar)),
                 "r"(count));
}
__device__ __forceinline__ void mbar_expect(u64 *bar, u32 bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                     (u32)__cvta_generic_to_shared(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(u64 *bar, u32 parity) {
    const u32 a = (u32)__cvta_generic_to_shared(bar);
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}" ::"r"(a),
        "r"(parity)
        : "memory");
}

__global__ void __launch_bounds__(256) stage_tma(const __grid_constant__ CUtensorMap map,
                                                 u64 nblocks, const u64 *__restrict__ keys, u64 n,
                                                 unsigned char *__restrict__ out) {
    __shared__ Stage st[kWarps][2];
    __shared__ __align__(8) u64 bar[kWarps][2];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const u64 warp = blockIdx.x * (u64)kWarps + w, nwarps = (u64)gridDim.x * kWarps;
    if (lane == 0) {
        mbar_init(&bar[w][0], 1);
        mbar_init(&bar[w][1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    auto issue = [&](u64 t, int buf) {
        const u64 i = t * 32 + lane;
        const u32 b = i < n ? (u32)__umul64hi(mix(__ldcs(keys + i)), nblocks) : 0u;
        // generic-proxy reads of this buffer (two steps ago) before async-proxy writes
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_expect(&bar[w][buf], 32 * 64);
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const u32 r0 = __shfl_sync(0xffffffffu, b, 4 * r), r1 = __shfl_sync(0xffffffffu, b, 4 * r + 1);
            const u32 r2 = __shfl_sync(0xffffffffu, b, 4 * r + 2), r3 = __shfl_sync(0xffffffffu, b, 4 * r + 3);
            if (lane == 0) {
                const u32 dst = (u32)__cvta_generic_to_shared(&st[w][buf].rows[4 * r][0]);
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::"
                    "complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
                    "l"(&map), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3),
                    "r"((u32)__cvta_generic_to_shared(&bar[w][buf]))
                    : "memory");
            }
        }
    };
    const u64 ntiles = (n + 31) / 32;
    u32 phase[2] = {0, 0};
    u64 t = warp;
    int buf = 0;
    if (t < ntiles) issue(t, 0);
    for (; t < ntiles; t += nwarps) {
        if (t + nwarps < ntiles) issue(t + nwarps, buf ^ 1);
        mbar_wait(&bar[w][buf], phase[buf]);
        phase[buf] ^= 1u;
        const u64 i = t * 32 + lane;
        const u32 v = fold(st[w][buf], lane);
        if (i < n) out[i] = (unsigned char)v;
        __syncwarp();
        buf ^= 1;
    }
}

__global__ void fill(u64 *p, u64 n) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
        p[i] = i * 0x9E3779B97F4A7C15ull;
}

// the same answers from the host's view: fold of block b of the fill pattern
static unsigned char ref_answer(u64 key, u64 nblocks) {
    u64 z = key + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    const u64 b = (u64)(((unsigned __int128)z * nblocks) >> 64);
    u32 v = 0;
    for (int j = 0; j < 8; ++j) {
        const u64 word = (b * 8 + j) * 0x9E3779B97F4A7C15ull;
        v ^= (u32)word ^ (u32)(word >> 32);
    }
    return (unsigned char)v;
}

typedef CUresult (*EncodeTiled)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char **argv) {
    const u64 mib = argc > 1 ? strtoull(argv[1], 0, 10) : 96;
    const int lg = argc > 2 ? atoi(argv[2]) : 27;
    const u64 nblocks = mib * (1ull << 20) / 64, n = 1ull << lg;
    uint4 *blocks;
    u64 *keys;
    unsigned char *out;
    cudaMalloc(&blocks, nblocks * 64);
    cudaMalloc(&keys, n * 8);
    cudaMalloc(&out, n);
    fill<<<1184, 256>>>((u64 *)blocks, nblocks * 8);
    fill<<<1184, 256>>>(keys, n);
    cudaDeviceSynchronize();
    cudaStream_t s = nullptr;
    if (getenv("PROBE_PERSIST") && atoi(getenv("PROBE_PERSIST"))) {
        int maxp = 0, maxw = 0;
        cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, 0);
        cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, 0);
        cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, maxp);
        cudaStreamCreate(&s);
        cudaStreamAttrValue v{};
        const size_t bytes = nblocks * 64;
        v.accessPolicyWindow.base_ptr = blocks;
        v.accessPolicyWindow.num_bytes = bytes < (size_t)maxw ? bytes : (size_t)maxw;
        v.accessPolicyWindow.hitRatio = bytes <= (size_t)maxp ? 1.0f : (float)maxp / (float)bytes;
        v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        v.accessPolicyWindow.missProp = cudaAccessPropertyNormal;
        cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &v);
    }
    // [M x 16] u32 tensor, one 64-byte row per block; box = one row (gather4
    // takes four row coordinates per instruction)
    EncodeTiled encode = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&encode, cudaEnableDefault, &q) !=
            cudaSuccess ||
        !encode) {
        printf("no cuTensorMapEncodeTiled\n");
        return 1;
    }
    CUtensorMap map;
    const cuuint64_t dims[2] = {16, nblocks};
    const cuuint64_t strides[1] = {64};
    const cuuint32_t box[2] = {16, 1};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, blocks, dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        printf("cuTensorMapEncodeTiled failed: %d\n", (int)r);
        return 1;
    }
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned char *host = (unsigned char *)malloc(1 << 20);
    for (int variant = 0; variant < 2; ++variant) {
        int per = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &per, variant ? (const void *)stage_tma : (const void *)stage_ldgsts, 256, 0);
        const dim3 grid(sms * per);
        auto launch = [&]() {
            if (variant)
                stage_tma<<<grid, 256, 0, s>>>(map, nblocks, keys, n, out);
            else
                stage_ldgsts<<<grid, 256, 0, s>>>(blocks, nblocks, keys, n, out);
        };
        cudaMemset(out, 0, n);
        launch();
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("variant %d: %s\n", variant, cudaGetErrorString(e));
            return 1;
        }
        // check the first 2^20 answers against the host
        std::vector<u64> hk(1 << 20);
        cudaMemcpy(hk.data(), keys, 8 << 20, cudaMemcpyDeviceToHost);
        cudaMemcpy(host, out, 1 << 20, cudaMemcpyDeviceToHost);
        u64 bad = 0;
        for (int i = 0; i < (1 << 20) && (u64)i < n; ++i) bad += host[i] != ref_answer(hk[i], nblocks);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        const int reps = 5;
        cudaEventRecord(a, s);
        for (int k = 0; k < reps; ++k) launch();
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        ms /= reps;
        printf("filter %llu MiB  lookups 2^%d  %-8s  CTAs/SM %d  %.3f ms  %.1f G blocks/s  %.0f GB/s "
               "of blocks  mismatches %llu/%d\n",
               mib, lg, variant ? "tma-g4" : "ldgsts", per, ms, n / ms / 1e6, n * 64.0 / ms / 1e6,
               bad, 1 << 20);
    }
    return 0;
}
