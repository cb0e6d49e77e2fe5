// Random 64-byte-block gather microbenchmark: the practical ceiling for the
// lookup kernel (SURVEY §8(d) "random-64B-gather microbenchmark").
//
// Four lanes read one 64-byte block (one LDG.128 each), blocks chosen by a
// splitmix hash of the lookup index, one 8-byte key streamed per lookup,
// one byte written per lookup -- the lookup kernel's memory pattern without
// its hashing.  Variants: cache-hint of the block load and the device L2
// fetch granularity.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o gather_probe tools/gather_probe.cu
//   ./gather_probe <filter MiB> <lookups log2>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstdint>

typedef unsigned long long u64;

// PROBE_PERSIST=1: launches go to a stream whose access-policy window marks
// the filter array L2-persisting (as libbbchoc does for filters that fit L2)
static cudaStream_t g_stream = nullptr;

static void maybe_persist(const void *base, size_t bytes) {
    const char *e = getenv("PROBE_PERSIST");
    if (!e || atoi(e) == 0) return;
    int maxp = 0, maxw = 0;
    cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, 0);
    cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, 0);
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, maxp);
    cudaStreamCreate(&g_stream);
    cudaStreamAttrValue v{};
    v.accessPolicyWindow.base_ptr = const_cast<void *>(base);
    v.accessPolicyWindow.num_bytes = bytes < (size_t)maxw ? bytes : (size_t)maxw;
    v.accessPolicyWindow.hitRatio = bytes <= (size_t)maxp ? 1.0f : (float)maxp / (float)bytes;
    v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    v.accessPolicyWindow.missProp = cudaAccessPropertyNormal;
    cudaStreamSetAttribute(g_stream, cudaStreamAttributeAccessPolicyWindow, &v);
    printf("persisting L2: max %d B, window %zu B, hit ratio %.3f\n", maxp,
           (size_t)v.accessPolicyWindow.num_bytes, v.accessPolicyWindow.hitRatio);
}

__device__ __forceinline__ u64 mix(u64 z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

template <int V>
__device__ __forceinline__ uint4 ld(const uint4 *p) {
    uint4 r;
    if (V == 0)
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    else if (V == 1)
        asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    else if (V == 2)
        asm volatile("ld.global.nc.L1::no_allocate.L2::64B.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    else if (V == 3)
        asm volatile("ld.global.nc.L1::no_allocate.L2::128B.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    else
        asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}

// UNR lookups in flight per 4-lane group
template <int V, int UNR>
__global__ void __launch_bounds__(256) gather(const uint4 *__restrict__ blocks, u64 nblocks,
                                              const u64 *__restrict__ keys, u64 n,
                                              unsigned char *__restrict__ out) {
    const int s = threadIdx.x & 3;
    const u64 g0 = (blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 2;
    const u64 groups = ((u64)gridDim.x * blockDim.x) >> 2;
    for (u64 base = g0; base < n; base += groups * UNR) {
        uint4 w[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const u64 i = base + u * groups;
            const u64 x = i < n ? __ldcs(keys + i) : 0;
            const u64 b = __umul64hi(mix(x), nblocks);
            w[u] = ld<V>(blocks + b * 4 + s);
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const u64 i = base + u * groups;
            const unsigned v = w[u].x ^ w[u].y ^ w[u].z ^ w[u].w;
            const unsigned all = __reduce_xor_sync(0xffffffffu, v);
            if (s == 0 && i < n) out[i] = (unsigned char)(all & 1);
        }
    }
}

template <int V, int UNR>
static float run(const uint4 *blocks, u64 nblocks, const u64 *keys, u64 n, unsigned char *out,
                 int reps) {
    int sms = 0, per = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, gather<V, UNR>, 256, 0);
    dim3 grid(sms * per);
    gather<V, UNR><<<grid, 256, 0, g_stream>>>(blocks, nblocks, keys, n, out);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, g_stream);
    for (int r = 0; r < reps; ++r) gather<V, UNR><<<grid, 256, 0, g_stream>>>(blocks, nblocks, keys, n, out);
    cudaEventRecord(b, g_stream);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return ms / reps;
}

__global__ void fill(u64 *p, u64 n) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
        p[i] = i * 0x9E3779B97F4A7C15ull;
}

extern "C" int scatter_main(u64 mib, int lg);

int main(int argc, char **argv) {
    if (argc > 1 && argv[1][0] == 's') return scatter_main(strtoull(argv[2], 0, 10), atoi(argv[3]));
    if (argc > 5 && argv[1][0] == 'g') {
        // single variant: g <MiB> <lookups log2> <variant 0..4> <L2 fetch granularity 0|32|64|128>
        const u64 mib = strtoull(argv[2], 0, 10), n = 1ull << atoi(argv[3]);
        const int v = atoi(argv[4]);
        const size_t gran = strtoull(argv[5], 0, 10);
        const u64 nb = mib * (1ull << 20) / 64;
        uint4 *blocks;
        u64 *keys;
        unsigned char *out;
        cudaMalloc(&blocks, nb * 64);
        cudaMalloc(&keys, n * 8);
        cudaMalloc(&out, n);
        fill<<<1184, 256>>>((u64 *)blocks, nb * 8);
        fill<<<1184, 256>>>(keys, n);
        if (gran) cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, gran);
        float ms = 0;
        switch (v) {
            case 0: ms = run<0, 2>(blocks, nb, keys, n, out, 1); break;
            case 1: ms = run<1, 2>(blocks, nb, keys, n, out, 1); break;
            case 2: ms = run<2, 2>(blocks, nb, keys, n, out, 1); break;
            case 3: ms = run<3, 2>(blocks, nb, keys, n, out, 1); break;
            default: ms = run<4, 2>(blocks, nb, keys, n, out, 1); break;
        }
        size_t g = 0;
        cudaDeviceGetLimit(&g, cudaLimitMaxL2FetchGranularity);
        printf("variant %d gran %zu: %.3f ms, %.1f G lookups/s\n", v, g, ms, n / ms / 1e6);
        return 0;
    }
    const u64 mib = argc > 1 ? strtoull(argv[1], 0, 10) : 512;
    const int lg = argc > 2 ? atoi(argv[2]) : 27;
    const int only = argc > 3 ? atoi(argv[3]) : -1;
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
    maybe_persist(blocks, nblocks * 64);
    const double bytes = (double)n * (64 + 8 + 1);
    const char *names[] = {"nc.L1::no_allocate", "cg", "nc.na.L2::64B", "nc.na.L2::128B",
                           "nc.na.L2::256B"};
    for (size_t gran : {0, 32, 64, 128}) {
        if (gran) cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, gran);
        size_t g = 0;
        cudaDeviceGetLimit(&g, cudaLimitMaxL2FetchGranularity);
        for (int v = 0; v < 5; ++v) {
            if (only >= 0 && v != only) continue;
            float ms1 = 0, ms2 = 0, ms4 = 0;
            switch (v) {
                case 0: ms1 = run<0, 1>(blocks, nblocks, keys, n, out, 5); ms2 = run<0, 2>(blocks, nblocks, keys, n, out, 5); ms4 = run<0, 4>(blocks, nblocks, keys, n, out, 5); break;
                case 1: ms1 = run<1, 1>(blocks, nblocks, keys, n, out, 5); ms2 = run<1, 2>(blocks, nblocks, keys, n, out, 5); ms4 = run<1, 4>(blocks, nblocks, keys, n, out, 5); break;
                case 2: ms1 = run<2, 1>(blocks, nblocks, keys, n, out, 5); ms2 = run<2, 2>(blocks, nblocks, keys, n, out, 5); ms4 = run<2, 4>(blocks, nblocks, keys, n, out, 5); break;
                case 3: ms1 = run<3, 1>(blocks, nblocks, keys, n, out, 5); ms2 = run<3, 2>(blocks, nblocks, keys, n, out, 5); ms4 = run<3, 4>(blocks, nblocks, keys, n, out, 5); break;
                case 4: ms1 = run<4, 1>(blocks, nblocks, keys, n, out, 5); ms2 = run<4, 2>(blocks, nblocks, keys, n, out, 5); ms4 = run<4, 4>(blocks, nblocks, keys, n, out, 5); break;
            }
            printf("filter %llu MiB  lookups 2^%d  gran %zu  %-20s  unr1 %.3f ms %.0f GB/s %.1f Gl/s | unr2 %.0f GB/s | unr4 %.0f GB/s\n",
                   mib, lg, g, names[v], ms1, bytes / ms1 / 1e6, n / ms1 / 1e6, bytes / ms2 / 1e6,
                   bytes / ms4 / 1e6);
        }
    }
    cudaError_t e = cudaGetLastError();
    printf("status: %s\n", cudaGetErrorString(e));
    return e != cudaSuccess;
}

// ---- insert-side probe: random 64-byte-block OR updates ---------------------------
// mode 0: 4 lanes x 2 RED.E.OR.64 per block; mode 1: plain ST.64 (racy, for
// the write-back comparison only); mode 2: atom.or (returning)
template <int MODE>
__global__ void __launch_bounds__(256) scatter(u64 *__restrict__ words, u64 nblocks,
                                               const u64 *__restrict__ keys, u64 n) {
    const int s = threadIdx.x & 3;
    const u64 g0 = (blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 2;
    const u64 groups = ((u64)gridDim.x * blockDim.x) >> 2;
    for (u64 i = g0; i < n; i += groups) {
        const u64 x = __ldcs(keys + i);
        const u64 b = __umul64hi(mix(x), nblocks);
        u64 *p = words + b * 8 + 2 * s;
        const u64 v = mix(x + s) & mix(x ^ s);
        if (MODE == 0) {
            atomicOr((unsigned long long *)p, v);
            atomicOr((unsigned long long *)p + 1, v >> 1);
        } else if (MODE == 1) {
            p[0] = v;
            p[1] = v >> 1;
        } else if (MODE == 2) {
            asm volatile("red.global.relaxed.gpu.or.b64 [%0], %1;" ::"l"(p), "l"(v));
            asm volatile("red.global.relaxed.gpu.or.b64 [%0], %1;" ::"l"(p + 1), "l"(v >> 1));
        } else if (MODE == 6) {
            // 4 lanes x 2 RED.64, each instruction on one 32-byte sector
            u64 *q = words + b * 8 + s;
            atomicOr((unsigned long long *)q, v);
            atomicOr((unsigned long long *)(q + 4), v >> 1);
        } else if (MODE == 5) {
            // 8 lanes per key, one RED.64 per word: the whole 64-byte block in
            // one instruction (keys of lanes 8h..8h+7 share the group's key)
            const u64 xk = __shfl_sync(0xffffffffu, x, threadIdx.x & 24);
            const u64 bk = __umul64hi(mix(xk), nblocks);
            atomicOr((unsigned long long *)(words + bk * 8 + (threadIdx.x & 7)), mix(xk + s));
        } else if (MODE == 3) {
            // 8 lanes per block, one RED.64 each (same block = 2 sectors per 4 lanes)
            u64 *q = words + b * 8 + (threadIdx.x & 7);
            atomicOr((unsigned long long *)q, v);
        } else {
            // 4 lanes per block, one 32-byte sector pair... each lane 1 RED.64 at word 2s
            atomicOr((unsigned long long *)p, v);
        }
    }
}

// mode 7: per key, one bulk OR-reduction (TMA, cp.reduce.async.bulk .or.b64) of
// a 64-byte mask staged in shared memory; double-buffered per warp
__global__ void __launch_bounds__(256) scatter_bulk(u64 *__restrict__ words, u64 nblocks,
                                                    const u64 *__restrict__ keys, u64 n) {
    __shared__ __align__(128) u64 stage[8][2][32][8];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const u64 nw = (u64)gridDim.x * 8;
    int buf = 0;
    for (u64 t = blockIdx.x * 8ull + warp; t * 32 < n; t += nw) {
        const u64 i = t * 32 + lane;
        // the copies that read this buffer two tiles ago must be done
        asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        __syncwarp();
        u64 *row = stage[warp][buf][lane];
        const u64 x = i < n ? __ldcs(keys + i) : 0;
#pragma unroll
        for (int w = 0; w < 8; ++w) row[w] = mix(x + w) & mix(x ^ w) & mix(x * 3 + w);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (i < n) {
            const u64 b = __umul64hi(mix(x), nblocks);
            const unsigned src = (unsigned)__cvta_generic_to_shared(row);
            asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.or.b64 [%0], [%1], 64;"
                         ::"l"(words + b * 8), "r"(src) : "memory");
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        buf ^= 1;
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

extern "C" int scatter_main(u64 mib, int lg) {
    const u64 nblocks = mib * (1ull << 20) / 64, n = 1ull << lg;
    u64 *words, *keys;
    cudaMalloc(&words, nblocks * 64);
    cudaMalloc(&keys, n * 8);
    fill<<<1184, 256>>>(keys, n);
    cudaMemset(words, 0, nblocks * 64);
    cudaDeviceSynchronize();
    maybe_persist(words, nblocks * 64);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int mode = 0; mode < 8; ++mode) {
        for (int rep = 0; rep < 3; ++rep) {
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            cudaEventRecord(a, g_stream);
            if (mode == 0) scatter<0><<<sms * 8, 256, 0, g_stream>>>(words, nblocks, keys, n);
            if (mode == 1) scatter<1><<<sms * 8, 256, 0, g_stream>>>(words, nblocks, keys, n);
            if (mode == 2) scatter<2><<<sms * 8, 256, 0, g_stream>>>(words, nblocks, keys, n);
            if (mode == 3) scatter<3><<<sms * 8, 256, 0, g_stream>>>(words, nblocks, keys, n);
            if (mode == 4) scatter<4><<<sms * 8, 256, 0, g_stream>>>(words, nblocks, keys, n);
            if (mode == 5) scatter<5><<<sms * 8, 256, 0, g_stream>>>(words, nblocks, keys, n);
            if (mode == 6) scatter<6><<<sms * 8, 256, 0, g_stream>>>(words, nblocks, keys, n);
            if (mode == 7) scatter_bulk<<<sms * 4, 256, 0, g_stream>>>(words, nblocks, keys, n);
            cudaEventRecord(b, g_stream);
            cudaEventSynchronize(b);
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            if (rep == 2)
                printf("scatter filter %llu MiB  2^%d updates  mode %d  %.3f ms  %.1f G/s\n", mib, lg,
                       mode, ms, n / ms / 1e6);
        }
    }
    cudaFree(words);
    cudaFree(keys);
    return 0;
}
