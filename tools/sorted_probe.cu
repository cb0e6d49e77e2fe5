// Feasibility probe: region-sorted lookups for filters far above L2.
//
// Direct lookups on a 512 MiB - 8 GiB filter run at the random 64-byte DRAM
// access ceiling (gather_probe: 43 G/s at 512 MiB, 33 G/s at 8 GiB).  With
// batches far larger than the block count (cfg3: 128 lookups per block,
// cfg5 too), the same answers can come from streaming work instead:
//
//   count    every (key, choice) record -> region = block >> 10 (64 KiB)
//   scan     region starts
//   scatter  records (key, idx | choice << 30) appended per region
//   lookup   one CTA per region: 64 KiB slab in shared memory, test every
//            record's k bits there, OR hits into an answer bitmap
//   expand   bitmap -> u8 answers
//
// This probe times each stage and checks the answers against a direct
// lookup.  Synthetic hashes with the hot path's shapes (SHIFT block hash,
// 9-bit bit hashes of a*x).
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o sorted_probe tools/sorted_probe.cu
//   ./sorted_probe <filter MiB (power of 2)> <log2 keys> <c> <k>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

typedef unsigned long long u64;
typedef unsigned u32;

#define CK(x)                                                                       \
    do {                                                                            \
        cudaError_t e_ = (x);                                                       \
        if (e_ != cudaSuccess) {                                                    \
            printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
            exit(1);                                                                \
        }                                                                           \
    } while (0)

__host__ __device__ __forceinline__ u64 mix(u64 z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

struct P {
    u64 ba[4];
    u32 alo[16], ahi[16];
    u32 k, c, shift;  // block = (a*x) >> shift
    u64 M;
};

constexpr int kRegShift = 10;
constexpr int kRegBlocks = 1 << kRegShift;

__device__ __forceinline__ u64 blk(const P &p, u64 x, int j) { return (p.ba[j] * x) >> p.shift; }
__device__ __forceinline__ u32 hi32(u32 alo, u32 ahi, u32 xlo, u32 xhi) {
    return __umulhi(alo, xlo) + alo * xhi + ahi * xlo;
}
__device__ __forceinline__ bool test(const P &p, const u32 *w, u64 x) {
    const u32 xlo = (u32)x, xhi = (u32)(x >> 32);
    u32 acc = 1;
    for (u32 i = 0; i < p.k; ++i) {
        const u32 h = hi32(p.alo[i], p.ahi[i], xlo, xhi);
        const u32 v = w[h >> 28];
        acc &= __funnelshift_r(v, v, h >> 23);
    }
    return acc & 1;
}

__global__ void fill_words(u32 *w, u64 n) {
    // P(bit) = 15/16: with k = 11..16, 35-50% of (key, choice) tests hit
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        const u64 a = mix(i * 2 + 1), b = mix(i * 2 + 2);
        w[i] = ~((u32)a & (u32)(a >> 32) & (u32)b & (u32)(b >> 32));
    }
}

__global__ void fill_keys(u64 *k, u64 n, u64 seed) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
        k[i] = mix(i ^ seed);
}

// direct: one thread per key, choices in order, 64-byte block via 4 x 16 B
__global__ void direct_kernel(P p, const u32 *__restrict__ w, const u64 *__restrict__ keys, u64 n,
                              unsigned char *out) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        const u64 x = keys[i];
        bool f = false;
        for (u32 j = 0; j < p.c && !f; ++j) {
            const uint4 *b4 = reinterpret_cast<const uint4 *>(w + blk(p, x, j) * 16);
            u32 s[16];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                uint4 v = __ldcg(b4 + q);
                s[4 * q] = v.x; s[4 * q + 1] = v.y; s[4 * q + 2] = v.z; s[4 * q + 3] = v.w;
            }
            const u32 xlo = (u32)x, xhi = (u32)(x >> 32);
            u32 acc = 1;
            for (u32 t = 0; t < p.k; ++t) {
                const u32 h = hi32(p.alo[t], p.ahi[t], xlo, xhi);
                u32 v = 0;
#pragma unroll
                for (int q = 0; q < 16; ++q) v = (h >> 28) == (u32)q ? s[q] : v;
                acc &= __funnelshift_r(v, v, h >> 23);
            }
            f = acc & 1;
        }
        out[i] = f;
    }
}

// ---- count -------------------------------------------------------------------
template <bool SMEM>
__global__ void __launch_bounds__(512) count_kernel(P p, const u64 *__restrict__ keys, u64 n, u32 R,
                                                    u32 *__restrict__ ghist) {
    extern __shared__ u32 h[];
    if (SMEM) {
        for (u32 r = threadIdx.x; r < R; r += blockDim.x) h[r] = 0;
        __syncthreads();
    }
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        const u64 x = __ldcs(keys + i);
        for (u32 j = 0; j < p.c; ++j) {
            const u32 r = (u32)(blk(p, x, j) >> kRegShift);
            if (SMEM) atomicAdd(&h[r], 1u);
            else atomicAdd(&ghist[r], 1u);
        }
    }
    if (SMEM) {
        __syncthreads();
        for (u32 r = threadIdx.x; r < R; r += blockDim.x)
            if (h[r]) atomicAdd(&ghist[r], h[r]);
    }
}

// single-CTA exclusive scan; starts[R] = total
__global__ void scan_kernel(const u32 *hist, u32 R, u32 *starts, u32 *cur) {
    __shared__ u32 part[1024];
    const u32 per = (R + 1023) / 1024, lo = threadIdx.x * per, hi = min(R, lo + per);
    u32 s = 0;
    for (u32 r = lo; r < hi; ++r) s += hist[r];
    part[threadIdx.x] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        u32 run = 0;
        for (int t = 0; t < 1024; ++t) { u32 v = part[t]; part[t] = run; run += v; }
        starts[R] = run;
    }
    __syncthreads();
    u32 run = part[threadIdx.x];
    for (u32 r = lo; r < hi; ++r) { starts[r] = run; cur[r] = run; run += hist[r]; }
}

// ---- scatter ---------------------------------------------------------------------
// SMEM: tiles of T keys; per-tile counts -> one global atomic per nonempty
// region -> records written at base + rank.  Else: one global atomic per record.
template <bool SMEM>
__global__ void __launch_bounds__(512) scatter_kernel(P p, const u64 *__restrict__ keys, u64 n, u32 R,
                                                      u32 *__restrict__ cur, u64 *__restrict__ rkey,
                                                      u32 *__restrict__ rmeta, u32 T) {
    extern __shared__ u32 sm[];
    if (!SMEM) {
        for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
            const u64 x = __ldcs(keys + i);
            for (u32 j = 0; j < p.c; ++j) {
                const u32 r = (u32)(blk(p, x, j) >> kRegShift);
                const u32 pos = atomicAdd(&cur[r], 1u);
                rkey[pos] = x;
                rmeta[pos] = (u32)i | (j << 30);
            }
        }
        return;
    }
    u32 *cnt = sm, *base = sm + R;
    for (u32 r = threadIdx.x; r < R; r += blockDim.x) cnt[r] = 0;
    __syncthreads();
    for (u64 t0 = (u64)blockIdx.x * T; t0 < n; t0 += (u64)gridDim.x * T) {
        const u64 t1 = min(n, t0 + T);
        for (u64 i = t0 + threadIdx.x; i < t1; i += blockDim.x) {
            const u64 x = keys[i];
            for (u32 j = 0; j < p.c; ++j) atomicAdd(&cnt[(u32)(blk(p, x, j) >> kRegShift)], 1u);
        }
        __syncthreads();
        for (u32 r = threadIdx.x; r < R; r += blockDim.x) {
            const u32 c = cnt[r];
            if (c) base[r] = atomicAdd(&cur[r], c);
            cnt[r] = 0;
        }
        __syncthreads();
        for (u64 i = t0 + threadIdx.x; i < t1; i += blockDim.x) {
            const u64 x = __ldcs(keys + i);
            for (u32 j = 0; j < p.c; ++j) {
                const u32 r = (u32)(blk(p, x, j) >> kRegShift);
                const u32 pos = base[r] + atomicAdd(&cnt[r], 1u);
                rkey[pos] = x;
                rmeta[pos] = (u32)i | (j << 30);
            }
        }
        __syncthreads();
        for (u32 r = threadIdx.x; r < R; r += blockDim.x) cnt[r] = 0;
        __syncthreads();
    }
}

// ---- region lookup -------------------------------------------------------------
__global__ void __launch_bounds__(512) region_lookup_kernel(P p, const u32 *__restrict__ w, u32 R,
                                                            const u32 *__restrict__ starts,
                                                            const u64 *__restrict__ rkey,
                                                            const u32 *__restrict__ rmeta,
                                                            u32 *__restrict__ bitmap) {
    extern __shared__ uint4 slab4[];
    const u32 *slab = reinterpret_cast<const u32 *>(slab4);
    for (u32 r = blockIdx.x; r < R; r += gridDim.x) {
        const uint4 *g4 = reinterpret_cast<const uint4 *>(w) + (u64)r * kRegBlocks * 4;
        for (u32 i = threadIdx.x; i < kRegBlocks * 4; i += blockDim.x) slab4[i] = __ldcs(g4 + i);
        __syncthreads();
        const u32 lo = starts[r], hi = starts[r + 1];
        const u64 b0 = (u64)r << kRegShift;
        for (u32 i = lo + threadIdx.x; i < hi; i += blockDim.x) {
            const u64 x = __ldcs(rkey + i);
            const u32 m = __ldcs(rmeta + i);
            const u32 b = (u32)(blk(p, x, m >> 30) - b0);
            if (test(p, slab + b * 16, x)) atomicOr(bitmap + ((m & 0x3fffffffu) >> 5), 1u << (m & 31));
        }
        __syncthreads();
    }
}

__global__ void expand_kernel(const u32 *__restrict__ bitmap, u64 n, unsigned char *out) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
        out[i] = (bitmap[i >> 5] >> (i & 31)) & 1u;
}

int main(int argc, char **argv) {
    const u64 mib = argc > 1 ? strtoull(argv[1], 0, 10) : 512;
    const int lg = argc > 2 ? atoi(argv[2]) : 28;
    const u32 c = argc > 3 ? atoi(argv[3]) : 3, k = argc > 4 ? atoi(argv[4]) : 16;
    const u32 T = argc > 5 ? atoi(argv[5]) : 16384;
    const u64 n = 1ull << lg, M = mib << 14;  // 64 B blocks
    int lgM = 0;
    while ((1ull << lgM) < M) ++lgM;
    P p{};
    for (u32 j = 0; j < c; ++j) p.ba[j] = mix(100 + j) | 1;
    for (u32 i = 0; i < k; ++i) { u64 a = mix(200 + i) | 1; p.alo[i] = (u32)a; p.ahi[i] = (u32)(a >> 32); }
    p.k = k; p.c = c; p.shift = 64 - lgM; p.M = M;
    const u32 R = (u32)(M >> kRegShift);
    int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    u32 *w, *ghist, *starts, *cur, *rmeta, *bitmap; u64 *keys, *rkey; unsigned char *o1, *o2;
    CK(cudaMalloc(&w, M * 64)); CK(cudaMalloc(&keys, n * 8));
    CK(cudaMalloc(&ghist, 4 * R)); CK(cudaMalloc(&starts, 4 * (R + 1))); CK(cudaMalloc(&cur, 4 * R));
    CK(cudaMalloc(&rkey, 8 * n * c)); CK(cudaMalloc(&rmeta, 4 * n * c));
    CK(cudaMalloc(&bitmap, n / 8 + 64)); CK(cudaMalloc(&o1, n)); CK(cudaMalloc(&o2, n));
    fill_words<<<sms * 8, 256>>>(w, M * 16);
    fill_keys<<<sms * 8, 256>>>(keys, n, 12345);
    CK(cudaDeviceSynchronize());
    const bool SM = R <= 8192;
    const size_t cnt_smem = SM ? 4 * R : 0, sc_smem = SM ? 8 * R : 0, slab = 64 * kRegBlocks;
    CK(cudaFuncSetAttribute(count_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
    CK(cudaFuncSetAttribute(scatter_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024));
    CK(cudaFuncSetAttribute(region_lookup_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)slab));
    cudaEvent_t ev[8];
    for (auto &e : ev) CK(cudaEventCreate(&e));
    float best[6] = {1e9, 1e9, 1e9, 1e9, 1e9, 1e9};
    for (int rep = 0; rep < 3; ++rep) {
        CK(cudaEventRecord(ev[0]));
        direct_kernel<<<sms * 16, 256>>>(p, w, keys, n, o1);
        CK(cudaEventRecord(ev[1]));
        CK(cudaMemsetAsync(ghist, 0, 4 * R));
        CK(cudaMemsetAsync(bitmap, 0, n / 8 + 64));
        if (SM) count_kernel<true><<<sms * 2, 512, cnt_smem>>>(p, keys, n, R, ghist);
        else count_kernel<false><<<sms * 4, 512>>>(p, keys, n, R, ghist);
        CK(cudaEventRecord(ev[2]));
        scan_kernel<<<1, 1024>>>(ghist, R, starts, cur);
        CK(cudaEventRecord(ev[3]));
        if (SM) scatter_kernel<true><<<sms * 1, 512, sc_smem>>>(p, keys, n, R, cur, rkey, rmeta, T);
        else scatter_kernel<false><<<sms * 4, 512>>>(p, keys, n, R, cur, rkey, rmeta, T);
        CK(cudaEventRecord(ev[4]));
        region_lookup_kernel<<<sms * 3, 512, slab>>>(p, w, R, starts, rkey, rmeta, bitmap);
        CK(cudaEventRecord(ev[5]));
        expand_kernel<<<sms * 8, 256>>>(bitmap, n, o2);
        CK(cudaEventRecord(ev[6]));
        CK(cudaEventSynchronize(ev[6]));
        CK(cudaGetLastError());
        for (int s = 0; s < 6; ++s) {
            float ms;
            CK(cudaEventElapsedTime(&ms, ev[s], ev[s + 1]));
            best[s] = std::min(best[s], ms);
        }
    }
    std::vector<unsigned char> h1(n), h2(n);
    CK(cudaMemcpy(h1.data(), o1, n, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(h2.data(), o2, n, cudaMemcpyDeviceToHost));
    u64 diff = 0, pos = 0;
    for (u64 i = 0; i < n; ++i) { diff += h1[i] != h2[i]; pos += h1[i]; }
    const float sorted = best[1] + best[2] + best[3] + best[4] + best[5];
    printf("filter %llu MiB M=2^%d R=%u keys 2^%d c=%u k=%u T=%u %s | direct %.3f ms (%.1f G/s) | count %.3f scan %.3f "
           "scatter %.3f lookup %.3f expand %.3f = %.3f ms (%.1f G/s, x%.2f) | pos %.3f diff %llu\n",
           mib, lgM, R, lg, c, k, T, SM ? "smem-agg" : "global-atomics", best[0], n / best[0] / 1e6, best[1],
           best[2], best[3], best[4], best[5], sorted, n / sorted / 1e6, best[0] / sorted, (double)pos / n, diff);
    return diff != 0;
}
