// Exact stream-order insert (c >= 2, 512-bit blocks, random strategy) for
// small filters, as a dataflow instead of claim rounds.
//
// The sequential rule (_kernels.py:133-174) makes key j depend on every
// earlier key that shares a candidate block with it: those keys' writes must
// be in the blocks j reads, and their reads must happen before j writes.
// Every later key touching a block waits for every earlier one, so each
// block is touched in stream order -- and nothing else is ordered.
//
//  1. tickets: for every (key, choice) pair, the number of earlier pairs on
//     the same block, i.e. its rank in a stable sort of the pairs by block
//     (cub::DeviceRadixSort over the block ids, then rank = sorted position -
//     start of the block's run);
//  2. execution: warps take 32-key tiles in stream order from a counter; a
//     key is ready when every one of its blocks' done-counters equals its
//     ticket there; it then reads its candidates, applies the reference's
//     decision, writes the chosen block (nobody else may touch it until this
//     key is done), and bumps the done-counter of every candidate
//     (release).  Keys whose predecessor is still running poll their
//     counters.
//
// No round barriers: the critical path is the longest chain of keys linked
// by shared blocks (274 keys for config 1's 2^20 keys on 2^15 blocks), each
// link one L2 round trip plus a commit, instead of one grid-wide round per
// link.  Deadlock-free without residency assumptions: tiles are taken in
// stream order and a warp takes its next tile only when it has finished the
// current one, so the earliest unfinished key is always held by a running
// warp and all its predecessors are done.
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <cstdlib>

#include "blocks.cuh"
#include "keysrc.cuh"
#include "launch.h"

#ifndef BC_TICKET_SLEEP
#define BC_TICKET_SLEEP 32  // ns between polls of a warp with waiting keys (0: spin)
#endif

namespace bc {

// Polls are relaxed (an acquire load would also invalidate L1 every time);
// one acq_rel fence after the poll that sees a key ready, and one before a
// key's counter increments, give the release/acquire pairing.
__device__ __forceinline__ u32 ld_relaxed_u32(const u32 *p) {
    u32 v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void fence_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

__device__ __forceinline__ void red_relaxed_add(u32 *p, u32 v) {
    asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Pairs (block of choice ci of key j, pair id j*C + ci); keys that do not
// exist (skipped q-gram windows) get the block id M, sorted past every real one.
template <class Src>
__global__ void __launch_bounds__(256) ticket_pairs_kernel(const __grid_constant__ KParams p,
                                                           const Src src, u64 n, u32 *blk,
                                                           u32 *pid) {
    const u64 stride = (u64)gridDim.x * blockDim.x;
    for (u64 j = blockIdx.x * (u64)blockDim.x + threadIdx.x; j < n; j += stride) {
        u64 x;
        const bool ok = src.admit(j, x);
        for (u32 ci = 0; ci < p.c; ++ci) {
            blk[j * p.c + ci] = ok ? (u32)block_index(p, x, ci) : (u32)p.num_blocks;
            pid[j * p.c + ci] = (u32)(j * p.c + ci);
        }
    }
}

// start[b] = first sorted position of block b's run
__global__ void __launch_bounds__(256) ticket_runs_kernel(const u32 *sblk, u64 m, u32 *start) {
    const u64 stride = (u64)gridDim.x * blockDim.x;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < m; i += stride)
        if (i == 0 || sblk[i - 1] != sblk[i]) start[sblk[i]] = (u32)i;
}

__global__ void __launch_bounds__(256) ticket_rank_kernel(const u32 *sblk, const u32 *spid, u64 m,
                                                          const u32 *start, u32 *ticket) {
    const u64 stride = (u64)gridDim.x * blockDim.x;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < m; i += stride)
        ticket[spid[i]] = (u32)i - start[sblk[i]];
}

template <int C, class Src>
__global__ void __launch_bounds__(256) ticket_exec_kernel(
    const __grid_constant__ KParams p, u64 *__restrict__ words, const Src src, u64 n,
    const u32 *__restrict__ ticket, u32 *__restrict__ done, u32 *__restrict__ tile_ctr,
    unsigned long long *__restrict__ admitted) {
    __shared__ u32 mcol[16][256];  // per-thread 512-bit mask columns
    const u32 tid = threadIdx.x, lane = tid & 31;
    u32 *col = &mcol[0][tid];
    const u64 ntiles = (n + 31) / 32;
    const uint4 *w4 = reinterpret_cast<const uint4 *>(words);
    u32 n_adm = 0;
    for (;;) {
        u32 t = 0;
        if (lane == 0) t = atomicAdd(tile_ctr, 1u);
        t = __shfl_sync(kFull, t, 0);
        if (t >= ntiles) break;
        const u64 j = (u64)t * 32 + lane;
        u64 x = 0;
        const bool valid = j < n && src.admit(j, x);
        n_adm += valid ? 1u : 0u;
        u32 bl[C], want[C];
        if (valid) {
#pragma unroll
            for (int ci = 0; ci < C; ++ci) {
                bl[ci] = (u32)block_index(p, x, ci);
                want[ci] = __ldg(ticket + j * C + ci);
            }
            // a block chosen twice by one key holds two consecutive tickets:
            // the key is ready when the first of them is reached
#pragma unroll
            for (int ci = 1; ci < C; ++ci)
#pragma unroll
                for (int cj = 0; cj < ci; ++cj) want[ci] -= (u32)(bl[cj] == bl[ci]);
#pragma unroll
            for (int w = 0; w < 16; ++w) col[w * 256] = 0u;
            const u32 xlo = (u32)x, xhi = (u32)(x >> 32);
            for (u32 i = 0; i < p.k; ++i) {
                const u32 hi = mul_hi32(p.bit_a_lo[i], p.bit_a_hi[i], xlo, xhi);
                atomicOr(&col[(hi >> 28) * 256], 1u << ((hi >> 23) & 31u));
            }
        }
        bool pend = valid;
        while (__any_sync(kFull, pend)) {
            if (pend) {
                bool ready = true;
#pragma unroll
                for (int ci = 0; ci < C; ++ci) ready &= ld_relaxed_u32(done + bl[ci]) == want[ci];
                if (ready) {
                    fence_gpu();  // acquire: the predecessors' writes
                    uint4 m[4], wv[C][4];
#pragma unroll
                    for (int ci = 0; ci < C; ++ci)
#pragma unroll
                        for (int q = 0; q < 4; ++q) wv[ci][q] = ld_block_cg(w4 + (u64)bl[ci] * 4 + q);
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        m[q] = make_uint4(col[(4 * q) * 256], col[(4 * q + 1) * 256],
                                          col[(4 * q + 2) * 256], col[(4 * q + 3) * 256]);
                    bool noop = false;
                    int best = 0;
                    u32 best_r = 0xffffffffu;
#pragma unroll
                    for (int ci = 0; ci < C; ++ci) {
                        u32 jj = 0, pres = 0;
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const uint4 w = wv[ci][q];
                            jj += popc4(make_uint4(w.x | m[q].x, w.y | m[q].y, w.z | m[q].z,
                                                   w.w | m[q].w));
                            pres += popc4(w);
                        }
                        noop |= jj == pres;
                        const u32 r = __ldg(p.rank + jj * (p.k + 1) + (jj - pres));
                        if (r < best_r) {
                            best_r = r;
                            best = ci;
                        }
                    }
                    if (!noop) {
#pragma unroll
                        for (int ci = 0; ci < C; ++ci)
                            if (ci == best)
#pragma unroll
                                for (int q = 0; q < 4; ++q) {
                                    const uint4 w = wv[ci][q];
                                    __stcg(reinterpret_cast<uint4 *>(words) + (u64)bl[ci] * 4 + q,
                                           make_uint4(w.x | m[q].x, w.y | m[q].y, w.z | m[q].z,
                                                      w.w | m[q].w));
                                }
                    }
                    // release: the write is visible before any successor sees the
                    // counters move
                    fence_gpu();
#pragma unroll
                    for (int ci = 0; ci < C; ++ci) red_relaxed_add(done + bl[ci], 1u);
                    pend = false;
                }
            }
#if BC_TICKET_SLEEP
            if (__any_sync(kFull, pend)) __nanosleep(BC_TICKET_SLEEP);
#endif
        }
    }
    if (Src::kCounts && admitted != nullptr) {
        for (int o = 16; o > 0; o >>= 1) n_adm += __shfl_xor_sync(kFull, n_adm, o);
        if (lane == 0 && n_adm) atomicAdd(admitted, (unsigned long long)n_adm);
    }
}

// ---- version-tagged block records (BC_TICKET_REC_MAX_BLOCKS) ---------------------------------------
// The hop from a key to its successor on a block above costs a fence after
// the block store, the counter increment, the successor's poll, a fence and
// the successor's block load: four L2 round trips on the critical path.  With
// records, the block's words and its done-count travel together: block b is
// kRecChunks 16-byte chunks, each three data words and the count as its tag.
// A key polls its candidates' records until every chunk's tag equals its
// ticket -- the data are then exactly the block after its predecessor -- and
// publishes each candidate (the chosen one OR-ed with its mask, the others
// as read) with the tag moved past its own ticket(s).  Each 16-byte chunk is
// one aligned vector store and load, single-copy atomic in practice (the
// assumption CUB's decoupled look-back makes for its 16-byte tile
// descriptors), so a chunk is either wholly before or wholly after a
// publication and no fences are needed: one store-to-load latency per hop.
// Tags are cumulative over ticket sets (the rank kernel adds the tag a block
// has when its set starts), so records are converted from and back to the
// filter's words once per insert.
constexpr int kRecChunks = 6;  // 16 data words in chunks of three

__device__ __forceinline__ uint4 ld_relaxed_v4(const uint4 *p) {
    uint4 v;
    asm volatile("ld.relaxed.gpu.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p)
                 : "memory");
    return v;
}

__device__ __forceinline__ void st_relaxed_v4(uint4 *p, uint4 v) {
    asm volatile("st.relaxed.gpu.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w)
                 : "memory");
}

__global__ void __launch_bounds__(256) rec_from_words_kernel(const u32 *__restrict__ words, u64 M,
                                                             uint4 *__restrict__ rec) {
    const u64 stride = (u64)gridDim.x * blockDim.x;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < M * kRecChunks; i += stride) {
        const u64 b = i / kRecChunks;
        const u32 q = (u32)(i - b * kRecChunks), w0 = 3 * q;
        const u32 *src = words + b * 16;
        rec[i] = make_uint4(src[w0], w0 + 1 < 16 ? src[w0 + 1] : 0u, w0 + 2 < 16 ? src[w0 + 2] : 0u,
                            0u);
    }
}

__global__ void __launch_bounds__(256) rec_to_words_kernel(const uint4 *__restrict__ rec, u64 M,
                                                           u32 *__restrict__ words) {
    const u64 stride = (u64)gridDim.x * blockDim.x;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < M * 16; i += stride) {
        const u64 b = i >> 4;
        const u32 w = (u32)(i & 15u), q = w / 3, r = w - 3 * q;
        const uint4 c = rec[b * kRecChunks + q];
        words[i] = r == 0 ? c.x : (r == 1 ? c.y : c.z);
    }
}

// ticket = rank in the set + the block's tag when the set starts
__global__ void __launch_bounds__(256) ticket_rank_rec_kernel(const u32 *sblk, const u32 *spid,
                                                              u64 m, const u32 *start, u64 M,
                                                              const uint4 *rec, u32 *ticket) {
    const u64 stride = (u64)gridDim.x * blockDim.x;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < m; i += stride) {
        const u32 b = sblk[i];
        ticket[spid[i]] = (u32)i - start[b] + (b < M ? rec[(u64)b * kRecChunks].w : 0u);
    }
}

template <int C, class Src>
__global__ void __launch_bounds__(256) ticket_rec_kernel(
    const __grid_constant__ KParams p, uint4 *__restrict__ rec, const Src src, u64 n,
    const u32 *__restrict__ ticket, u32 *__restrict__ tile_ctr,
    unsigned long long *__restrict__ admitted) {
    __shared__ u32 mcol[16][256];  // per-thread 512-bit mask columns
    const u32 tid = threadIdx.x, lane = tid & 31;
    u32 *col = &mcol[0][tid];
    const u64 ntiles = (n + 31) / 32;
    u32 n_adm = 0;
    for (;;) {
        u32 t = 0;
        if (lane == 0) t = atomicAdd(tile_ctr, 1u);
        t = __shfl_sync(kFull, t, 0);
        if (t >= ntiles) break;
        const u64 j = (u64)t * 32 + lane;
        u64 x = 0;
        const bool valid = j < n && src.admit(j, x);
        n_adm += valid ? 1u : 0u;
        u32 bl[C], want[C], nxt[C];
        u32 first = 0;  // bit ci: ci is the first occurrence of its block
        if (valid) {
#pragma unroll
            for (int ci = 0; ci < C; ++ci) {
                bl[ci] = (u32)block_index(p, x, ci);
                want[ci] = __ldg(ticket + j * C + ci);
            }
            // a block chosen m times by one key holds m consecutive tickets:
            // wait for the first, publish past the last
#pragma unroll
            for (int ci = 0; ci < C; ++ci) {
                u32 lo = want[ci], hi = want[ci];
#pragma unroll
                for (int cj = 0; cj < C; ++cj)
                    if (bl[cj] == bl[ci]) {
                        lo = min(lo, want[cj]);
                        hi = max(hi, want[cj]);
                    }
                bool dup = false;
#pragma unroll
                for (int cj = 0; cj < ci; ++cj) dup |= bl[cj] == bl[ci];
                first |= dup ? 0u : (1u << ci);
                want[ci] = lo;
                nxt[ci] = hi + 1;
            }
#pragma unroll
            for (int w = 0; w < 16; ++w) col[w * 256] = 0u;
            const u32 xlo = (u32)x, xhi = (u32)(x >> 32);
            for (u32 i = 0; i < p.k; ++i) {
                const u32 hi = mul_hi32(p.bit_a_lo[i], p.bit_a_hi[i], xlo, xhi);
                atomicOr(&col[(hi >> 28) * 256], 1u << ((hi >> 23) & 31u));
            }
        }
        bool pend = valid;
        // per candidate: its record read and current (held until this key
        // publishes: nobody else may advance it), or the predecessors still
        // ahead of the key there as last seen.  Two or more ahead: only the
        // tag of chunk 0 is polled (16 instead of 96 bytes), so keys queued
        // deep behind others do not flood L2 with full-record polls.
        uint4 d[C][kRecChunks];
        u32 got = 0, far = 0;
        while (__any_sync(kFull, pend)) {
            if (pend) {
#pragma unroll
                for (int ci = 0; ci < C; ++ci)
                    if (((first & ~got) >> ci) & 1u) {
                        const uint4 *r = rec + (u64)bl[ci] * kRecChunks;
                        if ((far >> ci) & 1u) {
                            const u32 tag = ld_relaxed_v4(r).w;
                            far = want[ci] - tag >= 2u ? far : far & ~(1u << ci);
                        } else {
                            bool ok = true;
#pragma unroll
                            for (int q = 0; q < kRecChunks; ++q) {
                                d[ci][q] = ld_relaxed_v4(r + q);
                                ok &= d[ci][q].w == want[ci];
                            }
                            got |= ok ? (1u << ci) : 0u;
                            far |= (!ok && want[ci] - d[ci][0].w >= 2u) ? (1u << ci) : 0u;
                        }
                    }
                if ((got & first) == first) {
                    u32 m[18];
#pragma unroll
                    for (int w = 0; w < 16; ++w) m[w] = col[w * 256];
                    m[16] = m[17] = 0u;
                    bool noop = false;
                    int best = 0;
                    u32 best_r = 0xffffffffu;
#pragma unroll
                    for (int ci = 0; ci < C; ++ci) {
                        // a repeated block: the data of its first occurrence
                        int src_ci = ci;
#pragma unroll
                        for (int cj = C - 1; cj >= 0; --cj)
                            if (cj < ci && bl[cj] == bl[ci]) src_ci = cj;
                        u32 jj = 0, pres = 0;
#pragma unroll
                        for (int q = 0; q < kRecChunks; ++q) {
                            uint4 w = d[0][q];
#pragma unroll
                            for (int cs = 1; cs < C; ++cs)
                                if (cs == src_ci) w = d[cs][q];
                            jj += __popc(w.x | m[3 * q]) + __popc(w.y | m[3 * q + 1]) +
                                  __popc(w.z | m[3 * q + 2]);
                            pres += __popc(w.x) + __popc(w.y) + __popc(w.z);
                        }
                        noop |= jj == pres;
                        const u32 r = __ldg(p.rank + jj * (p.k + 1) + (jj - pres));
                        if (r < best_r) {
                            best_r = r;
                            best = ci;
                        }
                    }
                    // the chosen block is the first occurrence of its id
                    u32 chosen = bl[best];
#pragma unroll
                    for (int ci = 0; ci < C; ++ci)
                        if ((first >> ci) & 1u) {
                            const bool orit = !noop && bl[ci] == chosen;
#pragma unroll
                            for (int q = 0; q < kRecChunks; ++q) {
                                const uint4 w = d[ci][q];
                                st_relaxed_v4(rec + (u64)bl[ci] * kRecChunks + q,
                                              orit ? make_uint4(w.x | m[3 * q], w.y | m[3 * q + 1],
                                                                w.z | m[3 * q + 2], nxt[ci])
                                                   : make_uint4(w.x, w.y, w.z, nxt[ci]));
                            }
                        }
                    pend = false;
                }
            }
#if BC_TICKET_SLEEP
            if (__any_sync(kFull, pend)) __nanosleep(BC_TICKET_SLEEP);
#endif
        }
    }
    if (Src::kCounts && admitted != nullptr) {
        for (int o = 16; o > 0; o >>= 1) n_adm += __shfl_xor_sync(kFull, n_adm, o);
        if (lane == 0 && n_adm) atomicAdd(admitted, (unsigned long long)n_adm);
    }
}

// ---- host side -------------------------------------------------------------------------

static u64 env_u64(const char *name, u64 dflt) {
    const char *e = std::getenv(name);
    return e ? std::strtoull(e, nullptr, 10) : dflt;
}

// Filters up to this many blocks run the ticket execution over version-tagged
// records (ticket_rec_kernel): there the chains of dependent keys set the
// rate, and a record hop is one store-to-load latency.  Above it the
// execution is throughput-bound and the records' wider polls and full
// rewrites of every candidate cost more than they save (BC_TICKET_REC_MAX_BLOCKS).
static u64 ticket_rec_max_blocks() { return env_u64("BC_TICKET_REC_MAX_BLOCKS", 1ull << 18); }

// Keys per ticket set (tickets are ranks within one set; sets run in stream
// order; BC_TICKET_CHUNK overrides, for tests).
static u64 ticket_chunk() { return std::max<u64>(1, env_u64("BC_TICKET_CHUNK", 1ull << 24)); }

// Filters up to 2^20 blocks (64 MiB), or 2^21 with three or more choices,
// where claim rounds pay for many conflicts per round (measured, B200,
// tools/ordered_probe.py bits:n:c:k at 14-16 bits per key: c = 2 at 2^18 /
// 2^19 / 2^20 blocks 3843 / 4009 / 4152 vs 2174 / 2850 / 3188 Mkeys/s, at
// 2^21 4148 vs 6017; c = 3 at 2^18 / 2^20 / 2^21 2026 / 1940 / 2376 vs
// 604 / 927 / 1783).  BC_TICKET_MAX_BLOCKS overrides, BC_ORDERED_TICKET=0
// disables.
bool ordered_ticket_supported(const KParams &p) {
    if (!(p.fast_random && p.wpb == 8 && p.c >= 2 && p.c <= 8)) return false;
    if (env_u64("BC_ORDERED_TICKET", 1) == 0) return false;
    // crossover with the one-array claim rounds at their M / (2 c^2) window
    // (tools/r2_crossover.sh, r2_crossover2.sh; Mkeys/s ticket / claims):
    // c = 2: 2^18 blocks 3 812 / 3 167, 3*2^17 4 078 / 4 013, 2^19 4 007 / 4 921;
    // c = 3: 3*2^17 2 242 / 1 431, 2^19 ~1 850 (erratic: 290 .. 1 850) / 2 000,
    // 3*2^18 2 152 / 2 575
    // Above 3*2^17 blocks the dataflow's rate is erratic for c = 3
    // (tools/r2_ticket_stability.sh: 7*2^16 blocks 1 092 .. 1 980 Mkeys/s over
    // four runs, 2^19 blocks 290 .. 1 851 over three sessions; steady at and
    // below 3*2^17), so both limits sit there.
    const u64 dflt = 3ull << 17;
    return p.num_blocks <= env_u64("BC_TICKET_MAX_BLOCKS", dflt);
}

template <int C, class Src>
static cudaError_t exec_launch(const KParams &p, u64 *words, const Src &src, u64 n,
                               const u32 *ticket, u32 *done, u32 *ctr,
                               unsigned long long *admitted, cudaStream_t s) {
    // keys in flight (8 warps x 32 per CTA) ~ M (BC_TICKET_INFLIGHT_PCT of
    // M): a window much wider than the filter only queues keys behind each
    // other on the same blocks and floods L2 with polls
    const void *fn = (const void *)ticket_exec_kernel<C, Src>;
    const u64 inflight = std::max<u64>(256, p.num_blocks * env_u64("BC_TICKET_INFLIGHT_PCT", 100) / 100);
    const unsigned grid = grid_for(fn, 256, 0, std::min<u64>((n + 255) / 256, (inflight + 255) / 256));
    ticket_exec_kernel<C, Src><<<grid, 256, 0, s>>>(p, words, src, n, ticket, done, ctr, admitted);
    count_launch();
    return cudaGetLastError();
}

template <int C, class Src>
static cudaError_t rec_launch(const KParams &p, uint4 *rec, const Src &src, u64 n,
                              const u32 *ticket, u32 *ctr, unsigned long long *admitted,
                              cudaStream_t s) {
    const void *fn = (const void *)ticket_rec_kernel<C, Src>;
    const u64 inflight = std::max<u64>(256, p.num_blocks * env_u64("BC_TICKET_INFLIGHT_PCT", 100) / 100);
    const unsigned grid = grid_for(fn, 256, 0, std::min<u64>((n + 255) / 256, (inflight + 255) / 256));
    ticket_rec_kernel<C, Src><<<grid, 256, 0, s>>>(p, rec, src, n, ticket, ctr, admitted);
    count_launch();
    return cudaGetLastError();
}

template <class Src>
static cudaError_t ticket_insert(const KParams &p, u64 *words, const Src &src, u64 n,
                                 unsigned long long *admitted, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const u64 c = p.c, M = p.num_blocks;
    const u64 per = std::min(n, ticket_chunk());
    const u64 m = per * c;
    int bits = 1;
    while ((1ull << bits) <= M) ++bits;  // block ids 0..M (M marks a skipped window)
    size_t cub_bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, cub_bytes, (const u32 *)nullptr, (u32 *)nullptr,
                                    (const u32 *)nullptr, (u32 *)nullptr, (int)m, 0, bits, s);
    // scratch: blk in/out, pid in/out, ticket (m each), start + done (M + 1 each), counter
    // (records: M x kRecChunks x 16 bytes after the cub scratch)
    const size_t words32 = 5 * m + 2 * (M + 1) + 1;
    const size_t cub_off = ((words32 * 4 + 255) / 256) * 256;
    const size_t rec_off = ((cub_off + cub_bytes + 255) / 256) * 256;
    const bool use_rec = M <= ticket_rec_max_blocks();
    const size_t rec_bytes = use_rec ? (size_t)M * kRecChunks * 16 : 0;
    unsigned char *scratch = nullptr;
    cudaError_t e = cudaMallocAsync((void **)&scratch, rec_off + rec_bytes, s);
    if (e != cudaSuccess) return e;
    u32 *blk = reinterpret_cast<u32 *>(scratch), *sblk = blk + m, *pid = sblk + m,
        *spid = pid + m, *ticket = spid + m, *start = ticket + m, *done = start + (M + 1),
        *ctr = done + (M + 1);
    void *cub_tmp = scratch + cub_off;
    uint4 *rec = reinterpret_cast<uint4 *>(scratch + rec_off);
    const KParams &kp = p;
    if (use_rec) {
        const unsigned g = grid_for((const void *)rec_from_words_kernel, 256, 0,
                                    (M * kRecChunks + 255) / 256);
        rec_from_words_kernel<<<g, 256, 0, s>>>(reinterpret_cast<const u32 *>(words), M, rec);
        count_launch();
    }
    for (u64 off = 0; off < n && e == cudaSuccess; off += per) {
        const u64 len = std::min(per, n - off);
        const u64 ml = len * c;
        Src sub = src;
        sub.advance(off);
        const unsigned g1 = grid_for((const void *)ticket_pairs_kernel<Src>, 256, 0,
                                     (len + 255) / 256);
        ticket_pairs_kernel<Src><<<g1, 256, 0, s>>>(kp, sub, len, blk, pid);
        count_launch();
        size_t tb = cub_bytes;
        e = cub::DeviceRadixSort::SortPairs(cub_tmp, tb, blk, sblk, pid, spid, (int)ml, 0, bits,
                                            s);
        if (e != cudaSuccess) break;
        const unsigned g2 = grid_for((const void *)ticket_runs_kernel, 256, 0, (ml + 255) / 256);
        ticket_runs_kernel<<<g2, 256, 0, s>>>(sblk, ml, start);
        if (use_rec)
            ticket_rank_rec_kernel<<<g2, 256, 0, s>>>(sblk, spid, ml, start, M, rec, ticket);
        else
            ticket_rank_kernel<<<g2, 256, 0, s>>>(sblk, spid, ml, start, ticket);
        count_launch(2);
        e = use_rec ? cudaMemsetAsync(ctr, 0, sizeof(u32), s)
                          : cudaMemsetAsync(done, 0, sizeof(u32) * (M + 2), s);  // done[] + counter
        if (e != cudaSuccess) break;
        switch (p.c) {
#define BC_TK(cc)                                                                             \
    case cc:                                                                                  \
        e = use_rec ? rec_launch<cc, Src>(kp, rec, sub, len, ticket, ctr, admitted, s)        \
                    : exec_launch<cc, Src>(kp, words, sub, len, ticket, done, ctr, admitted, s); \
        break;
            BC_TK(2) BC_TK(3) BC_TK(4) BC_TK(5) BC_TK(6) BC_TK(7) BC_TK(8)
#undef BC_TK
            default: e = cudaErrorInvalidValue;
        }
        if (e == cudaSuccess) e = cudaGetLastError();
    }
    if (use_rec && e == cudaSuccess) {
        const unsigned g = grid_for((const void *)rec_to_words_kernel, 256, 0, (M * 16 + 255) / 256);
        rec_to_words_kernel<<<g, 256, 0, s>>>(rec, M, reinterpret_cast<u32 *>(words));
        count_launch();
        e = cudaGetLastError();
    }
    cudaFreeAsync(scratch, s);
    return e;
}

cudaError_t launch_ordered_ticket(const KParams &p, u64 *words, const u64 *keys, u64 n,
                                  cudaStream_t s) {
    const ArrayKeys src{keys};
    return ticket_insert(p, words, src, n, nullptr, s);
}

cudaError_t launch_ordered_ticket_qgrams(const KParams &p, u64 *words, const u8 *seq, u64 nwin,
                                         int q, int canonical, RecSpec rec,
                                         unsigned long long *count, cudaStream_t s) {
    SeqKeys src;
    src.seq = seq;
    src.rec = rec;
    src.q = (u32)q;
    src.canonical = (u32)canonical;
    src.qmask = q == 32 ? ~0ull : ((1ull << (2 * q)) - 1ull);
    return ticket_insert(p, words, src, nwin, count, s);
}

}  // namespace bc
