// Per-key work of the blocked family, shared by the key-array kernels
// (filter_kernels.cu) and the fused q-gram kernels (qgram_kernels.cu).
//
// 512-bit blocks (the reference's default, one 64-byte line) use a two-phase
// tile of kTPB keys per CTA iteration:
//
//   phase 1, one thread per key: hash the key (shard + c block hashes + k
//     bit hashes) and build its 512-bit bit mask in shared memory
//     (layout mask[word32][key], so lanes touch distinct banks);
//   phase 2, four lanes per key: lane s owns bytes [16s, 16s+16) of every
//     block, so one warp-wide LDG.128 moves eight whole 64-byte blocks (one
//     L1 wavefront per block instead of four) and the test / popcount /
//     atomic OR of a block is spread over the four lanes.
//
// Semantics follow _kernels.py:112-211 exactly: membership = any choice
// whose block holds every address; insert with c == 1 ORs the mask; with
// c >= 2 the first candidate that already holds every address wins as a
// no-op, otherwise the candidate with the strictly smallest cost (lowest
// index on ties).  Costs are compared through a host-built rank table that
// preserves the float64 order of the reference formulas, ties included.
#pragma once

#include "common.cuh"
#include "launch.h"

namespace bc {

constexpr int kTPB = 256;            // keys per tile == threads per CTA
constexpr int kGroups = kTPB / 4;    // keys per phase-2 pass
constexpr int kPasses = kTPB / kGroups;
constexpr u32 kFull = 0xffffffffu;

template <int C>
struct TileSmem {
    u32 mask[16][kTPB];   // 512-bit masks, word-major
    u32 blk[C][kTPB];     // candidate block indices
    u8 out[kTPB];         // lookup answers of the tile
};

__device__ __forceinline__ DevHash load_hash(const DevHash *h) {
    DevHash r;
    r.a = __ldg(&h->a);
    r.b = __ldg(&h->b);
    r.magic = __ldg(&h->magic);
    r.mode = __ldg(&h->mode);
    r.shift = __ldg(&h->shift);
    return r;
}

// ---- phase 1: one thread per key ------------------------------------------------
template <int C>
__device__ __forceinline__ void phase1(const KParams &p, u64 x, bool valid, TileSmem<C> &sm,
                                       int tid) {
    u32 *col = &sm.mask[0][tid];
#pragma unroll
    for (int w = 0; w < 16; ++w) col[w * kTPB] = 0u;
    if (valid) {
        if (p.fast_random) {
            const u32 xlo = (u32)x, xhi = (u32)(x >> 32);
#pragma unroll 4
            for (u32 i = 0; i < p.k; ++i) {
                u32 h = bit512(p.bit_a_lo[i], p.bit_a_hi[i], xlo, xhi);
                col[(h >> 5) * kTPB] |= 1u << (h & 31);
            }
        } else if (p.strategy == 0) {
            for (u32 i = 0; i < p.k; ++i) {
                u32 h = (u32)hval(load_hash(p.bits + i), x);
                col[(h >> 5) * kTPB] |= 1u << (h & 31);
            }
        } else {
            // distinct: the r-th address not chosen so far (hashing.py:181-200),
            // i.e. the r-th zero of the mask built so far.
            for (u32 i = 0; i < p.k; ++i) {
                u32 r = (u32)hval(load_hash(p.bits + i), x);
                u32 w = 0;
                for (;; ++w) {
                    u32 z = 32u - __popc(col[w * kTPB]);
                    if (r < z) break;
                    r -= z;
                }
                u32 pos = select_bit32(~col[w * kTPB], r);
                col[w * kTPB] |= 1u << pos;
            }
        }
    }
#pragma unroll
    for (int ci = 0; ci < C; ++ci) sm.blk[ci][tid] = valid ? (u32)block_index(p, x, ci) : 0u;
}

__device__ __forceinline__ u32 popc4(uint4 v) {
    return __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w);
}

__device__ __forceinline__ bool covers(uint4 w, uint4 m) {
    return ((w.x & m.x) == m.x) & ((w.y & m.y) == m.y) & ((w.z & m.z) == m.z) &
           ((w.w & m.w) == m.w);
}

// ---- phase 2: four lanes per key ---------------------------------------------------
// Returns the number of hits among valid keys handled by this lane (lookups).
template <int OP, int C>
__device__ __forceinline__ u32 phase2(const KParams &p, u64 *words, TileSmem<C> &sm, u32 cnt,
                                      int tid) {
    constexpr bool kNoLoad = (OP == OP_INSERT && C == 1);
    constexpr int UNR = kNoLoad ? 4 : (C <= 2 ? 4 : (C <= 4 ? 2 : 1));
    constexpr int CL = kNoLoad ? 1 : C;
    const int g = tid >> 2, s = tid & 3, lane = tid & 31;
    const uint4 *w4 = reinterpret_cast<const uint4 *>(words);
    u32 hits = 0;
#pragma unroll
    for (int p0 = 0; p0 < kPasses; p0 += UNR) {
        uint4 m[UNR];
        uint4 w[UNR][CL];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const int kk = (p0 + u) * kGroups + g;
            m[u] = make_uint4(sm.mask[4 * s][kk], sm.mask[4 * s + 1][kk], sm.mask[4 * s + 2][kk],
                              sm.mask[4 * s + 3][kk]);
            if (!kNoLoad) {
#pragma unroll
                for (int ci = 0; ci < C; ++ci) {
                    const u64 b = sm.blk[ci][kk];
                    w[u][ci] = OP == OP_CONTAINS ? ld_block_nc(w4 + b * 4 + s)
                                                 : ld_block_cg(w4 + b * 4 + s);
                }
            }
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const int kk = (p0 + u) * kGroups + g;
            const u64 lo = (u64)m[u].x | ((u64)m[u].y << 32);
            const u64 hi = (u64)m[u].z | ((u64)m[u].w << 32);
            if (OP == OP_CONTAINS) {
                bool found = false;
#pragma unroll
                for (int ci = 0; ci < CL; ++ci) {
                    u32 bal = __ballot_sync(kFull, covers(w[u][ci], m[u]));
                    found |= ((bal >> (lane & 28)) & 0xFu) == 0xFu;
                }
                if (s == 0) {
                    sm.out[kk] = (u8)found;
                    hits += (found && (u32)kk < cnt) ? 1u : 0u;
                }
            } else if (C == 1) {
                u64 *dst = words + (u64)sm.blk[0][kk] * 8 + 2 * s;
                red_or(dst, lo);
                red_or(dst + 1, hi);
            } else {
                u32 v[CL];
#pragma unroll
                for (int ci = 0; ci < CL; ++ci) {
                    uint4 ww = w[u][ci];
                    uint4 uni = make_uint4(ww.x | m[u].x, ww.y | m[u].y, ww.z | m[u].z,
                                           ww.w | m[u].w);
                    u32 t = popc4(uni) | (popc4(ww) << 16);
                    t += __shfl_xor_sync(kFull, t, 1);
                    t += __shfl_xor_sync(kFull, t, 2);
                    v[ci] = t;
                }
                int best = 0;
                u32 best_r = 0xffffffffu;
                bool noop = false;
#pragma unroll
                for (int ci = 0; ci < CL; ++ci) {
                    if (!noop) {
                        const u32 j = v[ci] & 0xffffu;
                        const u32 a = j - (v[ci] >> 16);
                        if (a == 0) {
                            noop = true;
                        } else {
                            const u32 r = __ldg(p.rank + j * (p.k + 1) + a);
                            if (r < best_r) {
                                best_r = r;
                                best = ci;
                            }
                        }
                    }
                }
                if (!noop) {
                    u64 *dst = words + (u64)sm.blk[best][kk] * 8 + 2 * s;
                    red_or(dst, lo);
                    red_or(dst + 1, hi);
                }
            }
        }
    }
    return hits;
}

// ---- thread-per-key building blocks (any block width, ordered inserts) -------------

__device__ __forceinline__ void build_mask_generic(const KParams &p, u64 x, u64 *mask) {
    for (u32 w = 0; w < p.wpb; ++w) mask[w] = 0;
    for (u32 i = 0; i < p.k; ++i) {
        u64 f = hval(load_hash(p.bits + i), x);
        if (p.strategy == 1) {
            u32 r = (u32)f, w = 0;
            for (;; ++w) {
                u32 z = 64u - (u32)__popcll(mask[w]);
                if (r < z) break;
                r -= z;
            }
            f = (u64)w * 64 + select_bit64(~mask[w], r);
        }
        mask[f >> 6] |= 1ull << (f & 63);
    }
}

// Reference insert decision for one key against L2-coherent block reads.
__device__ __forceinline__ void insert_generic(const KParams &p, u64 *words, u64 x,
                                               const u64 *mask) {
    const u32 wpb = p.wpb;
    if (p.c == 1) {
        u64 b = block_index(p, x, 0) * wpb;
        for (u32 w = 0; w < wpb; ++w) red_or(words + b + w, mask[w]);
        return;
    }
    int best = 0;
    u32 best_r = 0xffffffffu;
    u64 bases[kMaxChoices];
    for (u32 ci = 0; ci < p.c; ++ci) {
        const u64 b = block_index(p, x, ci) * wpb;
        bases[ci] = b;
        u32 j = 0, pr = 0;
        for (u32 w = 0; w < wpb; ++w) {
            u64 wv = __ldcg(words + b + w);
            j += (u32)__popcll(wv | mask[w]);
            pr += (u32)__popcll(wv);
        }
        const u32 a = j - pr;
        if (a == 0) return;  // no-op: the key is already represented
        const u32 r = __ldg(p.rank + j * (p.k + 1) + a);
        if (r < best_r) {
            best_r = r;
            best = (int)ci;
        }
    }
    for (u32 w = 0; w < wpb; ++w) red_or(words + bases[best] + w, mask[w]);
}

}  // namespace bc
