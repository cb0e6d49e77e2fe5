// Per-key work of the blocked family, shared by the key-array kernels
// (filter_kernels.cu) and the fused q-gram kernels (qgram_kernels.cu).
//
// 512-bit blocks (the reference's default, one 64-byte line) are processed
// by each warp in tiles of 32 keys, warp-synchronously (no CTA barrier):
//
//   phase 1, one lane per key: hash the key (shard + c block hashes + k
//     bit hashes) and build its 512-bit mask in the warp's shared-memory
//     slice, layout mask[word][key] -- every access of a lane hits bank
//     `lane`, so the data-dependent word index never causes a conflict;
//   phase 2, four lanes per key: group g (lanes 4g..4g+3) handles keys
//     4g..4g+3 of the tile in four passes; lane s owns bytes [16s, 16s+16)
//     of every block, so one warp-wide LDG.128 moves eight whole 64-byte
//     blocks (one L1 wavefront per block instead of four).  The masks of
//     all four passes are read up front in a rotated order (lane s reads
//     key 4g + ((p + s) & 3) in read p), which makes those 16 reads per lane
//     bank-conflict-free; the right slot is then selected per pass.
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

constexpr int kTPB = 256;      // threads per CTA
constexpr int kWarps = kTPB / 32;
constexpr u32 kFull = 0xffffffffu;

template <int C>
struct WarpSmem {
    u32 mask[16][32];  // 512-bit masks of the warp's 32 keys, word-major
    u32 blk[C][32];    // candidate block indices
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

// Candidate entry of a lane without a key (SKIP): relaxed_load reads nothing
// for it.  Without it such lanes read block 0, and in tiles that mix keys and
// holes (the exact-order rounds' winners and losers) every warp queues on
// that one line's L2 slice.
constexpr u32 kNoBlock = 0xffffffffu;

// ---- phase 1: one lane per key ----------------------------------------------------
template <int C, bool SKIP = false>
__device__ __forceinline__ void phase1(const KParams &p, u64 x, bool valid, WarpSmem<C> &ws,
                                       int lane) {
    u32 *col = &ws.mask[0][lane];
#pragma unroll
    for (int w = 0; w < 16; ++w) col[w * 32] = 0u;
    if (valid) {
        if (p.fast_random) {
            const u32 xlo = (u32)x, xhi = (u32)(x >> 32);
#pragma unroll 4
            for (u32 i = 0; i < p.k; ++i) {
                const u32 hi = mul_hi32(p.bit_a_lo[i], p.bit_a_hi[i], xlo, xhi);
                // bit (hi >> 23) & 31 of word hi >> 28; one shared-memory atomic
                // instead of a load / or / store chain (each lane owns its column)
#ifdef BC_PHASE1_RMW
                col[(hi >> 28) * 32] |= __funnelshift_l(0u, 1u, hi >> 23);
#else
                atomicOr(&col[(hi >> 28) * 32], __funnelshift_l(0u, 1u, hi >> 23));
#endif
            }
        } else if (p.strategy == 0) {
            for (u32 i = 0; i < p.k; ++i) {
                u32 h = (u32)hval(load_hash(p.bits + i), x);
                col[(h >> 5) * 32] |= 1u << (h & 31);
            }
        } else {
            // distinct: the r-th address not chosen so far (hashing.py:181-200),
            // i.e. the r-th zero of the mask built so far.
            for (u32 i = 0; i < p.k; ++i) {
                u32 r = (u32)hval(load_hash(p.bits + i), x);
                u32 w = 0;
                for (;; ++w) {
                    u32 z = 32u - __popc(col[w * 32]);
                    if (r < z) break;
                    r -= z;
                }
                col[w * 32] |= 1u << select_bit32(~col[w * 32], r);
            }
        }
    }
#pragma unroll
    for (int ci = 0; ci < C; ++ci)
        ws.blk[ci][lane] = valid ? (u32)block_index(p, x, ci) : (SKIP ? kNoBlock : 0u);
}

__device__ __forceinline__ u32 popc4(uint4 v) {
    return __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w);
}

// every mask bit set in w: (m & ~w) == 0, folded with LOP3s
__device__ __forceinline__ bool covers(uint4 w, uint4 m) {
    return ((m.x & ~w.x) | (m.y & ~w.y) | (m.z & ~w.z) | (m.w & ~w.w)) == 0u;
}

// r = p ? a : b as a SEL (keeps ptxas from turning the lane-divergent
// selection into branches)
__device__ __forceinline__ u32 selp(u32 a, u32 b, u32 p) {
    u32 r;
    asm("{.reg .pred q; setp.ne.u32 q, %3, 0; selp.b32 %0, %1, %2, q;}"
        : "=r"(r)
        : "r"(a), "r"(b), "r"(p));
    return r;
}

__device__ __forceinline__ uint4 selp4(const uint4 &a, const uint4 &b, u32 p) {
    return make_uint4(selp(a.x, b.x, p), selp(a.y, b.y, p), selp(a.z, b.z, p),
                      selp(a.w, b.w, p));
}

// M[i] for a lane-dependent i in [0, 4): two levels of SELs, no branches.
__device__ __forceinline__ uint4 sel4(const uint4 (&M)[4], int i) {
    const uint4 lo = selp4(M[1], M[0], i & 1);
    const uint4 hi = selp4(M[3], M[2], i & 1);
    return selp4(hi, lo, i & 2);
}

// ---- relaxed multi-choice insert steps (four lanes per key) ------------------------
// A step covers keys 4g + p0 .. 4g + p0 + UNR - 1 of the tile: first the
// candidate slices are loaded (relaxed_load), then (relaxed_commit) every
// stage -- popcounts, the two shuffle rounds, the rank loads, the REDs -- runs
// over all UNR keys at once, so the keys are independent work instead of one
// dependent chain each.  Splitting the two lets a kernel overlap other work
// (the next tile's phase 1) with the loads.
constexpr int relaxed_unroll(int C) { return C <= 2 ? 4 : (C <= 4 ? 2 : 1); }

// Where block b's eight words are.  LocalWords: one array.  PartWords: the
// filter spread over the replicas of a partitioned multi-GPU build (block b
// is read and written in the replica of rank b / per, mapped into this
// process over peer memory, at the same offset).
struct LocalWords {
    u64 *words;
    __device__ __forceinline__ u64 *block(u64 b) const { return words + b * 8; }
};

struct PartWords {
    u64 *part[kMaxParts];  // rank r's replica (this process's address of it)
    u64 per;               // blocks per rank (ranks own contiguous block ranges)
    u64 magic;             // floor(2^64 / per)
    __device__ __forceinline__ u64 *block(u64 b) const {
        u64 q = __umul64hi(b, magic);
        if (b - q * per >= per) ++q;  // the estimate is exact or one short (common.cuh)
        return part[q] + b * 8;
    }
};

template <int C, int UNR, class A = LocalWords>
__device__ __forceinline__ void relaxed_load(const WarpSmem<C> &ws, const A &a, int lane, int p0,
                                             uint4 (&w)[UNR][C]) {
    const int g = lane >> 2, s = lane & 3;
#pragma unroll
    for (int u = 0; u < UNR; ++u)
#pragma unroll
        for (int ci = 0; ci < C; ++ci) {
            const u32 b = ws.blk[ci][4 * g + p0 + u];
            w[u][ci] = make_uint4(0u, 0u, 0u, 0u);  // a hole: all-zero mask too, a no-op
            if (b != kNoBlock)
                w[u][ci] = ld_block_cg(reinterpret_cast<const uint4 *>(a.block(b)) + s);
        }
}

template <int C, int UNR, class A = LocalWords>
__device__ __forceinline__ void relaxed_commit(const KParams &p, const A &a,
                                               const WarpSmem<C> &ws, const uint4 (&M)[4],
                                               int lane, int p0, const uint4 (&w)[UNR][C]) {
    const int g = lane >> 2, s = lane & 3;
    u32 t[UNR][C];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
        const uint4 m = sel4(M, (p0 + u - s) & 3);
#pragma unroll
        for (int ci = 0; ci < C; ++ci) {
            const uint4 ww = w[u][ci];
            const uint4 uni = make_uint4(ww.x | m.x, ww.y | m.y, ww.z | m.z, ww.w | m.w);
            t[u][ci] = popc4(uni) | (popc4(ww) << 16);  // j | present << 16
        }
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u)
#pragma unroll
        for (int ci = 0; ci < C; ++ci) t[u][ci] += __shfl_xor_sync(kFull, t[u][ci], 1);
#pragma unroll
    for (int u = 0; u < UNR; ++u)
#pragma unroll
        for (int ci = 0; ci < C; ++ci) t[u][ci] += __shfl_xor_sync(kFull, t[u][ci], 2);
    // a == 0 at any candidate -> no-op (_kernels.py:156-160); otherwise the
    // strict-< argmin of the cost rank, lowest index on ties
    u32 r[UNR][C];
#pragma unroll
    for (int u = 0; u < UNR; ++u)
#pragma unroll
        for (int ci = 0; ci < C; ++ci) {
            const u32 j = t[u][ci] & 0xffffu, a = j - (t[u][ci] >> 16);
            r[u][ci] = __ldg(p.rank + j * (p.k + 1) + a);
        }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
        bool noop = false;
        int best = 0;
        u32 best_r = 0xffffffffu;
#pragma unroll
        for (int ci = 0; ci < C; ++ci) {
            noop |= (t[u][ci] & 0xffffu) == (t[u][ci] >> 16);
            if (r[u][ci] < best_r) {
                best_r = r[u][ci];
                best = ci;
            }
        }
        if (!noop) {
            const uint4 m = sel4(M, (p0 + u - s) & 3);
            u64 *dst = a.block(ws.blk[best][4 * g + p0 + u]) + 2 * s;
            red_or_all(dst, (u64)m.x | ((u64)m.y << 32));
            red_or_all(dst + 1, (u64)m.z | ((u64)m.w << 32));
        }
    }
}

// The group's mask slices for the four passes, read in rotated order (see the
// file comment): lane s holds 64-bit words {2s, 2s+1}, or {s, s+4} (kNoLoad).
template <int C>
__device__ __forceinline__ void read_masks(const WarpSmem<C> &ws, int lane, bool no_load,
                                           uint4 (&M)[4]) {
    const int g = lane >> 2, s = lane & 3;
    const int w0 = no_load ? 2 * s : 4 * s, w2 = no_load ? 2 * s + 8 : 4 * s + 2;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const int kr = 4 * g + ((r + s) & 3);
        M[r] = make_uint4(ws.mask[w0][kr], ws.mask[w0 + 1][kr], ws.mask[w2][kr],
                          ws.mask[w2 + 1][kr]);
    }
}

// ---- phase 2: four lanes per key -------------------------------------------------
// Lookups: returns the answers of the group's four keys packed one per byte
// (key 4g + p in byte p), identical in the four lanes of the group.
template <int OP, int C, int UNRX = 0>
__device__ __forceinline__ u32 phase2(const KParams &p, u64 *words, WarpSmem<C> &ws,
                                      int lane) {
    constexpr bool kNoLoad = (OP == OP_INSERT && C == 1);
    constexpr int UNR = kNoLoad ? 4 : (UNRX ? UNRX : relaxed_unroll(C));
    constexpr int CL = kNoLoad ? 1 : C;
    const int g = lane >> 2, s = lane & 3;
    const uint4 *w4 = reinterpret_cast<const uint4 *>(words);
    // Lane s holds 64-bit mask words {2s, 2s+1} (matching its 16-byte slice of
    // a loaded block), or -- for single-choice inserts, which load nothing --
    // words {s, s+4}, so each of the two RED instructions of a group stays
    // inside one 32-byte sector (tools/gather_probe.cu scatter mode 6 vs 0).
    uint4 M[4];
    read_masks<C>(ws, lane, kNoLoad, M);
    u32 found_bytes = 0;
    if constexpr (OP == OP_INSERT && C >= 2) {
#pragma unroll
        for (int p0 = 0; p0 < 4; p0 += UNR) {
            uint4 w[UNR][C];
            const LocalWords lw{words};
            relaxed_load<C, UNR>(ws, lw, lane, p0, w);
            relaxed_commit<C, UNR>(p, lw, ws, M, lane, p0, w);
        }
        return 0;
    } else {
#pragma unroll
        for (int p0 = 0; p0 < 4; p0 += UNR) {
            uint4 w[UNR][CL];
            if (!kNoLoad) {
#pragma unroll
                for (int u = 0; u < UNR; ++u) {
                    const int kk = 4 * g + p0 + u;
#pragma unroll
                    for (int ci = 0; ci < C; ++ci) {
                        const u64 b = ws.blk[ci][kk];
                        w[u][ci] = ld_block_cg(w4 + b * 4 + s);
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < UNR; ++u) {
                const int pass = p0 + u;
                const int kk = 4 * g + pass;
                const uint4 m = sel4(M, (pass - s) & 3);
                const u64 lo = (u64)m.x | ((u64)m.y << 32);
                const u64 hi = (u64)m.z | ((u64)m.w << 32);
                if (OP == OP_CONTAINS) {
                    bool found = false;
#pragma unroll
                    for (int ci = 0; ci < CL; ++ci) {
                        const u32 bal = __ballot_sync(kFull, covers(w[u][ci], m));
                        found |= ((bal >> (lane & 28)) & 0xFu) == 0xFu;
                    }
                    found_bytes |= (found ? 1u : 0u) << (8 * pass);
                } else {  // single choice: order-free OR
                    u64 *dst = words + (u64)ws.blk[0][kk] * 8 + s;
                    red_or(dst, lo);
                    red_or(dst + 4, hi);
                }
            }
        }
        return found_bytes;
    }
}

// Write the group's four answers (keys 4g..4g+3 of a 32-key tile at `base`)
// and count hits among the first `cnt` keys of the tile.
__device__ __forceinline__ u32 emit_answers(u8 *out, u64 base, u32 cnt, u32 found_bytes,
                                            int lane) {
    const int g = lane >> 2, s = lane & 3;
    const u32 first = 4u * g;
    u32 valid_bytes = 0;
    if (first + 4 <= cnt) {
        valid_bytes = 0x01010101u;
    } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) valid_bytes |= (first + i < cnt ? 1u : 0u) << (8 * i);
    }
    const u32 f = found_bytes & valid_bytes;
    if (out != nullptr && s == 0) {
        u8 *dst = out + base + first;
        if (valid_bytes == 0x01010101u && ((uintptr_t)dst & 3u) == 0) {
            *reinterpret_cast<u32 *>(dst) = f;
        } else {
            for (int i = 0; i < 4; ++i)
                if (first + i < cnt) out[base + first + i] = (u8)((f >> (8 * i)) & 1u);
        }
    }
    return s == 0 ? (u32)__popc(f) : 0u;
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

// Reference insert decision for one key (c >= 2), B = 512 and the random
// strategy: the mask is built in the thread's private shared-memory column
// (col = &column[0][lane], stride 32 words) and read back into registers,
// candidates are read with four L2-coherent LDG.128 each.
__device__ __forceinline__ void insert_fast512(const KParams &p, u64 *words, u64 x, u32 *col) {
#pragma unroll
    for (int w = 0; w < 16; ++w) col[w * 32] = 0u;
    const u32 xlo = (u32)x, xhi = (u32)(x >> 32);
#pragma unroll 4
    for (u32 i = 0; i < p.k; ++i) {
        const u32 h = bit512(p.bit_a_lo[i], p.bit_a_hi[i], xlo, xhi);
        col[(h >> 5) * 32] |= 1u << (h & 31);
    }
    u32 m[16];
#pragma unroll
    for (int w = 0; w < 16; ++w) m[w] = col[w * 32];
    int best = 0;
    u32 best_r = 0xffffffffu;
    for (u32 ci = 0; ci < p.c; ++ci) {
        const uint4 *src = reinterpret_cast<const uint4 *>(words + block_index(p, x, ci) * 8);
        u32 j = 0, pr = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint4 v = ld_block_cg(src + q);
            j += __popc(v.x | m[4 * q]) + __popc(v.y | m[4 * q + 1]) +
                 __popc(v.z | m[4 * q + 2]) + __popc(v.w | m[4 * q + 3]);
            pr += popc4(v);
        }
        const u32 a = j - pr;
        if (a == 0) return;  // no-op: already represented
        const u32 r = __ldg(p.rank + j * (p.k + 1) + a);
        if (r < best_r) {
            best_r = r;
            best = (int)ci;
        }
    }
    u64 *dst = words + block_index(p, x, best) * 8;
#pragma unroll
    for (int w = 0; w < 8; ++w) red_or_all(dst + w, (u64)m[2 * w] | ((u64)m[2 * w + 1] << 32));
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
