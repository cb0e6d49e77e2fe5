// Lookup tile for 512-bit blocks and the random bit strategy
// (contains_blocks, _kernels.py:177-211).
//
// A warp answers 32 keys per iteration:
//
//   1. one lane per key computes the c candidate block indices;
//   2. per choice (in order): four lanes per pending key stage its 64-byte
//      block into the warp's shared-memory slice with one LDG.128 + STS.128
//      each (one L1 wavefront per block, conflict-free 128-bit stores);
//   3. one lane per pending key tests its k bit addresses against the staged
//      block -- a bit hash (3 IMAD) and one shared-memory word per address,
//      no mask is materialised;
//   4. keys found by this choice drop out; the next choice is only fetched
//      for keys still pending, so a positive costs the blocks up to its first
//      passing choice -- the reference's early exit (E[P] blocks, SURVEY
//      §8(d)) rather than all c.
//
// Staging uses cp.async (LDGSTS, .L2::64B: no 128-byte line fill for a
// 64-byte block).  Bit tests take bit (hi >> 23) of the low product word as a
// funnel-shift rotate of word hi >> 28; with k known at compile time
// (K > 0) they are fully unrolled.  Single-choice lookups use PipeStage /
// stage_blocks / test_staged instead: two tiles per warp in flight, the next
// tile's cp.async group outstanding while the current one is tested.
#pragma once

#include "common.cuh"

namespace bc {

template <int C>
struct LookupSmem {
    u32 blk[C][32];            // candidate block per choice and key
    uint4 blocks[32][4];       // staged blocks, row r(kk), 16-byte quarters
};

// Row of key kk: keys 8q+p and 8q+4+p (one quarter-warp of STS.128) land in
// different bank halves, so the staging stores are conflict-free.
__device__ __forceinline__ int stage_row(int kk) { return kk ^ ((kk >> 2) & 1); }

__device__ __forceinline__ u32 staged_bit(const u32 *mine, u32 hi);

template <int C, int K = 0>
__device__ __forceinline__ bool lookup_tile(const KParams &p, const u64 *__restrict__ words,
                                            LookupSmem<C> &ls, u64 x, bool valid, int lane) {
    constexpr u32 full = 0xffffffffu;
#pragma unroll
    for (int ci = 0; ci < C; ++ci) ls.blk[ci][lane] = valid ? (u32)block_index(p, x, ci) : 0u;
    u32 done = __ballot_sync(full, !valid);
    const u32 xlo = (u32)x, xhi = (u32)(x >> 32);
    const int g = lane >> 2, s = lane & 3;
    const uint4 *w4 = reinterpret_cast<const uint4 *>(words);
    const u32 *mine = reinterpret_cast<const u32 *>(&ls.blocks[stage_row(lane)][0]);
    bool found = false;
#pragma unroll
    for (int ci = 0; ci < C; ++ci) {
        if (done == full) break;
        __syncwarp();
        // stage with cp.async (LDGSTS): global -> shared without a register
        // round trip or a separate STS
#pragma unroll
        for (int pp = 0; pp < 4; ++pp) {
            const int kk = 4 * g + pp;
            if (!((done >> kk) & 1u)) {
                const u32 dst = (u32)__cvta_generic_to_shared(&ls.blocks[stage_row(kk)][s]);
                asm volatile("cp.async.cg.shared.global.L2::64B [%0], [%1], 16;" ::"r"(dst),
                             "l"(w4 + (u64)ls.blk[ci][kk] * 4 + s));
            }
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncwarp();
        if (!((done >> lane) & 1u)) {
            u32 acc = 1u;
            if (K > 0) {
#pragma unroll
                for (int i = 0; i < K; ++i)
                    acc &= staged_bit(mine, mul_hi32(p.bit_a_lo[i], p.bit_a_hi[i], xlo, xhi));
            } else {
#pragma unroll 4
                for (u32 i = 0; i < p.k; ++i)
                    acc &= staged_bit(mine, mul_hi32(p.bit_a_lo[i], p.bit_a_hi[i], xlo, xhi));
            }
            found = (acc & 1u) != 0u;
        }
        done |= __ballot_sync(full, found);
    }
    return found;
}

// ---- single choice, software-pipelined ---------------------------------------------
// With one choice there is no early exit to wait for, so a warp can keep two
// tiles in flight: the block fetch of tile t+1 (one cp.async group into the
// other stage) is outstanding while tile t is tested.  Block numbers reach the
// copying lanes by shuffle instead of a shared-memory round trip.
struct PipeStage {
    uint4 blocks[32][4];
};

__device__ __forceinline__ void stage_blocks(const u64 *__restrict__ words, PipeStage &st,
                                             u32 blk, u32 live, int lane) {
    const int g = lane >> 2, s = lane & 3;
    const uint4 *w4 = reinterpret_cast<const uint4 *>(words);
#pragma unroll
    for (int pp = 0; pp < 4; ++pp) {
        const int kk = 4 * g + pp;
        const u32 b = __shfl_sync(0xffffffffu, blk, kk);
        if ((live >> kk) & 1u) {
            const u32 dst = (u32)__cvta_generic_to_shared(&st.blocks[stage_row(kk)][s]);
            asm volatile("cp.async.cg.shared.global.L2::64B [%0], [%1], 16;" ::"r"(dst),
                         "l"(w4 + (u64)b * 4 + s));
        }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
}

// Bit h = hi >> 23 of the staged block, moved to bit 0: word hi >> 28 rotated
// right by (hi >> 23) & 31 (the funnel shift's wrap mode does the & 31).
__device__ __forceinline__ u32 staged_bit(const u32 *mine, u32 hi) {
    const u32 w = mine[hi >> 28];
    return __funnelshift_r(w, w, hi >> 23);
}

// All k bits of key x set in this lane's staged block?  K > 0: k known at
// compile time (fully unrolled); K == 0: runtime k.
template <int K>
__device__ __forceinline__ bool test_staged(const KParams &p, const PipeStage &st, u64 x,
                                            int lane) {
    const u32 xlo = (u32)x, xhi = (u32)(x >> 32);
    const u32 *mine = reinterpret_cast<const u32 *>(&st.blocks[stage_row(lane)][0]);
    u32 acc = 1u;
    if (K > 0) {
#pragma unroll
        for (int i = 0; i < K; ++i)
            acc &= staged_bit(mine, mul_hi32(p.bit_a_lo[i], p.bit_a_hi[i], xlo, xhi));
    } else {
#pragma unroll 4
        for (u32 i = 0; i < p.k; ++i)
            acc &= staged_bit(mine, mul_hi32(p.bit_a_lo[i], p.bit_a_hi[i], xlo, xhi));
    }
    return (acc & 1u) != 0u;
}

}  // namespace bc
