// Device-side building blocks shared by every kernel of the hot path.
//
// Hash family (reference: hashing.py:65-100, _kernels.py:61-70):
//   ax = a*x mod 2^64;  MOD_ODD: ax % b;  SHIFT_POW2: (ax >> s) % b (an
//   identity for b = 2^(64-s));  XOR_EVEN: (ax ^ (ax >> 32)) % b.
// The runtime-b modulo is a single-multiply Barrett reduction with the
// precomputed magic floor(2^64/b): the quotient estimate is exact or one too
// small (proof in DESIGN.md §3), so one conditional subtract is exact.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

typedef uint64_t u64;
typedef uint32_t u32;
typedef uint8_t u8;

namespace bc {

enum HashMode : u32 { MOD_ODD = 0, SHIFT_POW2 = 1, XOR_EVEN = 2, ZERO = 3 };

struct DevHash {
    u64 a;      // multiplier
    u64 b;      // range
    u64 magic;  // floor(2^64 / b) for MOD_ODD / XOR_EVEN
    u32 mode;   // HashMode (ZERO: b == 1)
    u32 shift;  // SHIFT_POW2: 64 - log2 b; XOR_EVEN: 32
};

constexpr int kMaxChoices = 8;
constexpr int kMaxFastK = 64;   // bit multipliers passed by value up to this k
constexpr int kMaxWpb = 64;     // generic path: block_bits <= 4096
constexpr int kMaxParts = 16;   // ranks of a partitioned (multi-GPU) build

// Everything a kernel needs about one filter, passed by value (param space).
struct KParams {
    DevHash shard;               // h0 (range T)
    DevHash block;               // range M/T; .a unused (per choice below)
    u64 block_a[kMaxChoices];
    u64 per_shard;               // blocks per shard
    u64 num_blocks;              // M
    u64 flat_b, flat_magic;      // standard kind: range m = M*B
    u32 flat_mode, flat_shift;
    u32 k, c, wpb, strategy, block_bits, fast_random;
    u32 max_ctas;                // launch cap (relaxed inserts: bounds keys in flight)
    const DevHash *bits;         // device, k entries
    const u32 *rank;             // device, (B+1)*(k+1) cost ranks (c >= 2)
    u32 bit_a_lo[kMaxFastK];     // fast_random: SHIFT 55 for every bit hash
    u32 bit_a_hi[kMaxFastK];
};

__device__ __forceinline__ u64 fastmod(u64 v, u64 b, u64 magic) {
    u64 q = __umul64hi(v, magic);
    u64 r = v - q * b;
    return r >= b ? r - b : r;
}

__device__ __forceinline__ u64 hval(u64 a, u64 x, u64 b, u64 magic, u32 mode, u32 shift) {
    u64 ax = a * x;
    if (mode == SHIFT_POW2) return ax >> shift;
    if (mode == ZERO) return 0;
    if (mode == XOR_EVEN) ax ^= ax >> shift;
    return fastmod(ax, b, magic);
}

__device__ __forceinline__ u64 hval(const DevHash &h, u64 x) {
    return hval(h.a, x, h.b, h.magic, h.mode, h.shift);
}

// Global block index of choice ci: h0(x)*(M/T) + h_ci(x)  (_kernels.py:135,143-150).
__device__ __forceinline__ u64 block_index(const KParams &p, u64 x, int ci) {
    u64 sb = p.shard.mode == ZERO ? 0 : hval(p.shard, x) * p.per_shard;
    return sb + hval(p.block_a[ci], x, p.block.b, p.block.magic, p.block.mode, p.block.shift);
}

// Top 9 bits of the low 64 bits of a*x: the SHIFT_POW2 hash with B = 512
// (s = 55), computed from 32-bit halves with three IMADs.
__device__ __forceinline__ u32 mul_hi32(u32 alo, u32 ahi, u32 xlo, u32 xhi) {
    return __umulhi(alo, xlo) + alo * xhi + ahi * xlo;  // bits 32..63 of a*x
}

__device__ __forceinline__ u32 bit512(u32 alo, u32 ahi, u32 xlo, u32 xhi) {
    return mul_hi32(alo, ahi, xlo, xhi) >> 23;
}

// Position of the r-th (0-based) set bit of v (requires r < popc(v)).
__device__ __forceinline__ u32 select_bit32(u32 v, u32 r) {
    u32 pos = 0;
#pragma unroll
    for (int sh = 16; sh >= 1; sh >>= 1) {
        u32 low = __popc(v & ((1u << sh) - 1u));
        if (r >= low) {
            r -= low;
            v >>= sh;
            pos += sh;
        }
    }
    return pos;
}

__device__ __forceinline__ u32 select_bit64(u64 v, u32 r) {
    u32 lo = (u32)v;
    u32 c = __popc(lo);
    if (r < c) return select_bit32(lo, r);
    return 32 + select_bit32((u32)(v >> 32), r - c);
}

// ---- memory access helpers (PTX cache hints) --------------------------------

// Streaming read-only load of a key (evict-first; keys are touched once).
__device__ __forceinline__ u64 ld_stream(const u64 *p) { return __ldcs(p); }

// Read-only gather of 16 bytes of a block that bypasses L1 allocation
// (random blocks have no intra-SM reuse).
__device__ __forceinline__ uint4 ld_block_nc(const uint4 *p) {
    uint4 r;
    asm("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
        : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
        : "l"(p));
    return r;
}

// L2-coherent gather (inserts: other CTAs are OR-ing into the same array).
// The .L2::64B size hint keeps an L2 miss on a random block from being filled
// as a whole 128-byte line: without it the DRAM reads of a random 64-byte
// gather are 2x the data (tools/gather_probe.cu + ncu, profiles/r1).
__device__ __forceinline__ uint4 ld_block_cg(const uint4 *p) {
    uint4 r;
    asm volatile("ld.global.cg.L2::64B.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

// OR a word into global memory (RED, no return value), skipping zero words:
// those still cost L2 atomic throughput, which bounds the L2-resident
// single-choice insert (cfg2: 67.5 Gkeys/s skipped vs 58 unconditional).
__device__ __forceinline__ void red_or(u64 *p, u64 v) {
    if (v) atomicOr((unsigned long long *)p, (unsigned long long)v);
}

// Unconditional RED: where the L2 atomics are not the bound (multi-choice
// inserts wait on DRAM and latency), the branch around each RED (BSSY /
// predicate / branch / BSYNC) costs more than the zero words (cfg5 relaxed
// inserts +10%, cfg3 +4%, cfg1 +5%).
__device__ __forceinline__ void red_or_all(u64 *p, u64 v) {
    atomicOr((unsigned long long *)p, (unsigned long long)v);
}

}  // namespace bc
