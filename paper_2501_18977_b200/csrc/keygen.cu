// Device generation of the reference's key streams.
//
// The reference draws keys with numpy: even_keys / odd_keys are
// default_rng(seed).integers(0, 2**64, n, uint64) with the low bit cleared /
// set (analysis.py:34-43).  For the full 64-bit range numpy returns the raw
// PCG64 outputs: state <- state * M + inc (mod 2^128), output =
// rotr64(hi ^ lo, hi >> 58) of the new state.  The seeded (state, inc) pair
// comes from numpy on the host (SeedSequence); here every thread jumps the
// LCG to the start of its run in O(log n) steps and then walks it, so the
// device stream is bit-identical to numpy's at any length.
#include "common.cuh"
#include "launch.h"

namespace bc {

struct U128 {
    u64 hi, lo;
};

__device__ __forceinline__ U128 mul128(U128 a, U128 b) {
    U128 r;
    r.lo = a.lo * b.lo;
    r.hi = __umul64hi(a.lo, b.lo) + a.lo * b.hi + a.hi * b.lo;
    return r;
}

__device__ __forceinline__ U128 add128(U128 a, U128 b) {
    U128 r;
    r.lo = a.lo + b.lo;
    r.hi = a.hi + b.hi + (r.lo < a.lo ? 1ull : 0ull);
    return r;
}

__device__ __forceinline__ u64 xsl_rr(U128 s) {
    const u64 x = s.hi ^ s.lo;
    const u32 rot = (u32)(s.hi >> 58);
    return (x >> rot) | (x << ((64u - rot) & 63u));
}

constexpr u64 kMulHi = 0x2360ED051FC65DA4ull, kMulLo = 0x4385DF649FCCF645ull;
constexpr int kRun = 64;  // outputs per thread run

__global__ void __launch_bounds__(256) pcg64_fill_kernel(U128 state0, U128 inc, u64 offset,
                                                         u64 n, u64 and_mask, u64 or_mask,
                                                         u64 *__restrict__ out) {
    const U128 mult = {kMulHi, kMulLo};
    const u64 runs = (n + kRun - 1) / kRun;
    for (u64 r = blockIdx.x * (u64)blockDim.x + threadIdx.x; r < runs;
         r += (u64)gridDim.x * blockDim.x) {
        // jump the LCG by offset + r*kRun steps
        u64 delta = offset + r * kRun;
        U128 acc_m = {0, 1}, acc_p = {0, 0}, cur_m = mult, cur_p = inc;
        while (delta) {
            if (delta & 1) {
                acc_m = mul128(acc_m, cur_m);
                acc_p = add128(mul128(acc_p, cur_m), cur_p);
            }
            cur_p = mul128(add128(cur_m, U128{0, 1}), cur_p);
            cur_m = mul128(cur_m, cur_m);
            delta >>= 1;
        }
        U128 s = add128(mul128(acc_m, state0), acc_p);
        const u64 i0 = r * kRun;
        const u64 cnt = min((u64)kRun, n - i0);
        for (u64 j = 0; j < cnt; ++j) {
            s = add128(mul128(s, mult), inc);
            out[i0 + j] = (xsl_rr(s) & and_mask) | or_mask;
        }
    }
}

cudaError_t launch_pcg64_fill(u64 state_hi, u64 state_lo, u64 inc_hi, u64 inc_lo, u64 offset,
                              u64 n, u64 and_mask, u64 or_mask, u64 *out, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const u64 runs = (n + kRun - 1) / kRun;
    const unsigned grid = grid_for((const void *)pcg64_fill_kernel, 256, 0, (runs + 255) / 256);
    pcg64_fill_kernel<<<grid, 256, 0, s>>>(U128{state_hi, state_lo}, U128{inc_hi, inc_lo}, offset,
                                           n, and_mask, or_mask, out);
    count_launch();
    return cudaGetLastError();
}

}  // namespace bc
