// Key sources of the exact-order insert (ordered512_kernel): where the keys
// that enter the claim window come from.
//
//   ArrayKeys  a uint64 key array (insert_many, filters.py:377-385)
//   SeqKeys    the q-gram windows of a DNA byte sequence, encoded on the fly
//              (insert_many(encode_qgrams(enc, seq)), io.py:158-177): key i
//              is window i, so the window index is the stream-order priority
//              and windows the reference skips never enter the window.  The
//              key array of the two-pass design is never materialised.
//
// admit(i, x) returns false for an index that yields no key (a skipped
// window); the stream order of the keys that remain is the index order.
#pragma once

#include "common.cuh"
#include "launch.h"

namespace bc {

struct ArrayKeys {
    static constexpr bool kCounts = false;
    const u64 *keys;
    __device__ __forceinline__ bool admit(u64 i, u64 &x) const {
        x = __ldcs(keys + i);
        return true;
    }
    // the same stream from key `off` on
    __host__ __device__ void advance(u64 off) { keys += off; }
};

// 0x80 in every byte of b that is not one of A C G T a c g t.
__device__ __forceinline__ u64 non_base_bytes(u64 b) {
    constexpr u64 lo7 = 0x7F7F7F7F7F7F7F7Full;
    const u64 u = b & 0xDFDFDFDFDFDFDFDFull;  // upper case (clears bit 5 only)
    u64 hit = 0;
    // exact zero-byte test of u ^ letter (no carries between bytes)
#define BC_ZERO_BYTES(pat)                                    \
    {                                                         \
        const u64 t = u ^ (pat);                              \
        hit |= ~(((t & lo7) + lo7) | t | lo7);                \
    }
    BC_ZERO_BYTES(0x4141414141414141ull)
    BC_ZERO_BYTES(0x4343434343434343ull)
    BC_ZERO_BYTES(0x4747474747474747ull)
    BC_ZERO_BYTES(0x5454545454545454ull)
#undef BC_ZERO_BYTES
    return ~hit & 0x8080808080808080ull;
}

// 2-bit codes held one per byte (0..3) -> 16 bits, byte 0 least significant.
__device__ __forceinline__ u64 pack_codes8(u64 c) {
    c = (c | (c >> 6)) & 0x000F000F000F000Full;
    c = (c | (c >> 12)) & 0x000000FF000000FFull;
    return (c | (c >> 24)) & 0xFFFFull;
}

struct SeqKeys {
    static constexpr bool kCounts = true;
    const u8 *seq;  // window i starts at seq[i]
    RecSpec rec;
    u64 qmask;      // low 2q bits
    u32 q;
    u32 canonical;

    // the same stream from window `off` on
    __host__ __device__ void advance(u64 off) {
        seq += off;
        if (rec.len) rec.phase = (rec.phase + off) % rec.len;
    }

    // Window w's key: A=0 C=1 G=2 T=3 (either case), first base most
    // significant, canonical = min(code, reverse complement) -- the
    // reference's encode_qgrams (io.py:126-177), as the rolling encoder of
    // qgram_kernels.cu computes it; here each window is encoded from its own
    // q bytes (four aligned 8-byte words, SWAR), so any window can be
    // (re)derived independently.
    __device__ __forceinline__ bool admit(u64 w, u64 &x) const {
        if (rec.len) {
            const u64 r = (w + rec.phase) % rec.len;
            if (r + q > rec.len) return false;  // crosses a record boundary
        }
        const uintptr_t a = reinterpret_cast<uintptr_t>(seq + w);
        const u32 o = (u32)(a & 7u);
        const u64 *base = reinterpret_cast<const u64 *>(a - o);
        const u32 last = o + q - 1;  // last window byte, relative to base
        // only words holding window bytes are read (an aligned word with one
        // byte inside the sequence lies in mapped memory)
        u64 A[5];
#pragma unroll
        for (int i = 0; i < 5; ++i) A[i] = (8u * i <= last) ? __ldg(base + i) : 0ull;
        const u32 sh = 8u * o;
        u64 bad = 0, P = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const u64 B = sh ? (A[i] >> sh) | (A[i + 1] << (64u - sh)) : A[i];
            const u32 nb = q > 8u * i ? min(8u, q - 8u * i) : 0u;
            const u64 keep = nb >= 8 ? ~0ull : ((1ull << (8u * nb)) - 1ull);
            bad |= non_base_bytes(B) & keep;
            const u64 c = ((B >> 1) ^ (B >> 2)) & 0x0303030303030303ull & keep;
            P |= pack_codes8(c) << (16 * i);
        }
        if (bad) return false;
        // P: base t at bits 2t..2t+1 (first base least significant).  Its
        // complement is the reverse complement; reversing the 2-bit groups
        // gives the forward code.
        const u64 rc = P ^ qmask;
        u64 r = __brevll(P);
        r = ((r >> 1) & 0x5555555555555555ull) | ((r & 0x5555555555555555ull) << 1);
        const u64 fw = r >> (64u - 2u * q);
        x = (canonical && rc < fw) ? rc : fw;
        return true;
    }
};

}  // namespace bc
