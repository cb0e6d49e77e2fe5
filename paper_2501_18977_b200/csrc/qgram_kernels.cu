// DNA q-gram path (reference: io.py:126-177 feeding filters.py:377-398).
//
// A tile of kQgramTile consecutive windows is staged per CTA iteration: the
// tile's bytes go to shared memory, each thread rolls kQgramPerThread
// consecutive windows (2-bit forward code, reverse complement, run length of
// valid bases), the valid windows of the tile are compacted in order with a
// CTA scan, and the compacted keys then flow through the same two-phase
// hash/probe pipeline as key arrays (blocks.cuh).  The key array of the
// reference's two-pass design (encode_qgrams, then insert_many) is never
// written to HBM.
//
// Encoding rules (io.py:126-177): A=0 C=1 G=2 T=3 (lower case too), first
// base most significant; a window touching any other byte is skipped;
// canonical = min(code, reverse complement).
#include "blocks.cuh"
#include "lookup.cuh"

namespace bc {

struct QgramSmem {
    u8 bytes[kQgramTile + 32];
    u64 keys[kQgramTile];
    u32 warp_tot[kQgramThreads / 32];
};

// bit i set for i = ('A','C','G','T','a','c','g','t') & 63
constexpr u64 kBaseMask = (1ull << 1) | (1ull << 3) | (1ull << 7) | (1ull << 20) | (1ull << 33) |
                          (1ull << 35) | (1ull << 39) | (1ull << 52);

struct Roller {
    u64 fw = 0, rc = 0, qmask;
    u32 run = 0, rshift;
    __device__ __forceinline__ Roller(int q)
        : qmask(q == 32 ? ~0ull : ((1ull << (2 * q)) - 1)), rshift(2 * q - 2) {}
    __device__ __forceinline__ void step(u32 b) {
        const u32 code = ((b >> 1) ^ (b >> 2)) & 3u;
        const bool ok = ((b >> 6) == 1u) && ((kBaseMask >> (b & 63u)) & 1ull);
        run = ok ? run + 1 : 0u;
        fw = ((fw << 2) | code) & qmask;
        rc = (rc >> 2) | ((u64)(3u - code) << rshift);
    }
};

// Stage, roll and compact one tile; returns the number of valid windows,
// whose keys are left in order in sm.keys[0..V).
// With records (rec.len > 0) a window is also invalid when it crosses a record
// boundary.
__device__ __forceinline__ u32 in_record_mask(u64 wfirst, int q, RecSpec rec) {
    if (rec.len == 0) return (1u << kQgramPerThread) - 1u;
    u64 r = (wfirst + rec.phase) % rec.len;
    u32 m = 0;
#pragma unroll
    for (int k = 0; k < kQgramPerThread; ++k) {
        m |= (r + (u64)q <= rec.len ? 1u : 0u) << k;
        r = r + 1 == rec.len ? 0 : r + 1;
    }
    return m;
}

__device__ __forceinline__ u32 tile_encode(const u8 *__restrict__ seq, u64 len, int q,
                                           int canonical, RecSpec rec, u64 w0, u64 nwin,
                                           QgramSmem &sm) {
    const int tid = threadIdx.x;
    const u64 nbytes_avail = len - w0;  // w0 < nwin <= len
    const int nbytes = kQgramTile + q - 1;
    for (int i = tid; i < nbytes; i += kQgramThreads)
        sm.bytes[i] = (u64)i < nbytes_avail ? __ldcs(seq + w0 + i) : (u8)'N';
    __syncthreads();

    Roller r(q);
    const u8 *b = sm.bytes + kQgramPerThread * tid;
    for (int j = 0; j < q - 1; ++j) r.step(b[j]);
    u64 code[kQgramPerThread];
    u32 vmask = 0;
    const u64 wfirst = w0 + (u64)kQgramPerThread * tid;
#pragma unroll
    for (int k = 0; k < kQgramPerThread; ++k) {
        r.step(b[q - 1 + k]);
        const bool v = r.run >= (u32)q && wfirst + k < nwin;
        code[k] = (canonical && r.rc < r.fw) ? r.rc : r.fw;
        vmask |= (v ? 1u : 0u) << k;
    }
    vmask &= in_record_mask(wfirst, q, rec);
    // CTA exclusive scan of the per-thread valid counts
    const u32 mine = __popc(vmask);
    u32 incl = mine;
    const int lane = tid & 31, warp = tid >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        u32 t = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) sm.warp_tot[warp] = incl;
    __syncthreads();
    u32 before = 0, total = 0;
#pragma unroll
    for (int w = 0; w < kQgramThreads / 32; ++w) {
        const u32 t = sm.warp_tot[w];
        before += w < warp ? t : 0u;
        total += t;
    }
    u32 pos = before + incl - mine;
#pragma unroll
    for (int k = 0; k < kQgramPerThread; ++k)
        if (vmask & (1u << k)) sm.keys[pos++] = code[k];
    __syncthreads();
    return total;
}

__global__ void __launch_bounds__(kQgramThreads) qgram_count_kernel(const u8 *__restrict__ seq,
                                                                    u64 len, int q, RecSpec rec,
                                                                    u64 nwin, u64 ntiles,
                                                                    u64 *__restrict__ counts) {
    __shared__ u8 bytes[kQgramTile + 32];
    __shared__ u32 warp_tot[kQgramThreads / 32];
    const int tid = threadIdx.x;
    for (u64 tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const u64 w0 = tile * kQgramTile;
        const int nbytes = kQgramTile + q - 1;
        for (int i = tid; i < nbytes; i += kQgramThreads)
            bytes[i] = (u64)i < len - w0 ? __ldcs(seq + w0 + i) : (u8)'N';
        __syncthreads();
        Roller r(q);
        const u8 *b = bytes + kQgramPerThread * tid;
        for (int j = 0; j < q - 1; ++j) r.step(b[j]);
        u32 vmask = 0;
        const u64 wfirst = w0 + (u64)kQgramPerThread * tid;
#pragma unroll
        for (int k = 0; k < kQgramPerThread; ++k) {
            r.step(b[q - 1 + k]);
            vmask |= ((r.run >= (u32)q && wfirst + k < nwin) ? 1u : 0u) << k;
        }
        u32 mine = __popc(vmask & in_record_mask(wfirst, q, rec));
        for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(kFull, mine, o);
        if ((tid & 31) == 0) warp_tot[tid >> 5] = mine;
        __syncthreads();
        if (tid == 0) {
            u64 t = 0;
            for (int w = 0; w < kQgramThreads / 32; ++w) t += warp_tot[w];
            counts[tile] = t;
        }
        __syncthreads();
    }
}

// In-place exclusive scan of n u64 values by one CTA; *total = sum.
__global__ void __launch_bounds__(1024) scan_kernel(u64 *__restrict__ v, u64 n,
                                                    unsigned long long *__restrict__ total) {
    __shared__ u64 warp_tot[32];
    __shared__ u64 carry;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) carry = 0;
    __syncthreads();
    for (u64 base = 0; base < n; base += 1024) {
        const u64 i = base + tid;
        const u64 x = i < n ? v[i] : 0ull;
        u64 incl = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            u64 t = __shfl_up_sync(kFull, incl, o);
            if (lane >= o) incl += t;
        }
        if (lane == 31) warp_tot[warp] = incl;
        __syncthreads();
        u64 before = carry, tot = 0;
        for (int w = 0; w < 32; ++w) {
            before += w < warp ? warp_tot[w] : 0ull;
            tot += warp_tot[w];
        }
        if (i < n) v[i] = before + incl - x;
        __syncthreads();
        if (tid == 0) carry += tot;
        __syncthreads();
    }
    if (tid == 0 && total) *total = carry;
}

__global__ void __launch_bounds__(kQgramThreads) qgram_encode_kernel(
    const u8 *__restrict__ seq, u64 len, int q, int canonical, RecSpec rec, u64 nwin, u64 ntiles,
    const u64 *__restrict__ tile_off, u64 *__restrict__ keys) {
    __shared__ QgramSmem sm;
    for (u64 tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const u32 v = tile_encode(seq, len, q, canonical, rec, tile * kQgramTile, nwin, sm);
        const u64 base = tile_off[tile];
        for (u32 i = threadIdx.x; i < v; i += kQgramThreads) keys[base + i] = sm.keys[i];
        __syncthreads();
    }
}

template <int OP, int C>
__global__ void __launch_bounds__(kQgramThreads) qgram_blocks_kernel(
    const __grid_constant__ KParams p, u64 *__restrict__ words, const u8 *__restrict__ seq,
    u64 len, int q, int canonical, RecSpec rec, u64 nwin, u64 ntiles,
    const u64 *__restrict__ tile_off, u8 *__restrict__ out, unsigned long long *__restrict__ hits,
    unsigned long long *__restrict__ count) {
    static_assert(kQgramThreads == kTPB, "tile pipeline assumes the CTA shape of blocks.cuh");
    __shared__ QgramSmem qs;
    __shared__ WarpSmem<C> smem[kWarps];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    WarpSmem<C> &ws = smem[warp];
    u32 my_hits = 0;
    for (u64 tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const u32 v = tile_encode(seq, len, q, canonical, rec, tile * kQgramTile, nwin, qs);
        const u64 obase = (OP == OP_CONTAINS && tile_off) ? tile_off[tile] : 0ull;
        if (count != nullptr && tid == 0 && v) atomicAdd(count, (unsigned long long)v);
        // each warp takes 32 consecutive compacted keys at a time
        for (u32 sub = 32u * warp; sub < v; sub += 32u * kWarps) {
            const u32 cnt = min(32u, v - sub);
            const bool valid = (u32)lane < cnt;
            phase1<C>(p, valid ? qs.keys[sub + lane] : 0ull, valid, ws, lane);
            __syncwarp();
            const u32 found = phase2<OP, C>(p, words, ws, lane);
            if (OP == OP_CONTAINS) my_hits += emit_answers(out, obase + sub, cnt, found, lane);
            __syncwarp();
        }
        __syncthreads();
    }
    if (OP == OP_CONTAINS && hits != nullptr) {
        for (int o = 16; o > 0; o >>= 1) my_hits += __shfl_xor_sync(kFull, my_hits, o);
        if (lane == 0 && my_hits) atomicAdd(hits, (unsigned long long)my_hits);
    }
}

// Lookups with the random strategy: the compacted keys go through the
// staged-block tile with early exit over the choices (lookup.cuh).
template <int C, int K>
__global__ void __launch_bounds__(kQgramThreads) qgram_lookup_kernel(
    const __grid_constant__ KParams p, const u64 *__restrict__ words, const u8 *__restrict__ seq,
    u64 len, int q, int canonical, RecSpec rec, u64 nwin, u64 ntiles,
    const u64 *__restrict__ tile_off, u8 *__restrict__ out, unsigned long long *__restrict__ hits) {
    __shared__ QgramSmem qs;
    __shared__ LookupSmem<C> smem[kWarps];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    LookupSmem<C> &ls = smem[warp];
    u32 my_hits = 0;
    for (u64 tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const u32 v = tile_encode(seq, len, q, canonical, rec, tile * kQgramTile, nwin, qs);
        const u64 obase = tile_off ? tile_off[tile] : 0ull;
        for (u32 sub = 32u * warp; sub < v; sub += 32u * kWarps) {
            const bool valid = sub + lane < v;
            const bool f = lookup_tile<C, K>(p, words, ls, valid ? qs.keys[sub + lane] : 0ull,
                                             valid, lane);
            if (out != nullptr && valid) out[obase + sub + lane] = (u8)f;
            my_hits += f ? 1u : 0u;
            __syncwarp();
        }
        __syncthreads();
    }
    if (hits != nullptr) {
        for (int o = 16; o > 0; o >>= 1) my_hits += __shfl_xor_sync(kFull, my_hits, o);
        if (lane == 0 && my_hits) atomicAdd(hits, (unsigned long long)my_hits);
    }
}

cudaError_t launch_scan(u64 *v, u64 n, unsigned long long *total, cudaStream_t s) {
    scan_kernel<<<1, 1024, 0, s>>>(v, n, total);
    count_launch();
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------------
static inline u64 n_windows(u64 len, int q) { return len >= (u64)q ? len - q + 1 : 0; }

cudaError_t launch_qgram_offsets(const u8 *seq, u64 len, int q, RecSpec rec, u64 *tile_off,
                                 u64 ntiles, unsigned long long *total, cudaStream_t s) {
    const u64 nwin = n_windows(len, q);
    if (nwin == 0) {
        if (total) return cudaMemsetAsync(total, 0, sizeof(*total), s);
        return cudaSuccess;
    }
    const unsigned grid = grid_for((const void *)qgram_count_kernel, kQgramThreads, 0, ntiles);
    qgram_count_kernel<<<grid, kQgramThreads, 0, s>>>(seq, len, q, rec, nwin, ntiles, tile_off);
    scan_kernel<<<1, 1024, 0, s>>>(tile_off, ntiles, total);
    count_launch(2);
    return cudaGetLastError();
}

cudaError_t launch_qgram_encode(const u8 *seq, u64 len, int q, int canonical, RecSpec rec,
                                const u64 *tile_off, u64 *keys, cudaStream_t s) {
    const u64 nwin = n_windows(len, q);
    if (nwin == 0) return cudaSuccess;
    const u64 ntiles = (nwin + kQgramTile - 1) / kQgramTile;
    const unsigned grid = grid_for((const void *)qgram_encode_kernel, kQgramThreads, 0, ntiles);
    qgram_encode_kernel<<<grid, kQgramThreads, 0, s>>>(seq, len, q, canonical, rec, nwin,
                                                       ntiles, tile_off, keys);
    count_launch();
    return cudaGetLastError();
}

template <int C, int K>
static cudaError_t launch_qgram_lookup_k(const KParams &p, const u64 *words, const u8 *seq,
                                         u64 len, int q, int canonical, RecSpec rec, u64 nwin,
                                         u64 ntiles, const u64 *tile_off, u8 *out,
                                         unsigned long long *hits, cudaStream_t s) {
    const void *fl = (const void *)qgram_lookup_kernel<C, K>;
    const unsigned g = grid_for(fl, kQgramThreads, 0, ntiles);
    qgram_lookup_kernel<C, K><<<g, kQgramThreads, 0, s>>>(p, words, seq, len, q, canonical, rec,
                                                          nwin, ntiles, tile_off, out, hits);
    count_launch();
    return cudaGetLastError();
}

// compile-time k (4..16) for one to three choices, as for key arrays
template <int C>
static cudaError_t launch_qgram_lookup(const KParams &p, const u64 *words, const u8 *seq,
                                       u64 len, int q, int canonical, RecSpec rec, u64 nwin,
                                       u64 ntiles, const u64 *tile_off, u8 *out,
                                       unsigned long long *hits, cudaStream_t s) {
    if (C <= 3) {
        switch (p.k) {
#define BC_QL_K(k)                                                                          \
    case k:                                                                                 \
        return launch_qgram_lookup_k<C, (C <= 3 ? k : 0)>(p, words, seq, len, q, canonical, \
                                                          rec, nwin, ntiles, tile_off, out,  \
                                                          hits, s);
            BC_QL_K(4) BC_QL_K(5) BC_QL_K(6) BC_QL_K(7) BC_QL_K(8) BC_QL_K(9) BC_QL_K(10)
            BC_QL_K(11) BC_QL_K(12) BC_QL_K(13) BC_QL_K(14) BC_QL_K(15) BC_QL_K(16)
#undef BC_QL_K
            default: break;
        }
    }
    return launch_qgram_lookup_k<C, 0>(p, words, seq, len, q, canonical, rec, nwin, ntiles,
                                       tile_off, out, hits, s);
}

template <int OP, int C>
static cudaError_t launch_qb(const KParams &p, u64 *words, const u8 *seq, u64 len, int q,
                             int canonical, RecSpec rec, const u64 *tile_off, u8 *out,
                             unsigned long long *hits, unsigned long long *count,
                             cudaStream_t s) {
    const u64 nwin = n_windows(len, q);
    if (nwin == 0) return cudaSuccess;
    const u64 ntiles = (nwin + kQgramTile - 1) / kQgramTile;
    if (OP == OP_CONTAINS && p.fast_random && count == nullptr)
        return launch_qgram_lookup<C>(p, words, seq, len, q, canonical, rec, nwin, ntiles,
                                      tile_off, out, hits, s);
    const void *fn = (const void *)qgram_blocks_kernel<OP, C>;
    const unsigned grid = grid_for(fn, kQgramThreads, 0, ntiles);
    qgram_blocks_kernel<OP, C><<<grid, kQgramThreads, 0, s>>>(p, words, seq, len, q, canonical,
                                                               rec, nwin, ntiles, tile_off, out,
                                                               hits, count);
    count_launch();
    return cudaGetLastError();
}

template <int OP>
static cudaError_t launch_qb_c(const KParams &p, u64 *words, const u8 *seq, u64 len, int q,
                               int canonical, RecSpec rec, const u64 *tile_off, u8 *out,
                               unsigned long long *hits, unsigned long long *count,
                               cudaStream_t s) {
    switch (p.c) {
        case 1: return launch_qb<OP, 1>(p, words, seq, len, q, canonical, rec, tile_off, out, hits, count, s);
        case 2: return launch_qb<OP, 2>(p, words, seq, len, q, canonical, rec, tile_off, out, hits, count, s);
        case 3: return launch_qb<OP, 3>(p, words, seq, len, q, canonical, rec, tile_off, out, hits, count, s);
        case 4: return launch_qb<OP, 4>(p, words, seq, len, q, canonical, rec, tile_off, out, hits, count, s);
        case 5: return launch_qb<OP, 5>(p, words, seq, len, q, canonical, rec, tile_off, out, hits, count, s);
        case 6: return launch_qb<OP, 6>(p, words, seq, len, q, canonical, rec, tile_off, out, hits, count, s);
        case 7: return launch_qb<OP, 7>(p, words, seq, len, q, canonical, rec, tile_off, out, hits, count, s);
        case 8: return launch_qb<OP, 8>(p, words, seq, len, q, canonical, rec, tile_off, out, hits, count, s);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_qgram_blocks(int op, const KParams &p, u64 *words, const u8 *seq, u64 len,
                                int q, int canonical, RecSpec rec, const u64 *tile_off, u8 *out,
                                unsigned long long *hits, unsigned long long *count,
                                cudaStream_t s) {
    if (p.wpb != 8) return cudaErrorInvalidValue;  // caller falls back to encode + array path
    l2_release();
    return op == OP_CONTAINS ? launch_qb_c<OP_CONTAINS>(p, words, seq, len, q, canonical, rec,
                                                        tile_off, out, hits, count, s)
                             : launch_qb_c<OP_INSERT>(p, words, seq, len, q, canonical, rec,
                                                      tile_off, out, hits, count, s);
}

}  // namespace bc
