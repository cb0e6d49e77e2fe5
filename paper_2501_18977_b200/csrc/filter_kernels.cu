// Kernels of the blocked / blowchoc / standard filter hot path.
//
//   blocks512_kernel<OP, C>  key array -> lookup answers or inserts, 512-bit
//                            blocks, two-phase tile (blocks.cuh)
//   generic_kernel<OP>       thread per key, any block width (toy 8/16/32,
//                            64..4096 bits)
//   relaxed512_kernel<C>     relaxed (atomic) multi-choice inserts, next
//                            tile's hashing overlapped with the loads
//   lookup512_kernel<C, K>   lookups: staged blocks, early exit over choices
//   lookup512_pipe_kernel<K> single-choice lookups, two tiles in flight
//   ordered1_kernel<C,Src>   exact stream-order insert for c >= 2, 512-bit
//                            blocks: claim rounds over a sliding window, one
//                            cooperative launch, one array of epoch-tagged
//                            claims, one grid sync per round, winners
//                            committed a warp tile at a time; keys from an
//                            array or encoded from a DNA sequence on the fly
//                            (keysrc.cuh)
//   ordered512_kernel<C,Src> its predecessor (BC_ORDERED_ONE=0): two claim
//                            arrays, claims reset by the winners' atomicCAS
//   ordered_window_kernel    the same rounds for any geometry, thread-per-key
//                            commits (ordered_kernel: fixed-chunk variant)
//   flat_kernel<OP>          standard Bloom filter (k global bits)
//   hist512_kernel / hist_generic_kernel   per-block popcount tally
//   eval_hash_kernel         one hash over a key array (routing)
#include <cooperative_groups.h>

#include <atomic>
#include <cstdio>
#include <mutex>
#include <unordered_map>

#include "blocks.cuh"
#include "keysrc.cuh"
#include "lookup.cuh"

namespace cg = cooperative_groups;

namespace bc {

static std::atomic<unsigned long long> g_launches{0};

void count_launch(unsigned n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

unsigned long long launch_count() { return g_launches.load(std::memory_order_relaxed); }

static int sm_count() {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms > 0 ? sms : 1;
}

unsigned grid_for(const void *kernel, int threads, size_t dyn_smem,
                  unsigned long long work_ctas) {
    static std::mutex mu;
    static std::unordered_map<const void *, int> occ;
    int per_sm = 0;
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = occ.find(kernel);
        if (it == occ.end()) {
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads,
                                                              dyn_smem) != cudaSuccess ||
                per_sm < 1)
                per_sm = 1;
            occ[kernel] = per_sm;
        } else {
            per_sm = it->second;
        }
    }
    unsigned long long cap = (unsigned long long)per_sm * (unsigned long long)sm_count();
    if (work_ctas < 1) work_ctas = 1;
    return (unsigned)(work_ctas < cap ? work_ctas : cap);
}

// ---------------------------------------------------------------------------------
template <int OP, int C>
__global__ void __launch_bounds__(kTPB) blocks512_kernel(const __grid_constant__ KParams p,
                                                         u64 *__restrict__ words,
                                                         const u64 *__restrict__ keys, u64 n,
                                                         u8 *__restrict__ out,
                                                         unsigned long long *__restrict__ hits) {
    __shared__ WarpSmem<C> smem[kWarps];
    WarpSmem<C> &ws = smem[threadIdx.x >> 5];
    const int lane = threadIdx.x & 31;
    const u64 ntiles = (n + 31) / 32;
    const u64 nwarps = (u64)gridDim.x * kWarps;
    u32 my_hits = 0;
    u64 tile = blockIdx.x * (u64)kWarps + (threadIdx.x >> 5);
    // the next tile's key is loaded while the current tile is processed
    u64 x_next = tile * 32 + lane < n ? ld_stream(keys + tile * 32 + lane) : 0ull;
    for (; tile < ntiles; tile += nwarps) {
        const u64 base = tile * 32;
        const u32 cnt = (u32)min((u64)32, n - base);
        const bool valid = (u32)lane < cnt;
        const u64 x = x_next;
        const u64 nb = base + nwarps * 32 + lane;
        x_next = nb < n ? ld_stream(keys + nb) : 0ull;
        phase1<C>(p, x, valid, ws, lane);
        __syncwarp();
        const u32 found = phase2<OP, C>(p, words, ws, lane);
        if (OP == OP_CONTAINS) my_hits += emit_answers(out, base, cnt, found, lane);
        __syncwarp();
    }
    if (OP == OP_CONTAINS && hits != nullptr) {
        for (int o = 16; o > 0; o >>= 1) my_hits += __shfl_xor_sync(kFull, my_hits, o);
        if (lane == 0 && my_hits) atomicAdd(hits, (unsigned long long)my_hits);
    }
}

// Relaxed multi-choice inserts, 512-bit blocks: the two-phase tile with the
// next tile's phase 1 (hashing, mask build -- no filter reads, so those keys
// are not yet in flight) issued while the current tile's candidate loads are
// outstanding.  Double-buffered warp slices.
template <int C, class A>
__device__ __forceinline__ void relaxed512_loop(const KParams &p, const A &a,
                                                const u64 *__restrict__ keys, u64 n) {
    constexpr int UNR = relaxed_unroll(C);
    __shared__ WarpSmem<C> smem[kWarps][2];
    WarpSmem<C> *ws = smem[threadIdx.x >> 5];
    const int lane = threadIdx.x & 31;
    const u64 ntiles = (n + 31) / 32;
    const u64 nwarps = (u64)gridDim.x * kWarps;
    u64 tile = blockIdx.x * (u64)kWarps + (threadIdx.x >> 5);
    if (tile >= ntiles) return;
    u64 i = tile * 32 + lane;
    phase1<C>(p, i < n ? ld_stream(keys + i) : 0ull, i < n, ws[0], lane);
    i = (tile + nwarps) * 32 + lane;
    u64 x_next = i < n ? ld_stream(keys + i) : 0ull;
    int b = 0;
    for (; tile < ntiles; tile += nwarps) {
        __syncwarp();
        const WarpSmem<C> &cur = ws[b];
        uint4 M[4];
        read_masks<C>(cur, lane, false, M);
        uint4 w[UNR][C];
        relaxed_load<C, UNR>(cur, a, lane, 0, w);
        // the next tile's phase 1 while the loads are in flight
        const u64 nt = tile + nwarps;
        const bool vn = nt * 32 + lane < n;
        phase1<C>(p, x_next, vn, ws[b ^ 1], lane);
        i = (nt + nwarps) * 32 + lane;
        x_next = i < n ? ld_stream(keys + i) : 0ull;
        relaxed_commit<C, UNR>(p, a, cur, M, lane, 0, w);
#pragma unroll
        for (int p0 = UNR; p0 < 4; p0 += UNR) {
            relaxed_load<C, UNR>(cur, a, lane, p0, w);
            relaxed_commit<C, UNR>(p, a, cur, M, lane, p0, w);
        }
        b ^= 1;
    }
}

template <int C>
__global__ void __launch_bounds__(kTPB) relaxed512_kernel(const __grid_constant__ KParams p,
                                                          u64 *__restrict__ words,
                                                          const u64 *__restrict__ keys, u64 n) {
    relaxed512_loop<C>(p, LocalWords{words}, keys, n);
}

// The same relaxed insert into a filter partitioned over the ranks' replicas
// (multi-GPU build over peer memory, bc_insert_peers): block reads and REDs
// go to the replica of the block's owner rank, over NVLink when remote.
template <int C>
__global__ void __launch_bounds__(kTPB) relaxed512_peer_kernel(const __grid_constant__ KParams p,
                                                               const __grid_constant__ PartWords pw,
                                                               const u64 *__restrict__ keys,
                                                               u64 n) {
    relaxed512_loop<C>(p, pw, keys, n);
}

// Lookups, 512-bit blocks, random strategy: staged blocks + per-address test
// (lookup.cuh), early exit over the choices.
template <int C, int K>
__global__ void __launch_bounds__(kTPB) lookup512_kernel(const __grid_constant__ KParams p,
                                                         const u64 *__restrict__ words,
                                                         const u64 *__restrict__ keys, u64 n,
                                                         u8 *__restrict__ out,
                                                         unsigned long long *__restrict__ hits) {
    __shared__ LookupSmem<C> smem[kWarps];
    LookupSmem<C> &ls = smem[threadIdx.x >> 5];
    const int lane = threadIdx.x & 31;
    const u64 ntiles = (n + 31) / 32;
    const u64 nwarps = (u64)gridDim.x * kWarps;
    u32 my_hits = 0;
    u64 tile = blockIdx.x * (u64)kWarps + (threadIdx.x >> 5);
    // the next tile's key is loaded while the current tile is probed
    u64 x_next = tile * 32 + lane < n ? ld_stream(keys + tile * 32 + lane) : 0ull;
    for (; tile < ntiles; tile += nwarps) {
        const u64 base = tile * 32;
        const bool valid = base + lane < n;
        const u64 x = x_next;
        const u64 nb = base + nwarps * 32 + lane;
        x_next = nb < n ? ld_stream(keys + nb) : 0ull;
        const bool f = lookup_tile<C, K>(p, words, ls, x, valid, lane);
        if (out != nullptr && valid) out[base + lane] = (u8)f;
        my_hits += f ? 1u : 0u;
        __syncwarp();
    }
    if (hits != nullptr) {
        for (int o = 16; o > 0; o >>= 1) my_hits += __shfl_xor_sync(kFull, my_hits, o);
        if (lane == 0 && my_hits) atomicAdd(hits, (unsigned long long)my_hits);
    }
}

// Single-choice lookups with two tiles per warp in flight (lookup.cuh).
template <int K>
__global__ void __launch_bounds__(kTPB) lookup512_pipe_kernel(const __grid_constant__ KParams p,
                                                              const u64 *__restrict__ words,
                                                              const u64 *__restrict__ keys, u64 n,
                                                              u8 *__restrict__ out,
                                                              unsigned long long *__restrict__ hits) {
    __shared__ PipeStage stages[kWarps][2];
    PipeStage *st = stages[threadIdx.x >> 5];
    const int lane = threadIdx.x & 31;
    const u64 ntiles = (n + 31) / 32;
    const u64 nwarps = (u64)gridDim.x * kWarps;
    u32 my_hits = 0;
    u64 tile = blockIdx.x * (u64)kWarps + (threadIdx.x >> 5);
    u64 i = tile * 32 + lane;
    bool valid = i < n;
    u64 x = valid ? ld_stream(keys + i) : 0ull;
    stage_blocks(words, st[0], valid ? (u32)block_index(p, x, 0) : 0u,
                 __ballot_sync(kFull, valid), lane);
    u64 tile_n = tile + nwarps;
    i = tile_n * 32 + lane;
    u64 x_n = i < n ? ld_stream(keys + i) : 0ull;
    int b = 0;
    for (; tile < ntiles; tile = tile_n, tile_n += nwarps) {
        const u64 base = tile * 32;
        const bool valid_n = tile_n * 32 + lane < n;
        stage_blocks(words, st[b ^ 1], valid_n ? (u32)block_index(p, x_n, 0) : 0u,
                     __ballot_sync(kFull, valid_n), lane);
        i = (tile_n + nwarps) * 32 + lane;
        const u64 x_nn = i < n ? ld_stream(keys + i) : 0ull;
        asm volatile("cp.async.wait_group 1;" ::: "memory");
        __syncwarp();
        const bool f = valid && test_staged<K>(p, st[b], x, lane);
        if (out != nullptr && valid) out[base + lane] = (u8)f;
        my_hits += f ? 1u : 0u;
        __syncwarp();
        x = x_n;
        x_n = x_nn;
        valid = valid_n;
        b ^= 1;
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    if (hits != nullptr) {
        for (int o = 16; o > 0; o >>= 1) my_hits += __shfl_xor_sync(kFull, my_hits, o);
        if (lane == 0 && my_hits) atomicAdd(hits, (unsigned long long)my_hits);
    }
}

// Multi-choice lookups with the next tile's first choice in flight: the
// choice-0 blocks of tile t+1 are staged (one cp.async group) before tile t is
// tested; tile t's later choices -- only for its still-pending keys, the
// reference's early exit -- are staged into tile t's own buffer once its
// choice-0 test is done.
template <int C, int K>
__global__ void __launch_bounds__(kTPB) lookup512_pipe_multi_kernel(
    const __grid_constant__ KParams p, const u64 *__restrict__ words,
    const u64 *__restrict__ keys, u64 n, u8 *__restrict__ out,
    unsigned long long *__restrict__ hits) {
    __shared__ PipeStage stages[kWarps][2];
    PipeStage *st = stages[threadIdx.x >> 5];
    const int lane = threadIdx.x & 31;
    const u64 ntiles = (n + 31) / 32;
    const u64 nwarps = (u64)gridDim.x * kWarps;
    u32 my_hits = 0;
    u64 tile = blockIdx.x * (u64)kWarps + (threadIdx.x >> 5);
    u64 i = tile * 32 + lane;
    bool valid = i < n;
    u64 x = valid ? ld_stream(keys + i) : 0ull;
    stage_blocks(words, st[0], valid ? (u32)block_index(p, x, 0) : 0u,
                 __ballot_sync(kFull, valid), lane);
    u64 tile_n = tile + nwarps;
    i = tile_n * 32 + lane;
    u64 x_n = i < n ? ld_stream(keys + i) : 0ull;
    int b = 0;
    for (; tile < ntiles; tile = tile_n, tile_n += nwarps) {
        const u64 base = tile * 32;
        const bool valid_n = tile_n * 32 + lane < n;
        stage_blocks(words, st[b ^ 1], valid_n ? (u32)block_index(p, x_n, 0) : 0u,
                     __ballot_sync(kFull, valid_n), lane);
        i = (tile_n + nwarps) * 32 + lane;
        const u64 x_nn = i < n ? ld_stream(keys + i) : 0ull;
        asm volatile("cp.async.wait_group 1;" ::: "memory");
        __syncwarp();
        bool f = valid && test_staged<K>(p, st[b], x, lane);
        u32 done = __ballot_sync(kFull, !valid || f);
#pragma unroll
        for (int ci = 1; ci < C; ++ci) {
            if (done == kFull) break;
            __syncwarp();  // every lane is done reading st[b]
            const bool pend = !((done >> lane) & 1u);
            stage_blocks(words, st[b], pend ? (u32)block_index(p, x, ci) : 0u, ~done, lane);
            asm volatile("cp.async.wait_group 0;" ::: "memory");
            __syncwarp();
            if (pend) f = test_staged<K>(p, st[b], x, lane);
            done |= __ballot_sync(kFull, f);
        }
        if (out != nullptr && valid) out[base + lane] = (u8)f;
        my_hits += f ? 1u : 0u;
        __syncwarp();
        x = x_n;
        x_n = x_nn;
        valid = valid_n;
        b ^= 1;
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    if (hits != nullptr) {
        for (int o = 16; o > 0; o >>= 1) my_hits += __shfl_xor_sync(kFull, my_hits, o);
        if (lane == 0 && my_hits) atomicAdd(hits, (unsigned long long)my_hits);
    }
}

template <int OP>
__global__ void __launch_bounds__(256) generic_kernel(const __grid_constant__ KParams p,
                                                      u64 *__restrict__ words,
                                                      const u64 *__restrict__ keys, u64 n,
                                                      u8 *__restrict__ out,
                                                      unsigned long long *__restrict__ hits) {
    u64 mask[kMaxWpb];
    u32 my_hits = 0;
    const u64 stride = (u64)gridDim.x * blockDim.x;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += stride) {
        const u64 x = ld_stream(keys + i);
        build_mask_generic(p, x, mask);
        if (OP == OP_CONTAINS) {
            bool found = false;
            for (u32 ci = 0; ci < p.c && !found; ++ci) {
                const u64 b = block_index(p, x, ci) * p.wpb;
                bool ok = true;
                for (u32 w = 0; w < p.wpb; ++w) ok &= (__ldg(words + b + w) & mask[w]) == mask[w];
                found = ok;
            }
            if (out) out[i] = (u8)found;
            my_hits += found ? 1u : 0u;
        } else {
            insert_generic(p, words, x, mask);
        }
    }
    if (OP == OP_CONTAINS && hits != nullptr) {
        for (int o = 16; o > 0; o >>= 1) my_hits += __shfl_xor_sync(kFull, my_hits, o);
        if ((threadIdx.x & 31) == 0 && my_hits) atomicAdd(hits, (unsigned long long)my_hits);
    }
}

// Exact stream order for c >= 2 (reference _kernels.py:133-174 is sequential).
// Keys of a chunk are applied in rounds: a pending key commits in a round iff
// it holds the smallest pending index on every one of its candidate blocks
// (claims are atomicMin'd into owner[]).  Committed keys of one round touch
// pairwise-disjoint blocks, and every earlier key sharing a block with them
// has already committed, so the result equals the sequential one.  Claims
// carry (~round) in the high word, so stale owner[] values of older rounds
// always lose and the array never needs clearing.
__global__ void __launch_bounds__(256) ordered_kernel(const __grid_constant__ KParams p,
                                                      u64 *__restrict__ words,
                                                      const u64 *__restrict__ keys, u64 n,
                                                      u64 chunk, u64 *__restrict__ owner,
                                                      u32 *__restrict__ lists,
                                                      u32 *__restrict__ state) {
    cg::grid_group grid = cg::this_grid();
    const u64 gtid = blockIdx.x * (u64)blockDim.x + threadIdx.x;
    const u64 gstride = (u64)gridDim.x * blockDim.x;
    __shared__ u32 ocol[8][16][32];  // fast path: per-thread mask columns
    u32 *col = &ocol[threadIdx.x >> 5][0][threadIdx.x & 31];
    const bool fast = p.fast_random && p.wpb == 8;
    u32 round = __ldcg(state);
    u32 *cur = lists, *nxt = lists + chunk;
    u64 mask[kMaxWpb];
    for (u64 c0 = 0; c0 < n; c0 += chunk) {
        u32 npend = (u32)min(chunk, n - c0);
        bool first = true;
        while (npend) {
            const u64 claim_hi = (u64)(0xffffffffu - round) << 32;
            u32 *cnt = state + 1 + (round & 1u);
            if (gtid == 0) *cnt = 0;
            for (u64 t = gtid; t < npend; t += gstride) {
                const u32 li = first ? (u32)t : __ldcg(cur + t);
                const u64 x = keys[c0 + li];
                for (u32 ci = 0; ci < p.c; ++ci)
                    atomicMin((unsigned long long *)(owner + block_index(p, x, ci)),
                              (unsigned long long)(claim_hi | li));
            }
            grid.sync();
            for (u64 t = gtid; t < npend; t += gstride) {
                const u32 li = first ? (u32)t : __ldcg(cur + t);
                const u64 x = keys[c0 + li];
                bool win = true;
                for (u32 ci = 0; ci < p.c; ++ci)
                    win &= __ldcg(owner + block_index(p, x, ci)) == (claim_hi | li);
                if (win && fast) {
                    insert_fast512(p, words, x, col);
                } else if (win) {
                    build_mask_generic(p, x, mask);
                    insert_generic(p, words, x, mask);
                }
                // losers go to the next pending list: one counter atomic per
                // warp (list order is irrelevant, priority is the key index)
                const u32 am = __activemask();
                const u32 lm = __ballot_sync(am, !win);
                if (lm) {
                    const int lane = threadIdx.x & 31, leader = __ffs(lm) - 1;
                    u32 base = 0;
                    if (lane == leader) base = atomicAdd(cnt, (u32)__popc(lm));
                    base = __shfl_sync(am, base, leader);
                    if (!win) nxt[base + __popc(lm & ((1u << lane) - 1u))] = li;
                }
            }
            grid.sync();
            npend = __ldcg(cnt);
            u32 *tmp = cur;
            cur = nxt;
            nxt = tmp;
            first = false;
            ++round;
        }
    }
    if (gtid == 0) state[0] = round;
}

// Exact stream order, sliding window.  Same commit rule as ordered_kernel (a
// pending key commits iff its claim is the minimum on every candidate), but:
//  * one pass and one grid sync per round: a key checks the claims made in
//    the previous round (owner[round & 1]), and if it loses it immediately
//    claims for the next round in the other owner array;
//  * instead of fixed chunks, a window of up to `window` pending keys is
//    refilled every round with the next keys of the stream, so rounds never
//    run near-empty at the tail of a chunk.
// Keys enter in index order, so every earlier key that shares a block with a
// pending key is either committed or pending (and then wins that block):
// the result is the sequential one.
//
// Claims are the 32-bit key index itself (launches cover < 2^32 - 1 keys;
// 0xffffffff is "unclaimed").  Every claimed slot has exactly one winner,
// which checks it in the next round and then resets it to unclaimed -- after
// reading all of its slots, so a key whose candidates share a slot still
// sees its own claim.  Losers read the slot before or after that reset and
// see a tag that is not theirs either way.  The last round of a launch has no
// losers (nothing is claimed in it), so both arrays are all-unclaimed between
// launches and no round number is needed in the tags: the arrays are half
// the size of 64-bit round-tagged claims, which lets the claims of a 2^23-block
// filter (64 MiB) stay L2-resident under a persisting window.  state[0] is
// the round counter (array parity); state[1..3] are rotating append counters
// (round r appends to counter r % 3 and zeroes counter (r + 1) % 3, last
// read two syncs ago).
// Claim slot of block b: the block itself (slot_shift == 0), or a
// multiplicative hash into 2^(64 - slot_shift) slots.  Two blocks sharing a
// slot only make their keys wait for each other (a spurious conflict); keys
// that share a block always share its slot, so commits stay exact, and the
// oldest pending key still wins every slot it claims.
__device__ __forceinline__ u64 owner_slot(u64 b, u32 slot_shift) {
    return slot_shift ? (b * 0x9E3779B97F4A7C15ull) >> slot_shift : b;
}

constexpr u32 kUnclaimed = 0xffffffffu;

// Round check of pending key li: does it hold the claim on every candidate?
// Its own claims are reset to unclaimed after all of them have been read.
__device__ __forceinline__ bool ordered_check(const KParams &p, u32 *own_cur, u32 slot_shift,
                                              u64 x, u32 li) {
    u32 mine = 0;  // candidates whose slot holds this key's claim
    for (u32 ci = 0; ci < p.c; ++ci)
        mine |= (u32)(__ldcg(own_cur + owner_slot(block_index(p, x, ci), slot_shift)) == li)
                << ci;
    for (u32 ci = 0; ci < p.c; ++ci)
        if ((mine >> ci) & 1u)
            __stcg(own_cur + owner_slot(block_index(p, x, ci), slot_shift), kUnclaimed);
    return mine == (1u << p.c) - 1u;
}

// The same check with one atomicCAS(slot, li -> unclaimed) per distinct slot:
// it reads the claim and resets it if it is this key's, in one L2 operation
// instead of a load and a store.  A slot repeated among the key's candidates
// is checked once (a second CAS would see it already reset).
template <int C>
__device__ __forceinline__ bool ordered_check_cas(const KParams &p, u32 *own_cur, u32 slot_shift,
                                                  u64 x, u32 li) {
    u64 sl[C];
#pragma unroll
    for (int ci = 0; ci < C; ++ci) sl[ci] = owner_slot(block_index(p, x, ci), slot_shift);
    bool held = true;
#pragma unroll
    for (int ci = 0; ci < C; ++ci) {
        bool dup = false;
#pragma unroll
        for (int cj = 0; cj < ci; ++cj) dup |= sl[cj] == sl[ci];
        if (!dup) held &= atomicCAS(own_cur + sl[ci], li, kUnclaimed) == li;
    }
    return held;
}

// The CAS check split in two, so a tile's checks can be issued before the
// previous tile's commit and consumed after it (BC_ORD_PIPE): issue returns
// the old claim of every candidate slot (a repeated slot is not CASed again
// and reports the key's own index: the first CAS answers for it).
template <int C>
__device__ __forceinline__ void ordered_cas_issue(const KParams &p, u32 *own_cur, u32 slot_shift,
                                                  u64 x, u32 li, bool on, u32 (&old)[C]) {
    u64 sl[C];
#pragma unroll
    for (int ci = 0; ci < C; ++ci) sl[ci] = owner_slot(block_index(p, x, ci), slot_shift);
#pragma unroll
    for (int ci = 0; ci < C; ++ci) {
        bool dup = false;
#pragma unroll
        for (int cj = 0; cj < ci; ++cj) dup |= sl[cj] == sl[ci];
        old[ci] = (on && !dup) ? atomicCAS(own_cur + sl[ci], li, kUnclaimed) : li;
    }
}

template <int C>
__device__ __forceinline__ bool ordered_cas_held(const u32 (&old)[C], u32 li) {
    bool held = true;
#pragma unroll
    for (int ci = 0; ci < C; ++ci) held &= old[ci] == li;
    return held;
}

// Epoch-tagged claims (ordered1_kernel): a claim is (tag << 24 | li - base),
// the tag falling by one every round and base a lower bound of every index
// claiming that round.  A newer round's claims are smaller than anything an
// older round left behind, so atomicMin overwrites stale claims and nothing
// is ever reset: the check is a plain load compared with the key's own value.
// The array is cleared in-kernel when the 8-bit tag wraps (every 256 rounds,
// counted across launches).
constexpr u32 kRelBits = 24;  // default; BC_ORDERED_REL_BITS narrows it (tests of the out-of-range path)

__device__ __forceinline__ u32 claim_tag(u32 round, u32 rel_bits) {
    return (255u - (round & 255u)) << rel_bits;
}

template <int C>
__device__ __forceinline__ void ordered_tag_issue(const KParams &p, const u32 *own_cur,
                                                  u32 slot_shift, u64 x, bool on, u32 (&old)[C]) {
#pragma unroll
    for (int ci = 0; ci < C; ++ci)
        old[ci] = on ? __ldcg(own_cur + owner_slot(block_index(p, x, ci), slot_shift)) : kUnclaimed;
}

template <int C>
__device__ __forceinline__ void ordered_claim_tag(const KParams &p, u32 *own_nxt, u32 slot_shift,
                                                  u64 x, u32 v) {
#pragma unroll
    for (int ci = 0; ci < C; ++ci)
        atomicMin(own_nxt + owner_slot(block_index(p, x, ci), slot_shift), v);
}

__device__ __forceinline__ void ordered_claim(const KParams &p, u32 *own_nxt, u32 slot_shift,
                                              u64 x, u32 li) {
    for (u32 ci = 0; ci < p.c; ++ci)
        atomicMin(own_nxt + owner_slot(block_index(p, x, ci), slot_shift), li);
}

// Losers of a round go to the next pending list: one counter atomic per warp
// (list order is irrelevant, priority is the key index).
__device__ __forceinline__ void ordered_append(u32 *cnt, u32 *nxt, bool lose, u32 li, int lane) {
    const u32 am = __activemask();
    const u32 lm = __ballot_sync(am, lose);
    if (lm) {
        const int leader = __ffs(lm) - 1;
        u32 base = 0;
        if (lane == leader) base = atomicAdd(cnt, (u32)__popc(lm));
        base = __shfl_sync(am, base, leader);
        if (lose) nxt[base + __popc(lm & ((1u << lane) - 1u))] = li;
    }
}

__global__ void __launch_bounds__(256) ordered_window_kernel(
    const __grid_constant__ KParams p, u64 *__restrict__ words, const u64 *__restrict__ keys,
    u64 n, u64 window, u32 *__restrict__ owner, u64 slots, u32 slot_shift,
    u32 *__restrict__ lists, u32 *__restrict__ state) {
    cg::grid_group grid = cg::this_grid();
    const u64 gtid = blockIdx.x * (u64)blockDim.x + threadIdx.x;
    const u64 gstride = (u64)gridDim.x * blockDim.x;
    const int lane = threadIdx.x & 31;
    __shared__ u32 ocol[8][16][32];  // fast path: per-thread mask columns
    u32 *col = &ocol[threadIdx.x >> 5][0][threadIdx.x & 31];
    const bool fast = p.fast_random && p.wpb == 8;
    u32 round = __ldcg(state);
    u32 *cur = lists, *nxt = lists + window;
    u64 npend = 0, next = 0;
    u64 mask[kMaxWpb];
    while (npend > 0 || next < n) {
        const u64 admit = min(window - npend, n - next);
        u32 *own_cur = owner + (round & 1u) * slots;
        u32 *own_nxt = owner + ((round + 1u) & 1u) * slots;
        u32 *cnt = state + 1 + round % 3u;
        if (gtid == 0) state[1 + (round + 1u) % 3u] = 0;
        for (u64 t = gtid; t < npend + admit; t += gstride) {
            u32 li;
            bool lose = true;
            u64 x;
            if (t < npend) {
                li = __ldcg(cur + t);
                x = keys[li];
                const bool win = ordered_check(p, own_cur, slot_shift, x, li);
                if (win && fast) {
                    insert_fast512(p, words, x, col);
                } else if (win) {
                    build_mask_generic(p, x, mask);
                    insert_generic(p, words, x, mask);
                }
                lose = !win;
            } else {
                li = (u32)(next + (t - npend));  // newly admitted
                x = keys[li];
            }
            if (lose) ordered_claim(p, own_nxt, slot_shift, x, li);
            ordered_append(cnt, nxt, lose, li, lane);
        }
        grid.sync();
        npend = __ldcg(cnt);
        next += admit;
        u32 *tmp = cur;
        cur = nxt;
        nxt = tmp;
        ++round;
    }
    if (gtid == 0) state[0] = round;
}

// The same rounds for 512-bit blocks with the random strategy (every BASELINE
// configuration): a round's winners are committed a warp tile at a time with
// the relaxed insert's two-phase step (masks built one lane per key, the C
// candidates of four keys at once read with one LDG.128 per lane, the
// reference's decision, two sector-wide REDs per key), instead of one thread
// per key issuing 4 C loads and 8 REDs.  Winners of one round touch pairwise
// disjoint blocks, so the blocks they read cannot change under them.
#ifndef BC_ORD_UNR
#define BC_ORD_UNR 0  // keys per load step of the commit (0: relaxed_unroll(C))
#endif
#ifndef BC_ORD_NT
#define BC_ORD_NT 256  // threads per CTA of the claim rounds
#endif
#ifndef BC_ORD_DYN
#define BC_ORD_DYN 1  // claim rounds: tiles after each warp's first taken from a CTA counter
#endif
#ifndef BC_ORD_CAS
#define BC_ORD_CAS 1  // claim checks as one atomicCAS per distinct slot
#endif
#ifndef BC_ORD_PIPE
#define BC_ORD_PIPE 1  // claim rounds: next tile's CAS checks issued before this tile's commit (cfg3 +1.8%, cfg5 +0.9%)
#endif
#ifndef BC_ORD_SKIP
#define BC_ORD_SKIP 1  // commit tiles: lanes without a winner read nothing (not block 0)
#endif
#ifndef BC_ORD_MINB
#define BC_ORD_MINB 3  // <= 80 registers: 3 CTAs per SM (cfg3 +4%, cfg5 +8% over 2 CTAs at 102)
#endif
// Pending lists are CTA-local (shared memory): a key that loses a round is
// retried by the CTA that holds it, so no grid-wide list or append counter
// exists (one counter hammered by every warp's append was a serialised L2
// hot spot, and the lists a DRAM round trip).  Each round every CTA refills
// its list to `cap` entries with the next keys of the stream, taken with ONE
// atomicAdd on a global cursor: the CTAs' slices of a round are disjoint and
// together contiguous, and every slice of a round precedes every slice of
// the next (a grid sync separates them), so keys still enter in index order
// -- the invariant the commit rule needs.  Termination: in one round the sum
// of the CTAs' pending counts (one atomic per CTA) is zero and some CTA's
// slice reached the end of the stream (bit 31 of the same word: the cursor
// itself cannot be compared after the sync, a fast CTA may already have
// taken its next slice).
// state (u32 x 16; [0..7] zeroed, [8..15] all-ones before each launch):
// [0..2] rotating round words (pending total | exhausted << 31), [4..5] the
// u64 stream cursor ([8..10] belong to ordered1_kernel).
template <int C, class Src>
__global__ void __launch_bounds__(BC_ORD_NT, BC_ORD_MINB) ordered512_kernel(
    const __grid_constant__ KParams p, u64 *__restrict__ words, const Src src, u64 n, u32 cap,
    u32 *__restrict__ owner, u64 slots, u32 slot_shift, u32 *__restrict__ state,
    unsigned long long *__restrict__ admitted) {
    cg::grid_group grid = cg::this_grid();
    __shared__ WarpSmem<C> smem[BC_ORD_NT / 32];
    __shared__ u32 s_cnt, s_pend, s_adm, s_exh, s_tile;
    __shared__ u64 s_start;
    extern __shared__ __align__(16) unsigned char dsm[];
    WarpSmem<C> &ws = smem[threadIdx.x >> 5];
    const int lane = threadIdx.x & 31;
    const u32 wid = threadIdx.x >> 5;
    // the CTA's pending lists: stream index (priority) and key, two buffers
    u64 *curk = reinterpret_cast<u64 *>(dsm), *nxtk = curk + cap;
    u32 *cur = reinterpret_cast<u32 *>(nxtk + cap), *nxt = cur + cap;
    unsigned long long *cursor = reinterpret_cast<unsigned long long *>(state + 4);
    if (threadIdx.x == 0) {
        s_pend = 0;
        s_cnt = 0;
    }
    u32 round = 0;
    u32 n_admitted = 0;
#ifdef BC_ORD_PROF
    long long t_work = 0, t_sync = 0, tq = clock64();
    long long t_chk = 0, t_com = 0, t_rest = 0;
    u32 ntiles = 0, ncom = 0;
#endif
    for (;;) {
        u32 *own_cur = owner + (round & 1u) * slots;
        u32 *own_nxt = owner + ((round + 1u) & 1u) * slots;
        if (threadIdx.x == 0) {
            // refill to cap from the stream (s_pend: this CTA's losers of last round)
            const u32 free = cap - s_pend;
            const u64 st = free ? atomicAdd(cursor, (unsigned long long)free) : 0ull;
            s_start = st;
            s_adm = (free && st < n) ? (u32)min((u64)free, n - st) : 0u;
            s_exh = free && st + free >= n;
            s_cnt = 0;
            s_tile = BC_ORD_NT;  // tiles past each warp's first, handed out on demand
            if (blockIdx.x == 0) state[(round + 1u) % 3u] = 0;  // last read in round r-1
        }
        __syncthreads();
        const u32 npend = s_pend, total = s_pend + s_adm;
        const u64 start = s_start;
        // tile entry t: a pending key from the list, or the next key of the slice
        auto fetch = [&](u32 t, u32 &li, u64 &x) -> bool {
            if (t >= total) return false;
            if (t < npend) {
                li = cur[t];
                x = curk[t];
                return true;
            }
            const u64 idx = start + (t - npend);
            li = (u32)idx;
            const bool ok = src.admit(idx, x);
            n_admitted += ok ? 1u : 0u;
            return ok;
        };
        // warp-uniform tiles; the next tile's entries are fetched while the
        // current tile's candidate blocks are read and committed
        u32 t0 = wid * 32;
#if BC_ORD_DYN
        // the warps' first tiles are static; later ones go to whichever warp
        // is free first, so a slow tile does not hold up its warp's share
        auto next_tile = [&]() -> u32 {
            u32 v = 0;
            if (lane == 0) v = atomicAdd(&s_tile, 32u);
            return __shfl_sync(kFull, v, 0);
        };
#endif
        u32 li = 0;
        u64 x = 0;
        bool valid = fetch(t0 + lane, li, x);
#if BC_ORD_PIPE
        u32 cas_old[C];
        ordered_cas_issue<C>(p, own_cur, slot_shift, x, li, valid && t0 + lane < npend, cas_old);
#endif
        while (t0 < total) {
#ifdef BC_ORD_PROF
            const long long ta = clock64();
#endif
            const u32 t = t0 + lane;
#if BC_ORD_PIPE
            const bool win = valid && t < npend && ordered_cas_held<C>(cas_old, li);
#elif BC_ORD_CAS
            const bool win =
                valid && t < npend && ordered_check_cas<C>(p, own_cur, slot_shift, x, li);
#else
            const bool win = valid && t < npend && ordered_check(p, own_cur, slot_shift, x, li);
#endif
            const bool lose = valid && !win;
            if (lose) ordered_claim(p, own_nxt, slot_shift, x, li);
            const u32 lm = __ballot_sync(kFull, lose);
#ifdef BC_ORD_PROF
            const long long tb_ = clock64();
            t_chk += tb_ - ta;
#endif
            u32 base = 0;
            if (lm && lane == 0) base = atomicAdd(&s_cnt, (u32)__popc(lm));
#if BC_ORD_DYN
            const u32 t1 = next_tile();
#else
            const u32 t1 = t0 + BC_ORD_NT;
#endif
            u32 li_n = 0;
            u64 x_n = 0;
            const bool valid_n = fetch(t1 + lane, li_n, x_n);
#if BC_ORD_PIPE
            // the next tile's checks are in flight during this tile's commit
            u32 cas_n[C];
            ordered_cas_issue<C>(p, own_cur, slot_shift, x_n, li_n, valid_n && t1 + lane < npend,
                                 cas_n);
#endif
#ifdef BC_ORD_PROF
            const long long tc_ = clock64();
            t_rest += tc_ - tb_;
#endif
            if (__ballot_sync(kFull, win)) {  // tiles of admitted keys only claim
                phase1<C, BC_ORD_SKIP != 0>(p, x, win, ws, lane);
                __syncwarp();
                phase2<OP_INSERT, C, BC_ORD_UNR>(p, words, ws, lane);
                __syncwarp();
#ifdef BC_ORD_PROF
                ++ncom;
#endif
            }
#ifdef BC_ORD_PROF
            const long long td_ = clock64();
            t_com += td_ - tc_;
#endif
            if (lm) {
                base = __shfl_sync(kFull, base, 0);
                if (lose) {
                    const u32 slot = base + __popc(lm & ((1u << lane) - 1u));
                    nxt[slot] = li;
                    nxtk[slot] = x;
                }
            }
            li = li_n;
            x = x_n;
            valid = valid_n;
#if BC_ORD_PIPE
#pragma unroll
            for (int ci = 0; ci < C; ++ci) cas_old[ci] = cas_n[ci];
#endif
            t0 = t1;
#ifdef BC_ORD_PROF
            ++ntiles;
#endif
        }
        __syncthreads();  // the round's local appends are complete
        if (threadIdx.x == 0) {
            s_pend = s_cnt;
            if (s_cnt) atomicAdd(state + round % 3u, s_cnt);
            if (s_exh) atomicOr(state + round % 3u, 0x80000000u);
        }
#ifdef BC_ORD_PROF
        {
            const long long t_ = clock64();
            t_work += t_ - tq;
            tq = t_;
        }
#endif
        grid.sync();
#ifdef BC_ORD_PROF
        {
            const long long t_ = clock64();
            t_sync += t_ - tq;
            tq = t_;
        }
#endif
        const u32 rw = __ldcg(state + round % 3u);
        const bool more = (rw & 0x7fffffffu) != 0 || !(rw >> 31);
        u32 *tmp = cur;
        cur = nxt;
        nxt = tmp;
        u64 *tmpk = curk;
        curk = nxtk;
        nxtk = tmpk;
        ++round;
        if (!more) break;
    }
    if (Src::kCounts && admitted != nullptr) {
        for (int o = 16; o > 0; o >>= 1) n_admitted += __shfl_xor_sync(kFull, n_admitted, o);
        if (lane == 0 && n_admitted) atomicAdd(admitted, (unsigned long long)n_admitted);
    }
#ifdef BC_ORD_PROF
    if (lane == 0 && (blockIdx.x % 64) == 0 && wid == 0)
        printf("ord prof cta %u rounds %u tiles %u (commit %u) work/round %lld sync/round %lld "
               "per tile: check %lld fetch %lld commit-tile %lld\n",
               blockIdx.x, round, ntiles, ncom, t_work / max(round, 1u), t_sync / max(round, 1u),
               t_chk / max(ntiles, 1u), t_rest / max(ntiles, 1u), t_com / max(ncom, 1u));
#endif
}


// One claim array, one grid sync per round, and a key claims and commits in
// the same round (BC_ORDERED_ONE, the default for the tiled path):
//
//   phase A  every key the CTA holds -- last round's losers and the next
//            slice of the stream -- claims its candidate slots:
//            atomicMin(slot, tag_r | li - base_r);
//   grid sync
//   phase B  every such key loads its slots; it holds a slot that still shows
//            its own value.  Holders of all their slots commit (a warp tile at
//            a time, as in ordered512_kernel), the others go to the next list.
//
// There is no sync between phase B and the next round's phase A, so a fast
// CTA's round r+1 claims (smaller tag) may overwrite a slot before a slow
// CTA's key has checked it in round r.  That key then sees a foreign value
// and waits one more round: a false loss, never a false win -- a key wins
// only where its own round-r value survived, i.e. no earlier key claimed the
// slot in round r, and every uncommitted earlier key did claim (keys enter in
// index order, slices of different rounds being separated by a sync).  The
// commits of round r and the block loads of round r+1 are separated by
// round r+1's sync.
//
// Against ordered512_kernel's two reset-on-win arrays this halves the claim
// footprint in the L2 (what the rounds are most sensitive to), replaces the
// c atomicCAS checks of a key by c loads, and commits a window's keys per
// sync instead of half a window's.
//
// Rotating state words (written in phase B of round r, complete at round
// r+1's sync, read in phase B of round r+1, re-armed in phase B of round r+2):
// [r % 3] pending total | exhausted << 31, [8 + r % 3] the minimum of the
// losers' indices and the CTAs' slice ends -- a lower bound of every index
// that claims from round r+1 on, used as the claim base two rounds later.
// A key further than 2^24 - 2 above the base skips its claim and waits.
// -DBC_ORD_CHECK: index checks of ordered1_kernel's lists and claim slots
// (compute-sanitizer is not available on the pool); a violation traps.
#ifdef BC_ORD_CHECK
#define BC_ORD_ASSERT(cond)                                                              \
    do {                                                                                 \
        if (!(cond)) {                                                                   \
            printf("ordered1_kernel check failed: %s (line %d, cta %u thread %u)\n", #cond, \
                   __LINE__, blockIdx.x, threadIdx.x);                                   \
            __trap();                                                                    \
        }                                                                                \
    } while (0)
#else
#define BC_ORD_ASSERT(cond) ((void)0)
#endif
#ifndef BC_ORD1_MINB2
#define BC_ORD1_MINB2 2  // c = 2: 2 CTAs per SM at <= 128 registers (cfg5 9 112 -> 9 497 Mkeys/s, cfg4's geometry equal)
#endif
constexpr int ord1_minb(int C) { return C == 2 ? BC_ORD1_MINB2 : BC_ORD_MINB; }

template <int C, class Src>
__global__ void __launch_bounds__(BC_ORD_NT, ord1_minb(C)) ordered1_kernel(
    const __grid_constant__ KParams p, u64 *__restrict__ words, const Src src, u64 n, u32 cap,
    u32 *__restrict__ owner, u64 slots, u32 slot_shift, u32 *__restrict__ state,
    unsigned long long *__restrict__ admitted, u32 rel_bits) {
    cg::grid_group grid = cg::this_grid();
    const u32 kRelLimit = (1u << rel_bits) - 1u;  // 0xffffffff is never a claim
    __shared__ WarpSmem<C> smem[BC_ORD_NT / 32];
    __shared__ u32 s_cnt, s_adm, s_exh, s_tile, s_min, s_new;
    __shared__ u64 s_start;
    extern __shared__ __align__(16) unsigned char dsm[];
    WarpSmem<C> &ws = smem[threadIdx.x >> 5];
    const int lane = threadIdx.x & 31;
    const u32 wid = threadIdx.x >> 5;
    u64 *curk = reinterpret_cast<u64 *>(dsm), *nxtk = curk + cap;
    u32 *cur = reinterpret_cast<u32 *>(nxtk + cap), *nxt = cur + cap;
    unsigned long long *cursor = reinterpret_cast<unsigned long long *>(state + 4);
    u32 round = 0, n_admitted = 0;
    u32 npend = 0;  // this CTA's losers of the last round, at the front of cur
    u32 base = 0, base_next = 0;
    // the tags run on across launches (state[12], zero when the scratch is
    // allocated): an earlier launch's claims are older rounds' claims, so a
    // short insert does not pay for a clear of the array
    const u32 epoch0 = __ldcg(state + 12);
#ifdef BC_ORD_PROF
    long long t_a = 0, t_sync = 0, t_b = 0, tq = clock64();
    u32 n_lost = 0, n_seen = 0;
#endif
    for (;;) {
        const u32 epoch = epoch0 + round;
        if ((epoch & 255u) == 0) {
            // the tag restarts: what the array holds (checked until the end of
            // the last round) would outrank it
            if (round) grid.sync();
            for (u64 i = blockIdx.x * (u64)BC_ORD_NT + threadIdx.x; i < slots;
                 i += (u64)gridDim.x * BC_ORD_NT)
                __stcg(owner + i, kUnclaimed);
            grid.sync();
        }
        const u32 tag = claim_tag(epoch, rel_bits);
        // ---- phase A: claims ----
        // the slice's round trip to the cursor runs under the losers' claims
        if (threadIdx.x == 0) {
            const u32 free = cap - npend;
            const u64 st = free ? atomicAdd(cursor, (unsigned long long)free) : 0ull;
            s_start = st;
            s_adm = (free && st < n) ? (u32)min((u64)free, n - st) : 0u;
            s_exh = free && st + free >= n;
            s_new = 0;
            s_min = kUnclaimed;
            s_tile = BC_ORD_NT;
        }
        BC_ORD_ASSERT(npend <= cap);
        for (u32 t = threadIdx.x; t < npend; t += BC_ORD_NT) {
            const u32 rel = cur[t] - base;
            BC_ORD_ASSERT(cur[t] >= base && cur[t] < n);
#ifdef BC_ORD_CHECK
            for (int ci = 0; ci < C; ++ci)
                BC_ORD_ASSERT(owner_slot(block_index(p, curk[t], ci), slot_shift) < slots &&
                              block_index(p, curk[t], ci) < p.num_blocks);
#endif
            if (rel < kRelLimit) ordered_claim_tag<C>(p, owner, slot_shift, curk[t], tag | rel);
        }
        __syncthreads();
        const u32 adm = s_adm;
        const u64 start = s_start;
        // new keys, four tiles of loads in flight per warp
        for (u32 t0 = wid * 32; t0 < adm; t0 += 4 * BC_ORD_NT) {  // warp-uniform
            u64 xs[4];
            bool oks[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const u32 t = t0 + u * BC_ORD_NT + lane;
                xs[u] = 0;
                oks[u] = t < adm && src.admit(start + t, xs[u]);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const u32 om = __ballot_sync(kFull, oks[u]);
                if (om == 0) continue;  // warp-uniform
                u32 at = 0;
                if (lane == 0) at = atomicAdd(&s_new, (u32)__popc(om));
                at = __shfl_sync(kFull, at, 0);
                if (oks[u]) {
                    const u32 idx = (u32)(start + t0 + u * BC_ORD_NT + lane);
                    const u32 slot = npend + at + __popc(om & ((1u << lane) - 1u));
                    BC_ORD_ASSERT(slot < cap && idx >= base && (u64)idx < n);
                    cur[slot] = idx;
                    curk[slot] = xs[u];
                    const u32 rel = idx - base;
                    if (rel < kRelLimit)
                        ordered_claim_tag<C>(p, owner, slot_shift, xs[u], tag | rel);
                    ++n_admitted;
                }
            }
        }
        __syncthreads();
        const u32 total = npend + s_new;
        BC_ORD_ASSERT(total <= cap && s_new <= adm);
        if (threadIdx.x == 0) s_cnt = 0;  // every thread has read last round's count
#ifdef BC_ORD_PROF
        {
            const long long t_ = clock64();
            t_a += t_ - tq;
            tq = t_;
        }
#endif
        grid.sync();
#ifdef BC_ORD_PROF
        {
            const long long t_ = clock64();
            t_sync += t_ - tq;
            tq = t_;
        }
#endif
        // ---- last round's outcome ----
        if (round) {
            const u32 rw = __ldcg(state + (round - 1u) % 3u);
            if ((rw & 0x7fffffffu) == 0 && (rw >> 31)) break;  // nothing pending, stream ended
            const u32 mp = __ldcg(state + 8u + (round - 1u) % 3u);
            base_next = mp != kUnclaimed ? mp : base;
        }
        if (blockIdx.x == 0 && threadIdx.x == 0) {  // round r-2's words: read in round r-1
            state[(round + 1u) % 3u] = 0;
            state[8u + (round + 1u) % 3u] = kUnclaimed;
        }
        // ---- phase B: checks and commits ----
        auto fetch = [&](u32 t, u32 &li, u64 &x) -> bool {
            if (t >= total) return false;
            li = cur[t];
            x = curk[t];
            return true;
        };
        auto next_tile = [&]() -> u32 {
            u32 v = 0;
            if (lane == 0) v = atomicAdd(&s_tile, 32u);
            return __shfl_sync(kFull, v, 0);
        };
        u32 t0 = wid * 32;
        u32 li = 0;
        u64 x = 0;
        bool valid = fetch(t0 + lane, li, x);
        u32 rel = li - base;
        u32 seen[C];
        ordered_tag_issue<C>(p, owner, slot_shift, x, valid && rel < kRelLimit, seen);
        while (t0 < total) {
            const bool win = valid && rel < kRelLimit && ordered_cas_held<C>(seen, tag | rel);
            const bool lose = valid && !win;
            const u32 lm = __ballot_sync(kFull, lose);
#ifdef BC_ORD_PROF
            n_lost += __popc(lm);
            n_seen += __popc(__ballot_sync(kFull, valid));
#endif
            u32 at = 0;
            if (lm) {
                const u32 mn = __reduce_min_sync(kFull, lose ? li : kUnclaimed);
                if (lane == 0) {
                    atomicMin(&s_min, mn);
                    at = atomicAdd(&s_cnt, (u32)__popc(lm));
                }
            }
            const u32 t1 = next_tile();
            u32 li_n = 0;
            u64 x_n = 0;
            const bool valid_n = fetch(t1 + lane, li_n, x_n);
            const u32 rel_n = li_n - base;
            u32 seen_n[C];  // the next tile's claim loads fly during this tile's commit
            ordered_tag_issue<C>(p, owner, slot_shift, x_n, valid_n && rel_n < kRelLimit, seen_n);
            if (__ballot_sync(kFull, win)) {
                phase1<C, true>(p, x, win, ws, lane);
                __syncwarp();
                phase2<OP_INSERT, C, BC_ORD_UNR>(p, words, ws, lane);
                __syncwarp();
            }
            if (lm) {
                at = __shfl_sync(kFull, at, 0);
                if (lose) {
                    const u32 slot = at + __popc(lm & ((1u << lane) - 1u));
                    BC_ORD_ASSERT(slot < cap);
                    nxt[slot] = li;
                    nxtk[slot] = x;
                }
            }
            li = li_n;
            x = x_n;
            valid = valid_n;
            rel = rel_n;
#pragma unroll
            for (int ci = 0; ci < C; ++ci) seen[ci] = seen_n[ci];
            t0 = t1;
        }
        __syncthreads();
        npend = s_cnt;
        if (threadIdx.x == 0) {
            u32 m = s_min;
            if (adm) m = min(m, (u32)(start + adm));  // bounds every later slice from below
            if (m != kUnclaimed) atomicMin(state + 8u + round % 3u, m);
            if (npend) atomicAdd(state + round % 3u, npend);
            if (s_exh) atomicOr(state + round % 3u, 0x80000000u);
        }
        u32 *tmp = cur;
        cur = nxt;
        nxt = tmp;
        u64 *tmpk = curk;
        curk = nxtk;
        nxtk = tmpk;
        base = base_next;
        ++round;
#ifdef BC_ORD_PROF
        {
            const long long t_ = clock64();
            t_b += t_ - tq;
            tq = t_;
        }
#endif
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) state[12] = epoch0 + round + 1u;
#ifdef BC_ORD_PROF
    if (lane == 0 && (blockIdx.x % 64) == 0 && wid == 0)
        printf("ord1 prof cta %u rounds %u per round: claims %lld sync %lld commits %lld; warp 0 saw %u "
               "keys, %u lost\n",
               blockIdx.x, round, t_a / max(round, 1u), t_sync / max(round, 1u),
               t_b / max(round, 1u), n_seen, n_lost);
#endif
    if (Src::kCounts && admitted != nullptr) {
        for (int o = 16; o > 0; o >>= 1) n_admitted += __shfl_xor_sync(kFull, n_admitted, o);
        if (lane == 0 && n_admitted) atomicAdd(admitted, (unsigned long long)n_admitted);
    }
}

template <int OP>
__global__ void __launch_bounds__(256) flat_kernel(const __grid_constant__ KParams p,
                                                   u64 *__restrict__ words,
                                                   const u64 *__restrict__ keys, u64 n,
                                                   u8 *__restrict__ out,
                                                   unsigned long long *__restrict__ hits) {
    u32 my_hits = 0;
    const u64 stride = (u64)gridDim.x * blockDim.x;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += stride) {
        const u64 x = ld_stream(keys + i);
        bool ok = true;
        for (u32 b = 0; b < p.k; ++b) {
            const u64 f = hval(__ldg(&p.bits[b].a), x, p.flat_b, p.flat_magic, p.flat_mode,
                               p.flat_shift);
            const u64 bit = 1ull << (f & 63);
            if (OP == OP_INSERT) {
                atomicOr((unsigned long long *)(words + (f >> 6)), (unsigned long long)bit);
            } else if ((__ldg(words + (f >> 6)) & bit) == 0) {
                // early exit at the first clear bit; measured faster than
                // loading the addresses four at a time (19.6 vs 17.7 G/s)
                ok = false;
                break;
            }
        }
        if (OP == OP_CONTAINS) {
            if (out) out[i] = (u8)ok;
            my_hits += ok ? 1u : 0u;
        }
    }
    if (OP == OP_CONTAINS && hits != nullptr) {
        for (int o = 16; o > 0; o >>= 1) my_hits += __shfl_xor_sync(kFull, my_hits, o);
        if ((threadIdx.x & 31) == 0 && my_hits) atomicAdd(hits, (unsigned long long)my_hits);
    }
}

// 512-bit blocks: four lanes per block, one coalesced LDG.128 each.
__global__ void __launch_bounds__(256) hist512_kernel(const u64 *__restrict__ words,
                                                      u64 num_blocks,
                                                      unsigned long long *__restrict__ counts) {
    __shared__ u32 sh[513];
    for (int j = threadIdx.x; j < 513; j += blockDim.x) sh[j] = 0;
    __syncthreads();
    const uint4 *w4 = reinterpret_cast<const uint4 *>(words);
    const u64 lanes = (u64)gridDim.x * blockDim.x;
    const u64 total = num_blocks * 4;
    // iterate in whole warps so the 4-lane shuffles see full groups
    for (u64 i0 = (blockIdx.x * (u64)blockDim.x + threadIdx.x) & ~31ull; i0 < total;
         i0 += lanes) {
        const u64 i = i0 + (threadIdx.x & 31);
        u32 c = i < total ? popc4(ld_block_nc(w4 + i)) : 0u;
        c += __shfl_xor_sync(kFull, c, 1);
        c += __shfl_xor_sync(kFull, c, 2);
        if ((i & 3) == 0 && i < total) atomicAdd(&sh[c], 1u);
    }
    __syncthreads();
    for (int j = threadIdx.x; j < 513; j += blockDim.x)
        if (sh[j]) atomicAdd(counts + j, (unsigned long long)sh[j]);
}

__global__ void __launch_bounds__(256) hist_generic_kernel(const u64 *__restrict__ words,
                                                           u64 num_blocks, u32 wpb,
                                                           unsigned long long *__restrict__ counts) {
    const u64 stride = (u64)gridDim.x * blockDim.x;
    for (u64 b = blockIdx.x * (u64)blockDim.x + threadIdx.x; b < num_blocks; b += stride) {
        u32 c = 0;
        for (u32 w = 0; w < wpb; ++w) c += (u32)__popcll(__ldg(words + b * wpb + w));
        atomicAdd(counts + c, 1ull);
    }
}

__global__ void __launch_bounds__(256) eval_hash_kernel(DevHash h, const u64 *__restrict__ keys,
                                                        u64 n, u64 *__restrict__ out) {
    const u64 stride = (u64)gridDim.x * blockDim.x;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += stride)
        out[i] = hval(h, keys[i]);
}

// ---------------------------------------------------------------------------------
static bool lookup_pipe_enabled() {
    static const bool on = [] {
        const char *e = getenv("BC_LOOKUP_PIPE");
        return e == nullptr || atoi(e) != 0;
    }();
    return on;
}

// L2 residency of the filter words.  A filter that fits in L2 is launched with
// an access-policy window marking its words persisting (the streamed keys stay
// normal): on B200 this keeps the 96 MiB cfg2 filter's dirty lines in L2
// instead of writing them back under the key stream, +42% single-choice insert
// rate.  Filters larger than L2 are left alone (a partial window slows relaxed
// inserts: cfg3 11.9 -> 6.5 Gkeys/s).  BC_L2_PERSIST=0 disables, =1 forces.
struct L2Info {
    size_t l2 = 0, persist = 0, window = 0;
    bool init = false;
    bool on = false;  // persisting set-aside carved out on this device
    size_t limit = 0;  // its current size
};

constexpr int kMaxDevices = 64;
static std::mutex g_l2_mu;
static L2Info g_l2[kMaxDevices];

static int current_device() {
    int dev = 0;
    cudaGetDevice(&dev);
    return dev >= 0 && dev < kMaxDevices ? dev : -1;
}

// per-device attributes; the first call on a device also resets lines left
// persisting by an earlier process, which would shrink the L2 for everything
// this one does.  Call with g_l2_mu held.
static L2Info *l2_info_locked(int dev) {
    if (dev < 0) return nullptr;
    L2Info &i = g_l2[dev];
    if (!i.init) {
        int v = 0;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrL2CacheSize, dev) == cudaSuccess) i.l2 = v;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxAccessPolicyWindowSize, dev) == cudaSuccess)
            i.window = v;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxPersistingL2CacheSize, dev) == cudaSuccess)
            i.persist = v > 0 ? v : 0;
        cudaCtxResetPersistingL2Cache();
        cudaGetLastError();
        i.init = true;
    }
    return &i;
}

static int l2_persist_mode() {  // -1 auto, 0 off, 1 forced
    static const int m = [] {
        const char *e = getenv("BC_L2_PERSIST");
        return e ? atoi(e) : -1;
    }();
    return m;
}

// The persisting set-aside is carved out only while windows are in use: it and
// the persisting lines are given back (reset + limit 0) by the first launch
// that runs without a window, by filter teardown and at exit (bc_l2_release).
static void l2_release_locked(L2Info &i) {
    if (i.on) {
        cudaCtxResetPersistingL2Cache();
        cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, 0);
        cudaGetLastError();
        i.on = false;
    }
}

// Window for a filter of fbytes on the current device, or false.
// `fit`: carve out no more than the window needs (the rest of the L2 stays
// with everything else the kernel touches) instead of the device maximum.
static bool l2_window(size_t fbytes, size_t *bytes, float *hit_ratio, bool fit = false,
                      size_t cap = 0) {
    const int mode = l2_persist_mode();
    std::lock_guard<std::mutex> lk(g_l2_mu);
    L2Info *i = l2_info_locked(current_device());
    if (!i) return false;
    const bool want = mode != 0 && i->persist && i->window && (mode == 1 || fbytes <= i->l2);
    if (!want) {
        l2_release_locked(*i);
        return false;
    }
    size_t limit = fit ? std::min(i->persist, (fbytes + (1u << 20) - 1) & ~(size_t)((1u << 20) - 1))
                       : i->persist;
    if (cap) limit = std::min(i->persist, cap);  // explicit size (experiments)
    if (!i->on || i->limit != limit) {
        if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, limit) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        i->on = true;
        i->limit = limit;
    }
    *bytes = std::min(fbytes, i->window);
    *hit_ratio = std::min(1.0f, (float)limit / (float)std::max<size_t>(*bytes, 1));
    return true;
}

void l2_release() {
    std::lock_guard<std::mutex> lk(g_l2_mu);
    const int dev = current_device();
    if (dev >= 0) l2_release_locked(g_l2[dev]);
}

void l2_release_all() {
    std::lock_guard<std::mutex> lk(g_l2_mu);
    int prev = 0;
    cudaGetDevice(&prev);
    for (int d = 0; d < kMaxDevices; ++d) {
        if (!g_l2[d].on) continue;
        cudaSetDevice(d);
        l2_release_locked(g_l2[d]);
    }
    cudaSetDevice(prev);
    cudaGetLastError();
}

template <typename K, typename... Args>
static cudaError_t launch_words(K kernel, unsigned grid, const KParams &p, const u64 *words,
                                cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kTPB);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    size_t bytes = 0;
    float hit = 0.f;
    if (l2_window((size_t)p.num_blocks * p.wpb * 8, &bytes, &hit)) {
        attr[0].id = cudaLaunchAttributeAccessPolicyWindow;
        attr[0].val.accessPolicyWindow.base_ptr = const_cast<u64 *>(words);
        attr[0].val.accessPolicyWindow.num_bytes = bytes;
        attr[0].val.accessPolicyWindow.hitRatio = hit;
        attr[0].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        attr[0].val.accessPolicyWindow.missProp = cudaAccessPropertyNormal;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
    }
    count_launch();
    return cudaLaunchKernelEx(&cfg, kernel, args...);
}

template <int K>
static cudaError_t launch_pipe_k(const KParams &p, const u64 *words, const u64 *keys, u64 n,
                                 u8 *out, unsigned long long *hits, cudaStream_t s) {
    const void *fl = (const void *)lookup512_pipe_kernel<K>;
    const unsigned g = grid_for(fl, kTPB, 0, (n + kTPB - 1) / kTPB);
    return launch_words(lookup512_pipe_kernel<K>, g, p, words, s, p, words, keys, n, out, hits);
}

// k known at compile time for the common 4..16 (fully unrolled bit tests)
static cudaError_t launch_pipe(const KParams &p, const u64 *words, const u64 *keys, u64 n,
                               u8 *out, unsigned long long *hits, cudaStream_t s) {
    switch (p.k) {
#define BC_PIPE_K(k) \
    case k: return launch_pipe_k<k>(p, words, keys, n, out, hits, s);
        BC_PIPE_K(4) BC_PIPE_K(5) BC_PIPE_K(6) BC_PIPE_K(7) BC_PIPE_K(8) BC_PIPE_K(9)
        BC_PIPE_K(10) BC_PIPE_K(11) BC_PIPE_K(12) BC_PIPE_K(13) BC_PIPE_K(14) BC_PIPE_K(15)
        BC_PIPE_K(16)
#undef BC_PIPE_K
        default: return launch_pipe_k<0>(p, words, keys, n, out, hits, s);
    }
}

template <int C, int K>
static cudaError_t launch_lookup_k(const KParams &p, const u64 *words, const u64 *keys, u64 n,
                                   u8 *out, unsigned long long *hits, cudaStream_t s) {
    if (C <= 3 && lookup_pipe_enabled()) {
        const void *fp = (const void *)lookup512_pipe_multi_kernel<C, K>;
        const unsigned g = grid_for(fp, kTPB, 0, (n + kTPB - 1) / kTPB);
        return launch_words(lookup512_pipe_multi_kernel<C, K>, g, p, words, s, p, words, keys, n,
                            out, hits);
    }
    const void *fl = (const void *)lookup512_kernel<C, K>;
    const unsigned g = grid_for(fl, kTPB, 0, (n + kTPB - 1) / kTPB);
    return launch_words(lookup512_kernel<C, K>, g, p, words, s, p, words, keys, n, out, hits);
}

// multi-choice lookups: compile-time k for two and three choices
template <int C>
static cudaError_t launch_lookup(const KParams &p, const u64 *words, const u64 *keys, u64 n,
                                 u8 *out, unsigned long long *hits, cudaStream_t s) {
    if (C <= 3) {
        switch (p.k) {
#define BC_LOOKUP_K(k) \
    case k: return launch_lookup_k<C, (C <= 3 ? k : 0)>(p, words, keys, n, out, hits, s);
            BC_LOOKUP_K(4) BC_LOOKUP_K(5) BC_LOOKUP_K(6) BC_LOOKUP_K(7) BC_LOOKUP_K(8)
            BC_LOOKUP_K(9) BC_LOOKUP_K(10) BC_LOOKUP_K(11) BC_LOOKUP_K(12) BC_LOOKUP_K(13)
            BC_LOOKUP_K(14) BC_LOOKUP_K(15) BC_LOOKUP_K(16)
#undef BC_LOOKUP_K
            default: break;
        }
    }
    return launch_lookup_k<C, 0>(p, words, keys, n, out, hits, s);
}

static bool relaxed_pipe_enabled() {  // BC_RELAXED_PIPE=0: the unpipelined tile
    static const bool on = [] {
        const char *e = getenv("BC_RELAXED_PIPE");
        return e == nullptr || atoi(e) != 0;
    }();
    return on;
}

template <int OP, int C>
static cudaError_t launch512(const KParams &p, u64 *words, const u64 *keys, u64 n, u8 *out,
                             unsigned long long *hits, cudaStream_t s) {
    if (OP == OP_CONTAINS && p.fast_random && C == 1 && lookup_pipe_enabled()) {
        return launch_pipe(p, words, keys, n, out, hits, s);
    }
    if (OP == OP_CONTAINS && p.fast_random) {
        return launch_lookup<C>(p, words, keys, n, out, hits, s);
    }
    // pipelined tile for 2..4 choices (double-buffered slices fit 48 KiB)
    constexpr int CR = (C >= 2 && C <= 4) ? C : 2;
    if (OP == OP_INSERT && C == CR && relaxed_pipe_enabled()) {
        const void *fr = (const void *)relaxed512_kernel<CR>;
        unsigned grid = grid_for(fr, kTPB, 0, (n + kTPB - 1) / kTPB);
        if (p.max_ctas && grid > p.max_ctas) grid = p.max_ctas;
        return launch_words(relaxed512_kernel<CR>, grid, p, words, s, p, words, keys, n);
    }
    const void *fn = (const void *)blocks512_kernel<OP, C>;
    unsigned grid = grid_for(fn, kTPB, 0, (n + kTPB - 1) / kTPB);
    if (p.max_ctas && grid > p.max_ctas) grid = p.max_ctas;
    return launch_words(blocks512_kernel<OP, C>, grid, p, words, s, p, words, keys, n, out, hits);
}

cudaError_t launch_relaxed_peers(const KParams &p, u64 *const *parts, int nparts,
                                 const u64 *keys, u64 n, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    if (nparts < 1 || nparts > kMaxParts || !p.fast_random || p.wpb != 8 || p.c < 2 || p.c > 4)
        return cudaErrorInvalidValue;
    PartWords pw{};
    for (int r = 0; r < nparts; ++r) pw.part[r] = parts[r];
    pw.per = (p.num_blocks + nparts - 1) / nparts;
    pw.magic = ~0ull / pw.per;  // floor((2^64 - 1) / per): still exact or one short
    const void *fn = p.c == 2 ? (const void *)relaxed512_peer_kernel<2>
                   : p.c == 3 ? (const void *)relaxed512_peer_kernel<3>
                              : (const void *)relaxed512_peer_kernel<4>;
    unsigned grid = grid_for(fn, kTPB, 0, (n + kTPB - 1) / kTPB);
    if (p.max_ctas && grid > p.max_ctas) grid = p.max_ctas;
    count_launch();
    switch (p.c) {
        case 2: relaxed512_peer_kernel<2><<<grid, kTPB, 0, s>>>(p, pw, keys, n); break;
        case 3: relaxed512_peer_kernel<3><<<grid, kTPB, 0, s>>>(p, pw, keys, n); break;
        default: relaxed512_peer_kernel<4><<<grid, kTPB, 0, s>>>(p, pw, keys, n); break;
    }
    return cudaGetLastError();
}

template <int OP>
static cudaError_t launch512_c(const KParams &p, u64 *words, const u64 *keys, u64 n, u8 *out,
                               unsigned long long *hits, cudaStream_t s) {
    switch (p.c) {
        case 1: return launch512<OP, 1>(p, words, keys, n, out, hits, s);
        case 2: return launch512<OP, 2>(p, words, keys, n, out, hits, s);
        case 3: return launch512<OP, 3>(p, words, keys, n, out, hits, s);
        case 4: return launch512<OP, 4>(p, words, keys, n, out, hits, s);
        case 5: return launch512<OP, 5>(p, words, keys, n, out, hits, s);
        case 6: return launch512<OP, 6>(p, words, keys, n, out, hits, s);
        case 7: return launch512<OP, 7>(p, words, keys, n, out, hits, s);
        case 8: return launch512<OP, 8>(p, words, keys, n, out, hits, s);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_blocks(int op, const KParams &p, u64 *words, const u64 *keys, u64 n, u8 *out,
                          unsigned long long *hits, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    if (p.wpb == 8) {
        return op == OP_CONTAINS ? launch512_c<OP_CONTAINS>(p, words, keys, n, out, hits, s)
                                 : launch512_c<OP_INSERT>(p, words, keys, n, out, hits, s);
    }
    l2_release();
    const void *fn = op == OP_CONTAINS ? (const void *)generic_kernel<OP_CONTAINS>
                                       : (const void *)generic_kernel<OP_INSERT>;
    unsigned grid = grid_for(fn, 256, 0, (n + 255) / 256);
    if (p.max_ctas && grid > p.max_ctas) grid = p.max_ctas;
    if (op == OP_CONTAINS)
        generic_kernel<OP_CONTAINS><<<grid, 256, 0, s>>>(p, words, keys, n, out, hits);
    else
        generic_kernel<OP_INSERT><<<grid, 256, 0, s>>>(p, words, keys, n, out, hits);
    count_launch();
    return cudaGetLastError();
}

bool ordered_window_mode() {  // BC_ORDERED_WINDOW=0: fixed chunks
    static const bool on = [] {
        const char *e = getenv("BC_ORDERED_WINDOW");
        return e == nullptr || atoi(e) != 0;
    }();
    return on;
}

// BC_ORDERED_TILES=0: winners committed one thread per key (insert_fast512)
static bool ordered_tiles() {
    static const bool on = [] {
        const char *e = getenv("BC_ORDERED_TILES");
        return e == nullptr || atoi(e) != 0;
    }();
    return on;
}

template <class Src>
static const void *ordered512_ptr(u32 c) {
    switch (c) {
        case 2: return (const void *)ordered512_kernel<2, Src>;
        case 3: return (const void *)ordered512_kernel<3, Src>;
        case 4: return (const void *)ordered512_kernel<4, Src>;
        case 5: return (const void *)ordered512_kernel<5, Src>;
        case 6: return (const void *)ordered512_kernel<6, Src>;
        case 7: return (const void *)ordered512_kernel<7, Src>;
        default: return (const void *)ordered512_kernel<8, Src>;
    }
}

// BC_ORDERED_ONE=0: the two-array reset-on-win rounds (ordered512_kernel)
bool ordered_one() {
    static const bool on = [] {
        const char *e = getenv("BC_ORDERED_ONE");
        return e == nullptr || atoi(e) != 0;
    }();
    return on;
}

template <class Src>
static const void *ordered1_ptr(u32 c) {
    switch (c) {
        case 2: return (const void *)ordered1_kernel<2, Src>;
        case 3: return (const void *)ordered1_kernel<3, Src>;
        case 4: return (const void *)ordered1_kernel<4, Src>;
        case 5: return (const void *)ordered1_kernel<5, Src>;
        case 6: return (const void *)ordered1_kernel<6, Src>;
        case 7: return (const void *)ordered1_kernel<7, Src>;
        default: return (const void *)ordered1_kernel<8, Src>;
    }
}

u64 ordered_owner_words(u64 num_blocks, u64 slots) {
    // window kernel: two arrays of `slots` u32 claims; fixed-chunk kernel:
    // one array of num_blocks u64 round-tagged claims
    return ordered_window_mode() ? slots : num_blocks;
}

bool ordered_tiles_supported(const KParams &p) {
    return p.fast_random && p.wpb == 8 && p.c >= 2 && p.c <= 8 && ordered_tiles();
}

// Cooperative launch of the sliding-window kernel: the claim arrays (not the
// filter: ordered builds run on filters of any size) persist in L2 when they
// fit, since every pending key reads and claims c random slots per round.
template <class Src>
static cudaError_t launch_window(const KParams &p, u64 *words, const Src *src, const u64 *keys,
                                 u64 n, u64 chunk, u64 *owner, u64 slots, u32 *lists, u64 *lkeys,
                                 u32 *state, unsigned long long *admitted, cudaStream_t s) {
    if (chunk == 0) return cudaErrorInvalidValue;  // no window: the rounds could never admit
    // the append counters state[1..3] start at zero, the round counter
    // state[0] (array parity) carries over
    cudaError_t e = cudaMemsetAsync(state + 1, 0, 3 * sizeof(u32), s);
    if (e != cudaSuccess) return e;
    const bool tile = src != nullptr;
    const bool one = tile && ordered_one();
    const void *fw = one    ? ordered1_ptr<Src>(p.c)
                     : tile ? ordered512_ptr<Src>(p.c)
                            : (const void *)ordered_window_kernel;
    const unsigned grid = grid_for(fw, 256, 0, (chunk + 255) / 256);
    u32 slot_shift = 0;  // identity slots when there is one per block
    if (slots < p.num_blocks) slot_shift = 64u - (u32)__builtin_ctzll(slots);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    size_t bytes = 0;
    float hit = 0.f;
    const size_t claim_bytes = sizeof(u32) * (one ? 1 : 2) * slots;
    // The set-aside is sized to the claims, not to the device maximum: what
    // it takes beyond them is lost to the candidate blocks and the dirty
    // lines of the commits (B200: cfg3 5 395 -> 6 140 Mkeys/s, cfg5 with 2^22
    // slots 5 986 -> 7 661; BC_ORDERED_PERSIST_FIT=0 restores the maximum,
    // BC_ORDERED_PERSIST_MB caps it).
    static const bool fit = [] {
        const char *e = getenv("BC_ORDERED_PERSIST_FIT");
        return e == nullptr || atoi(e) != 0;
    }();
    static const size_t cap_mb = [] {
        const char *e = getenv("BC_ORDERED_PERSIST_MB");
        return e ? (size_t)atoi(e) : (size_t)0;
    }();
    if (l2_window(claim_bytes, &bytes, &hit, fit, cap_mb << 20)) {
        attr[1].id = cudaLaunchAttributeAccessPolicyWindow;
        attr[1].val.accessPolicyWindow.base_ptr = owner;
        attr[1].val.accessPolicyWindow.num_bytes = bytes;
        attr[1].val.accessPolicyWindow.hitRatio = hit;
        attr[1].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        attr[1].val.accessPolicyWindow.missProp = cudaAccessPropertyNormal;
        cfg.numAttrs = 2;
    }
    u32 *own = reinterpret_cast<u32 *>(owner);
    if (!tile) {
        count_launch();
        return cudaLaunchKernelEx(&cfg, ordered_window_kernel, p, words, keys, n, chunk, own,
                                  slots, slot_shift, lists, state);
    }
    // CTA-local pending lists of `cap` entries (24 bytes each, two buffers):
    // the window is spread over as many co-resident CTAs as fit, at least
    // 256 entries per CTA
    e = cudaMemsetAsync(state, 0, 8 * sizeof(u32), s);  // round words, cursor
    if (e == cudaSuccess) e = cudaMemsetAsync(state + 8, 0xff, 4 * sizeof(u32), s);  // minima
    // state[12], ordered1_kernel's tag epoch, carries over from launch to launch
    if (e != cudaSuccess) return e;
    const int sms = (int)sm_count();
    const int minb = one ? ord1_minb((int)p.c) : BC_ORD_MINB;
    u64 ctas = std::max<u64>(1, std::min<u64>((u64)sms * minb, chunk / BC_ORD_NT));
    u32 cap = 0;
    size_t smem = 0;
    for (int it = 0;; ++it) {
        cap = (u32)((chunk + ctas - 1) / ctas);
        // whole tiles, the same number for each of the CTA's warps: a list
        // of 257 entries would cost a ninth tile per round for one key
        if (one && cap >= 128) cap = std::max(256u, (cap + 128u) & ~255u);
        smem = (size_t)cap * 24;
        // static + dynamic shared memory above 48 KB needs the opt-in
        if (cudaFuncSetAttribute(fw, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
            cudaSuccess)
            return cudaErrorInvalidValue;
        int per_sm = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fw, BC_ORD_NT, smem) != cudaSuccess ||
            per_sm < 1)
            return cudaErrorInvalidConfiguration;
        if ((u64)per_sm * sms >= ctas) break;
        if (it == 8) return cudaErrorInvalidConfiguration;
        ctas = (u64)per_sm * sms;  // fewer co-resident CTAs: larger lists, re-check
    }
    cfg.gridDim = dim3((unsigned)ctas);
    cfg.blockDim = dim3(BC_ORD_NT);
    cfg.dynamicSmemBytes = smem;
    static const u32 rel_bits = [] {
        const char *e = getenv("BC_ORDERED_REL_BITS");
        const int v = e ? atoi(e) : (int)kRelBits;
        return (u32)std::min(std::max(v, 1), (int)kRelBits);
    }();
    count_launch();
    switch (p.c) {
#define BC_ORD_C(c)                                                                         \
    case c:                                                                                 \
        if (one)                                                                            \
            return cudaLaunchKernelEx(&cfg, ordered1_kernel<c, Src>, p, words, *src, n,     \
                                      cap, own, slots, slot_shift, state, admitted,         \
                                      rel_bits);                                            \
        return cudaLaunchKernelEx(&cfg, ordered512_kernel<c, Src>, p, words, *src, n, cap,   \
                                  own, slots, slot_shift, state, admitted);
        BC_ORD_C(2) BC_ORD_C(3) BC_ORD_C(4) BC_ORD_C(5) BC_ORD_C(6) BC_ORD_C(7) BC_ORD_C(8)
#undef BC_ORD_C
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_ordered(const KParams &p, u64 *words, const u64 *keys, u64 n, u64 chunk,
                           u64 *owner, u64 slots, u32 *lists, u64 *lkeys, u32 *state,
                           cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    if (ordered_window_mode()) {
        const ArrayKeys src{keys};
        return launch_window<ArrayKeys>(p, words, ordered_tiles_supported(p) ? &src : nullptr,
                                        keys, n, chunk, owner, slots, lists, lkeys, state,
                                        nullptr, s);
    }
    if (chunk == 0) return cudaErrorInvalidValue;
    l2_release();
    const void *fn = (const void *)ordered_kernel;
    const unsigned grid = grid_for(fn, 256, 0, (chunk + 255) / 256);
    KParams pp = p;
    void *args[] = {(void *)&pp, (void *)&words, (void *)&keys, (void *)&n,
                    (void *)&chunk, (void *)&owner, (void *)&lists, (void *)&state};
    cudaError_t e = cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(256), args, 0, s);
    count_launch();
    return e;
}

cudaError_t launch_ordered_qgrams(const KParams &p, u64 *words, const u8 *seq, u64 nwin, int q,
                                  int canonical, RecSpec rec, u64 chunk, u64 *owner, u64 slots,
                                  u32 *lists, u64 *lkeys, u32 *state,
                                  unsigned long long *count, cudaStream_t s) {
    if (nwin == 0) return cudaSuccess;
    if (!ordered_window_mode() || !ordered_tiles_supported(p)) return cudaErrorInvalidValue;
    SeqKeys src;
    src.seq = seq;
    src.rec = rec;
    src.q = (u32)q;
    src.canonical = (u32)canonical;
    src.qmask = q == 32 ? ~0ull : ((1ull << (2 * q)) - 1ull);
    return launch_window<SeqKeys>(p, words, &src, nullptr, nwin, chunk, owner, slots, lists,
                                  lkeys, state, count, s);
}

cudaError_t launch_flat(int op, const KParams &p, u64 *words, const u64 *keys, u64 n, u8 *out,
                        unsigned long long *hits, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const void *fn = op == OP_CONTAINS ? (const void *)flat_kernel<OP_CONTAINS>
                                       : (const void *)flat_kernel<OP_INSERT>;
    const unsigned grid = grid_for(fn, kTPB, 0, (n + kTPB - 1) / kTPB);
    if (op == OP_INSERT)  // a bit array that fits L2 keeps its dirty lines there:
        // 96 MiB, 2^26 keys, k = 12: 10.0 -> 16.0 Gkeys/s (bench_next.py)
        return launch_words(flat_kernel<OP_INSERT>, grid, p, words, s, p, words, keys, n, out,
                            hits);
    // lookups are faster without the window (19.6 vs 15.6 Gkeys/s, same run)
    l2_release();
    flat_kernel<OP_CONTAINS><<<grid, kTPB, 0, s>>>(p, words, keys, n, out, hits);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_histogram(const u64 *words, u64 num_blocks, int block_bits,
                             unsigned long long *counts, cudaStream_t s) {
    if (num_blocks == 0) return cudaSuccess;
    if (block_bits == 512) {
        const unsigned grid =
            grid_for((const void *)hist512_kernel, 256, 0, (num_blocks * 4 + 255) / 256);
        hist512_kernel<<<grid, 256, 0, s>>>(words, num_blocks, counts);
    } else {
        const u32 wpb = block_bits >= 64 ? (u32)(block_bits / 64) : 1u;
        const unsigned grid =
            grid_for((const void *)hist_generic_kernel, 256, 0, (num_blocks + 255) / 256);
        hist_generic_kernel<<<grid, 256, 0, s>>>(words, num_blocks, wpb, counts);
    }
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_eval_hash(DevHash h, const u64 *keys, u64 n, u64 *out, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const unsigned grid = grid_for((const void *)eval_hash_kernel, 256, 0, (n + 255) / 256);
    eval_hash_kernel<<<grid, 256, 0, s>>>(h, keys, n, out);
    count_launch();
    return cudaGetLastError();
}

}  // namespace bc
