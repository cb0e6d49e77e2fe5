// Host-side launchers shared between the kernel translation units and the C ABI.
#pragma once

#include <cuda_runtime.h>

#include "common.cuh"

namespace bc {

enum Op : int { OP_CONTAINS = 0, OP_INSERT = 1 };

// Kernel launch accounting (bc_launch_count()).
void count_launch(unsigned n = 1);

// Demote the filter words' persisting L2 lines to normal and give back the
// set-aside: on the current device (teardown, launches without a window), or
// on every device this process used (bc_l2_release).
void l2_release();
void l2_release_all();

// Persistent-grid size: min(work_ctas, SMs x resident CTAs of `kernel`).
unsigned grid_for(const void *kernel, int threads, size_t dyn_smem, unsigned long long work_ctas);

// ---- blocked family (filter_kernels.cu) ---------------------------------------
// One launch over n keys.  OP_INSERT with c == 1 is an order-free OR; with
// c >= 2 it is the relaxed (atomic) insert -- the caller bounds n per launch.
cudaError_t launch_blocks(int op, const KParams &p, u64 *words, const u64 *keys, u64 n,
                          u8 *out, unsigned long long *hits, cudaStream_t s);

// Relaxed insert (c in 2..4, 512-bit blocks, random strategy) into a filter
// partitioned over nparts replicas: rank r's replica holds the authoritative
// words of blocks [r*per, (r+1)*per), per = ceil(M / nparts); parts[r] is this
// process's address of rank r's replica (peer memory).  p.max_ctas bounds the
// keys in flight (256 per CTA).
cudaError_t launch_relaxed_peers(const KParams &p, u64 *const *parts, int nparts,
                                 const u64 *keys, u64 n, cudaStream_t s);

// Exact stream-order insert for c >= 2 (claim rounds, one cooperative launch).
// owner: the claim arrays, ordered_owner_words(num_blocks, slots) u64 words,
// all-ones before the first launch (slots == num_blocks: one per block, else
// a power of two, blocks hashed onto slots).  n < 2^32 - 1 per launch.
// lists: 2 * chunk u32 stream indices; lkeys: 2 * chunk u64 keys (the
// pending lists of the tiled kernel).  chunk == 0 is rejected.
bool ordered_window_mode();
bool ordered_one();  // one claim array, same-round commits (ordered1_kernel)
bool ordered_tiles_supported(const KParams &p);
u64 ordered_owner_words(u64 num_blocks, u64 slots);
cudaError_t launch_ordered(const KParams &p, u64 *words, const u64 *keys, u64 n, u64 chunk,
                           u64 *owner, u64 slots, u32 *lists, u64 *lkeys, u32 *state,
                           cudaStream_t s);

// ---- standard (flat) kind --------------------------------------------------------
cudaError_t launch_flat(int op, const KParams &p, u64 *words, const u64 *keys, u64 n, u8 *out,
                        unsigned long long *hits, cudaStream_t s);

// ---- utilities -------------------------------------------------------------------
cudaError_t launch_histogram(const u64 *words, u64 num_blocks, int block_bits,
                             unsigned long long *counts, cudaStream_t s);
cudaError_t launch_eval_hash(DevHash h, const u64 *keys, u64 n, u64 *out, cudaStream_t s);

// ---- q-grams (qgram_kernels.cu) ----------------------------------------------------
// Valid windows per tile of kQgramTile windows, then an exclusive scan.
constexpr int kQgramThreads = 256;
constexpr int kQgramPerThread = 8;
constexpr int kQgramTile = kQgramThreads * kQgramPerThread;
// Records of a q-gram sequence: len > 0 means consecutive records of len
// bytes (windows never cross them), phase = offset of seq[0] in its record.
struct RecSpec {
    u64 len = 0;
    u64 phase = 0;
};
cudaError_t launch_qgram_offsets(const u8 *seq, u64 len, int q, RecSpec rec, u64 *tile_off,
                                 u64 ntiles, unsigned long long *total, cudaStream_t s);
cudaError_t launch_qgram_encode(const u8 *seq, u64 len, int q, int canonical, RecSpec rec,
                                const u64 *tile_off, u64 *keys, cudaStream_t s);
// Fused: encode + (insert | contains).  tile_off may be NULL when no ordered
// output is needed (inserts, count-only lookups).
cudaError_t launch_qgram_blocks(int op, const KParams &p, u64 *words, const u8 *seq, u64 len,
                                int q, int canonical, RecSpec rec, const u64 *tile_off, u8 *out,
                                unsigned long long *hits, unsigned long long *count,
                                cudaStream_t s);

// Exact stream-order insert of the q-gram windows of seq (nwin windows, i.e.
// seq holds nwin + q - 1 bytes): == launch_ordered on encode_qgrams(seq),
// keys encoded on the fly (keysrc.cuh), window index = stream priority.
// Needs ordered_tiles_supported(p).  *count += windows inserted (valid ones).
cudaError_t launch_ordered_qgrams(const KParams &p, u64 *words, const u8 *seq, u64 nwin, int q,
                                  int canonical, RecSpec rec, u64 chunk, u64 *owner, u64 slots,
                                  u32 *lists, u64 *lkeys, u32 *state,
                                  unsigned long long *count, cudaStream_t s);

// Exact stream-order insert of small filters as a dataflow (ordered_ticket.cu):
// per-block tickets from a stable sort of (block, key) pairs, then keys commit
// as soon as every earlier key sharing a block is done.  c in 2..8, 512-bit
// blocks, random strategy, up to BC_TICKET_MAX_BLOCKS blocks (default 2^20,
// 2^21 for c >= 3).
bool ordered_ticket_supported(const KParams &p);
cudaError_t launch_ordered_ticket(const KParams &p, u64 *words, const u64 *keys, u64 n,
                                  cudaStream_t s);
cudaError_t launch_ordered_ticket_qgrams(const KParams &p, u64 *words, const u8 *seq, u64 nwin,
                                         int q, int canonical, RecSpec rec,
                                         unsigned long long *count, cudaStream_t s);

// numpy PCG64 stream (default_rng(seed).integers(0, 2**64, uint64)) from a
// seeded (state, inc): outputs [offset, offset+n), then & and_mask | or_mask.
cudaError_t launch_pcg64_fill(u64 state_hi, u64 state_lo, u64 inc_hi, u64 inc_lo, u64 offset,
                              u64 n, u64 and_mask, u64 or_mask, u64 *out, cudaStream_t s);

// In-place exclusive scan of n u64 by one CTA (*total = sum, nullable).
cudaError_t launch_scan(u64 *v, u64 n, unsigned long long *total, cudaStream_t s);

// ---- region-partitioned single-choice insert (partition_insert.cu) -----------------
bool partition_supported(const KParams &p);
u32 partition_regions(const KParams &p);
size_t partition_scratch_bytes(const KParams &p, u64 n);
cudaError_t launch_partitioned_insert(const KParams &p, u64 *words, const u64 *keys, u64 n,
                                      void *scratch, cudaStream_t s);

}  // namespace bc
