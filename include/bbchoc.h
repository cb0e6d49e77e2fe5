/*
 * bbchoc.h -- C ABI of the B200 (sm_100a) blocked-Bloom-with-choices hot path.
 *
 * This is the drop-in boundary for the reference's compiled layer
 * (pkg/src/blowchoc/_kernels.py).  The reference's Python filter API
 * (Filter.insert_many / contains_many / count_hits, filters.py:377-398)
 * crosses into numba at exactly four call sites; each one maps to an entry
 * point here:
 *
 *   _kernels.insert_blocks   (filters.py:383-384, _kernels.py:112-174) -> bc_insert
 *   _kernels.contains_blocks (filters.py:394,     _kernels.py:177-211) -> bc_contains
 *   _kernels.insert_flat     (filters.py:381,     _kernels.py:214-222) -> bc_insert
 *   _kernels.contains_flat   (filters.py:392,     _kernels.py:225-237) -> bc_contains
 *
 * The numba kernels take the flat tuple built by Filter._kernel_args() and
 * _cost_args() (filters.py:347-375) on every call.  Here that tuple is
 * handed over once, as a bc_filter_desc, and turned into a bc_filter handle
 * holding the derived device constants (fast-modulo magics, the cost rank
 * table) and the scratch of the ordered insert.  Every later call takes the
 * handle plus plain pointers and sizes.
 *
 * The fused DNA k-mer path replaces the composition
 * insert_many(encode_qgrams(enc, seq)) / contains_many(encode_qgrams(enc, seq))
 * (io.py:158-177 feeding filters.py:377-398; demos/05_dna_qgrams.py:29-52)
 * with bc_insert_qgrams / bc_contains_qgrams, and encode_qgrams itself with
 * bc_encode_qgrams.  bc_block_histogram replaces block_load_histogram's
 * popcount tally (analysis.py:135-146); bc_route replaces route_many
 * (sharding.py:50-51, filters.py:400-402).
 *
 * Conventions
 *  - Return 0 on success, a negative BC_E* code on error; bc_last_error()
 *    gives a thread-local message.  Nothing is thrown across the ABI.
 *  - d_* pointers are device pointers (cudaMalloc / torch), h_* pointers
 *    are host pointers (pinned or pageable).  `stream` is a cudaStream_t
 *    (NULL = legacy default stream).  All calls are stream-ordered and do
 *    not synchronise unless documented (the *_host entry points return
 *    after their results are in host memory).
 *  - Like the reference kernels, inserts require a single writer per shard;
 *    lookups are read-only and may run concurrently.
 */
#ifndef BBCHOC_H
#define BBCHOC_H

#include <stdint.h>

#if defined(__GNUC__)
#define BC_API __attribute__((visibility("default")))
#else
#define BC_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define BC_OK 0
#define BC_EINVAL (-1)  /* bad argument (mirrors ConfigError / ValueError) */
#define BC_ECUDA (-2)   /* CUDA runtime error */
#define BC_ENOMEM (-3)  /* device or pinned allocation failed */
#define BC_EUNSUP (-4)  /* geometry outside what the kernels support */

#define BC_KIND_STANDARD 0
#define BC_KIND_BLOCKED 1
#define BC_KIND_BLOWCHOC 2

#define BC_INSERT_ORDERED 0 /* bit-identical to the reference's stream order */
#define BC_INSERT_RELAXED 1 /* atomic OR, <= M/2 keys in flight per launch  */

#define BC_MAX_CHOICES 8

/* POD mirror of Filter._kernel_args() + _cost_args() (filters.py:347-375).
 * Hash modes and shifts are NOT passed: they are a function of each range
 * (hashing.py:65-76) and are re-derived, exactly as the reference's
 * hash_branch does. */
typedef struct bc_filter_desc {
    int32_t kind;            /* BC_KIND_*                                       */
    int32_t k;               /* bit-address functions per key                   */
    int32_t choices;         /* c: 0 standard, 1 blocked, 2..8 blowchoc          */
    int32_t strategy;        /* 0 random, 1 distinct                            */
    int32_t block_bits;      /* B: multiple of 64, or 8/16/32 (toy widths)       */
    int32_t reserved0;
    uint64_t num_blocks;     /* M                                               */
    uint64_t shards;         /* T (M % T == 0)                                  */
    uint64_t shard_a;        /* h0 multiplier, range T                          */
    uint64_t block_a[BC_MAX_CHOICES]; /* h_1..h_c multipliers, range M/T        */
    const uint64_t *bit_a;   /* host, k multipliers                              */
    const uint64_t *bit_b;   /* host, k ranges (B, or B-i for distinct, m for standard) */
    int32_t cost_code;       /* 0 exp, 1 mix, 2 la (ignored for c < 2)          */
    int32_t reserved1;
    double cost_param;       /* beta / sigma / mu                               */
    /* Optional host table of (B+1)*(k+1) float64 costs, cost[j*(k+1)+a].  NULL:
     * the library evaluates the reference formulas (_kernels.py:100-109). */
    const double *cost_table;
} bc_filter_desc;

typedef struct bc_filter bc_filter;

/* Build a handle (uploads the per-filter constants to the current device). */
BC_API int bc_filter_create(const bc_filter_desc *desc, bc_filter **out);
BC_API void bc_filter_destroy(bc_filter *f);

/* Batched insertion of n keys into d_words (num_blocks*wpb uint64 words).
 * mode: BC_INSERT_ORDERED (exact reference semantics, any c) or
 * BC_INSERT_RELAXED (c >= 2 only differs).  Replaces insert_blocks /
 * insert_flat. */
BC_API int bc_insert(bc_filter *f, uint64_t *d_words, const uint64_t *d_keys, uint64_t n,
              int mode, void *stream);

/* Batched membership.  d_out (nullable) receives 0/1 per key; d_hits
 * (nullable) is incremented by the number of hits (count_hits).
 * Replaces contains_blocks / contains_flat. */
BC_API int bc_contains(bc_filter *f, const uint64_t *d_words, const uint64_t *d_keys, uint64_t n,
                uint8_t *d_out, unsigned long long *d_hits, void *stream);

/* Host-buffer variants: keys are read from, and answers written to, host
 * memory; the library stages through its pinned buffers (or reads pinned
 * user memory directly) and overlaps copies with the kernels.  They return
 * once the work is complete. */
BC_API int bc_insert_host(bc_filter *f, uint64_t *d_words, const uint64_t *h_keys, uint64_t n,
                   int mode, void *stream);
BC_API int bc_contains_host(bc_filter *f, const uint64_t *d_words, const uint64_t *h_keys,
                     uint64_t n, uint8_t *h_out, unsigned long long *h_hits, void *stream);

/* 2-bit canonical q-gram keys of a device byte sequence (io.py:158-177).
 * Windows touching any byte outside ACGTacgt are skipped, so several records
 * concatenated with a separator byte (e.g. '\n') never produce a window that
 * spans two records.  record_len > 0 declares the sequence to be consecutive
 * records of record_len bytes with no separator (a reads matrix): windows that
 * cross a record boundary are skipped too.  d_keys must hold len-q+1 keys;
 * *d_count receives the number written. */
BC_API int bc_encode_qgrams(const uint8_t *d_seq, uint64_t len, int q, int canonical,
                            uint64_t record_len, uint64_t *d_keys, unsigned long long *d_count,
                            void *stream);

/* Fused encode + insert: == bc_insert(f, words, encode_qgrams(seq), mode).
 * *d_count (nullable) receives the number of keys (valid windows) inserted. */
BC_API int bc_insert_qgrams(bc_filter *f, uint64_t *d_words, const uint8_t *d_seq, uint64_t len,
                            int q, int canonical, uint64_t record_len, int mode,
                            unsigned long long *d_count, void *stream);

/* Fused encode + lookup: == bc_contains(f, words, encode_qgrams(seq)).
 * d_out (nullable) must hold len-q+1 bytes; *d_count (nullable) receives the
 * number of valid windows (= number of answers written). */
BC_API int bc_contains_qgrams(bc_filter *f, const uint64_t *d_words, const uint8_t *d_seq,
                              uint64_t len, int q, int canonical, uint64_t record_len,
                              uint8_t *d_out, unsigned long long *d_count,
                              unsigned long long *d_hits, void *stream);

/* counts[j] += number of blocks holding j set bits, j in [0, block_bits]. */
BC_API int bc_block_histogram(const uint64_t *d_words, uint64_t num_blocks, int block_bits,
                       unsigned long long *d_counts, void *stream);

/* Shard index h0(x) per key (route_many). */
BC_API int bc_route(bc_filter *f, const uint64_t *d_keys, uint64_t n, uint64_t *d_shard,
             void *stream);

/* Generic ((a*x mod 2^64) folded) mod b over a key array (eval_hash_many,
 * hashing.py:90-100). */
BC_API int bc_eval_hash(uint64_t a, uint64_t b, const uint64_t *d_keys, uint64_t n,
                 uint64_t *d_out, void *stream);

/* The reference's key streams on the device: outputs [offset, offset+n) of
 * numpy's default_rng(seed).integers(0, 2**64, dtype=uint64) -- PCG64 from
 * the seeded 128-bit (state, inc) that numpy reports -- each masked as
 * (v & and_mask) | or_mask.  even_keys: and_mask = ~1; odd_keys: or_mask = 1
 * (analysis.py:34-43). */
BC_API int bc_pcg64_fill(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                         uint64_t offset, uint64_t n, uint64_t and_mask, uint64_t or_mask,
                         uint64_t *d_out, void *stream);

/* Host-side query output of the CLI (cli.py:141-142): writes one line
 * "<decimal key>\t<0|1>\n" per key into h_out (at most 23 * n bytes, which
 * out_cap must cover) and stores the byte count in *written. */
BC_API int bc_format_answers(const uint64_t *h_keys, const uint8_t *h_answers, uint64_t n,
                             char *h_out, uint64_t out_cap, uint64_t *written);

/* Host-side text key ingestion (read_keys(..., "text"), io.py:206-223): parses
 * the complete lines of h_text[0, len) -- one decimal key per line, surrounding
 * ASCII whitespace and blank lines ignored, an optional sign and single
 * underscores between digits accepted, as Python's int() does -- into h_keys
 * (capacity cap).  Parsing stops after the last '\n' (the caller carries the
 * partial tail) or when cap keys are stored.  *consumed = bytes of h_text
 * used, *lines = lines used, *n_keys = keys stored.  A line that is not an
 * integer, or whose value is outside [0, 2^64), stops the parse with
 * BC_EINVAL; *lines is then the 0-based index of that line among the ones
 * given (the caller re-reads it to word the error). */
BC_API int bc_parse_keys_text(const char *h_text, uint64_t len, uint64_t *h_keys, uint64_t cap,
                              uint64_t *consumed, uint64_t *lines, uint64_t *n_keys);

/* Host-side FASTA ingestion (read_keys(..., "fasta"), io.py:226-242 _read_fasta,
 * and the CLI's build from FASTA): joins the sequence lines of every record of
 * h_text[0, len) -- lines split at '\n', stripped of surrounding ASCII
 * whitespace, blank lines skipped, a line starting with '>' closing the record
 * in progress -- into h_out, consecutive records separated by one `sep` byte (a
 * non-ACGT byte, so no q-gram window spans two records: the input of
 * bc_insert_qgrams / bc_contains_qgrams).  Output is appended at
 * h_out[out_len_in...]; the caller sizes h_out for out_len_in + len + 1 bytes.
 * *state carries bit 0 "a header was seen" and bit 1 "the record at the end of
 * h_out is still open" from call to call; h_out[0, out_len_in) is the output so
 * far (closed records, then the open one's sequence if bit 1 is set; a call
 * may also start from an empty buffer that holds only the carried open
 * record).  rec_ends[i] = end
 * offset in h_out of the i-th record closed by this call.  When the table is
 * full (*n_recs == rec_cap) the call stops before the line that would close
 * another record, state unchanged: call again from h_text + *consumed with more
 * table space (at the end of the text too: with len 0 and at_eof, to close
 * the last record).  Without at_eof,
 * parsing stops after the last '\n' (*consumed bytes used; the caller carries
 * the partial line); with it the last line needs no '\n' and an open record is
 * closed.  Sequence before the first header is BC_EINVAL, as the reference's
 * KeyFormatError. */
BC_API int bc_fasta_join(const char *h_text, uint64_t len, int at_eof, uint8_t sep,
                         uint32_t *state, uint8_t *h_out, uint64_t out_len_in,
                         uint64_t *out_len, uint64_t *rec_ends, uint64_t rec_cap,
                         uint64_t *n_recs, uint64_t *consumed);

/* ---- multi-GPU replica merge over peer memory (distributed.py) ----------------
 * CUDA IPC mapping of a device buffer for the other ranks: the 64-byte handle
 * of the allocation holding d_ptr and d_ptr's offset in it (torch's caching
 * allocator hands out interior pointers).  bc_ipc_import maps a peer's
 * allocation on the current device (lazy peer access) and returns the
 * buffer's address there; bc_ipc_close unmaps it. */
BC_API int bc_ipc_export(const void *d_ptr, void *handle, uint64_t *offset);
BC_API int bc_ipc_import(const void *handle, uint64_t offset, void **d_ptr);
BC_API int bc_ipc_close(void *d_ptr, uint64_t offset);

/* Words per rank range of the merge: ceil(nwords / world) rounded up to 32. */
BC_API int bc_peer_span(uint64_t nwords, int world, uint64_t *span);

/* Bitwise-OR all-reduce of `world` replicas of nwords words, this rank's
 * share: ORs word range `rank` of every replica (h_peer_words: host array of
 * the replicas' addresses on this device, own one included) and stores the
 * result into that range of every replica -- one kernel, loads and stores
 * over NVLink.  Ranges of different ranks are disjoint and no kernel waits on
 * another; the caller runs every rank's call between two cross-rank barriers
 * (all replicas written before, all calls finished after).  Replaces the
 * NCCL all-to-all + OR + all-gather of the order-free multi-GPU build. */
BC_API int bc_or_allreduce_peers(uint64_t *const *h_peer_words, int world, int rank,
                                 uint64_t nwords, void *stream);

/* Relaxed insert of this rank's key slice into a filter PARTITIONED over the
 * ranks' replicas (the multi-GPU build of multi-choice filters,
 * distributed.py): rank r's replica holds the authoritative words of blocks
 * [r*per, (r+1)*per), per = ceil(M / nparts); h_parts is a host array of the
 * replicas' addresses on this device (own one included; peers mapped with
 * bc_ipc_import).  Each key reads its candidates and ORs its mask into the
 * chosen block in the owner's replica, over NVLink when remote -- one kernel,
 * no separate exchange.  keys_in_flight bounds this rank's keys in flight
 * (0: M/2); the caller passes its share of M/2 so the whole build keeps the
 * relaxed tolerance.  All ranks' calls run between two cross-rank barriers;
 * an all-gather of the ranges then replicates the filter.  c in 2..4,
 * 512-bit blocks, random strategy (BC_EUNSUP otherwise). */
BC_API int bc_insert_peers(bc_filter *f, uint64_t *const *h_parts, int nparts,
                           const uint64_t *d_keys, uint64_t n, uint64_t keys_in_flight,
                           void *stream);

/* Thread-local description of the last error on this thread. */
BC_API const char *bc_last_error(void);

/* Number of kernels this library has launched (process-wide counter). */
BC_API unsigned long long bc_launch_count(void);

/* Library version string. */
BC_API const char *bc_version(void);

/* Filters that fit in L2 are launched with their words marked L2-persisting
 * (BC_L2_PERSIST=0 disables).  This demotes the persisting lines and returns
 * the set-aside on the current device; call it at teardown (the Python layer
 * does so at exit).  Launches that do not use the window call it themselves. */
BC_API void bc_l2_release(void);

#ifdef __cplusplus
}
#endif

#endif /* BBCHOC_H */
