/*
 * bbchoc_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, single-key-at-a-time restatement of the reference's compiled
 * hot loops (pkg/src/blowchoc/_kernels.py) and of its q-gram encoder
 * (pkg/src/blowchoc/io.py:126-177).  It exists to CHECK the CUDA path
 * (tests/, __graft_entry__.smoke(), bench.py's cpu_baseline leg and the
 * `--impl reference` arm).  Nothing in paper_2501_18977_b200/ links or
 * calls it.
 *
 * Parity pin: tests/test_oracle_golden.py compares every entry point below
 * against golden vectors produced by the reference itself
 * (tests/golden/make_golden.py imports /root/reference/pkg/src/blowchoc).
 *
 * Argument order of the four filter loops follows the reference's numba
 * signatures (_kernels.py:113-116, 178-180, 215, 226) with array lengths
 * made explicit.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef uint64_t u64;
typedef int64_t i64;

enum { MOD_ODD = 0, SHIFT_POW2 = 1, XOR_EVEN = 2 }; /* hashing.py:18-21 */

/* _kernels.py:61-70: multiply (wrapping mod 2^64) then one of three folds */
static inline u64 orc_hval(u64 a, u64 x, u64 b, i64 mode, u64 shift)
{
    u64 ax = a * x;
    if (mode == MOD_ODD)
        return ax % b;
    if (mode == SHIFT_POW2)
        return (ax >> shift) % b;
    return (ax ^ (ax >> shift)) % b;
}

u64 orc_hash(u64 a, u64 x, u64 b, i64 mode, u64 shift)
{
    return orc_hval(a, x, b, mode, shift);
}

/* _kernels.py:73-97: k in-block addresses; distinct = dynamic insertion
 * sort with the bump-past-chosen rule (hashing.py:181-200). */
static void orc_fill_addrs(u64 x, const u64 *bit_a, const u64 *bit_b,
                           const i64 *bit_mode, const u64 *bit_shift, int k,
                           int strategy, i64 *addrs)
{
    if (strategy == 0) {
        for (int i = 0; i < k; ++i)
            addrs[i] = (i64)orc_hval(bit_a[i], x, bit_b[i], bit_mode[i], bit_shift[i]);
        return;
    }
    for (int i = 0; i < k; ++i) {
        i64 v = (i64)orc_hval(bit_a[i], x, bit_b[i], bit_mode[i], bit_shift[i]);
        int pos = 0;
        for (int t = 0; t < i; ++t) {
            if (addrs[t] <= v) {
                ++v;
                pos = t + 1;
            } else {
                break;
            }
        }
        for (int t = i; t > pos; --t)
            addrs[t] = addrs[t - 1];
        addrs[pos] = v;
    }
}

/* _kernels.py:100-109 (and filters.py:40-62): float64 cost of a candidate */
static inline double orc_cost(u64 j, u64 a, double kf, int code, double param,
                              double quarter, double half)
{
    double jf = (double)j, af = (double)a;
    if (code == 0)
        return pow(param, jf / quarter) + af / kf;
    if (code == 1)
        return param * kf * pow(jf / half, kf) + af;
    return kf * pow((jf + param * kf) / half, kf) + af;
}

double orc_cost_value(u64 j, u64 a, int k, int code, double param, int block_bits)
{
    return orc_cost(j, a, (double)k, code, param, block_bits / 4.0, block_bits / 2.0);
}

/* _kernels.py:112-174: insertion in stream order. */
void orc_insert_blocks(u64 *words, const u64 *keys, u64 n,
                       u64 shard_a, u64 shard_b, i64 shard_mode, u64 shard_shift,
                       u64 wps, const u64 *block_a, int c, u64 block_b,
                       i64 block_mode, u64 block_shift, const u64 *bit_a,
                       const u64 *bit_b, const i64 *bit_mode, const u64 *bit_shift,
                       int k, int strategy, int wpb, int cost_code,
                       double cost_param, double quarter, double half)
{
    i64 *addrs = malloc(sizeof(i64) * (size_t)k);
    u64 *mask = malloc(sizeof(u64) * (size_t)wpb);
    u64 bases[8];
    double kf = (double)k;
    for (u64 n_i = 0; n_i < n; ++n_i) {
        u64 x = keys[n_i];
        u64 shard_base = orc_hval(shard_a, x, shard_b, shard_mode, shard_shift) * wps;
        orc_fill_addrs(x, bit_a, bit_b, bit_mode, bit_shift, k, strategy, addrs);
        memset(mask, 0, sizeof(u64) * (size_t)wpb);
        for (int i = 0; i < k; ++i)
            mask[addrs[i] >> 6] |= (u64)1 << (addrs[i] & 63);
        if (c == 1) {
            u64 base = shard_base +
                       orc_hval(block_a[0], x, block_b, block_mode, block_shift) * (u64)wpb;
            for (int w = 0; w < wpb; ++w)
                words[base + w] |= mask[w];
            continue;
        }
        for (int ci = 0; ci < c; ++ci)
            bases[ci] = shard_base +
                        orc_hval(block_a[ci], x, block_b, block_mode, block_shift) * (u64)wpb;
        int best = 0, noop = 0;
        double best_cost = INFINITY;
        for (int ci = 0; ci < c; ++ci) {
            u64 j = 0, present = 0;
            for (int w = 0; w < wpb; ++w) {
                u64 wv = words[bases[ci] + w];
                j += (u64)__builtin_popcountll(wv | mask[w]);
                present += (u64)__builtin_popcountll(wv);
            }
            u64 a = j - present;
            if (a == 0) {
                noop = 1;
                break;
            }
            double cost = orc_cost(j, a, kf, cost_code, cost_param, quarter, half);
            if (cost < best_cost) {
                best_cost = cost;
                best = ci;
            }
        }
        if (!noop)
            for (int w = 0; w < wpb; ++w)
                words[bases[best] + w] |= mask[w];
    }
    free(addrs);
    free(mask);
}

/* _kernels.py:177-211: membership, stop at first unset bit / first passing
 * choice.  Writes out[i] in {0,1}; returns the number of hits. */
u64 orc_contains_blocks(const u64 *words, const u64 *keys, u64 n,
                        u64 shard_a, u64 shard_b, i64 shard_mode, u64 shard_shift,
                        u64 wps, const u64 *block_a, int c, u64 block_b,
                        i64 block_mode, u64 block_shift, const u64 *bit_a,
                        const u64 *bit_b, const i64 *bit_mode, const u64 *bit_shift,
                        int k, int strategy, int wpb, uint8_t *out)
{
    i64 *addrs = malloc(sizeof(i64) * (size_t)k);
    u64 hits = 0;
    for (u64 n_i = 0; n_i < n; ++n_i) {
        u64 x = keys[n_i];
        u64 shard_base = orc_hval(shard_a, x, shard_b, shard_mode, shard_shift) * wps;
        if (strategy == 1)
            orc_fill_addrs(x, bit_a, bit_b, bit_mode, bit_shift, k, strategy, addrs);
        int found = 0;
        for (int ci = 0; ci < c && !found; ++ci) {
            u64 base = shard_base +
                       orc_hval(block_a[ci], x, block_b, block_mode, block_shift) * (u64)wpb;
            int ok = 1;
            for (int i = 0; i < k; ++i) {
                i64 f = strategy == 1
                            ? addrs[i]
                            : (i64)orc_hval(bit_a[i], x, bit_b[i], bit_mode[i], bit_shift[i]);
                if (((words[base + (u64)(f >> 6)] >> (f & 63)) & 1) == 0) {
                    ok = 0;
                    break;
                }
            }
            found = ok;
        }
        if (out)
            out[n_i] = (uint8_t)found;
        hits += (u64)found;
    }
    free(addrs);
    return hits;
}

/* _kernels.py:214-222 */
void orc_insert_flat(u64 *words, const u64 *keys, u64 n, const u64 *bit_a, int k,
                     u64 flat_b, i64 flat_mode, u64 flat_shift)
{
    for (u64 n_i = 0; n_i < n; ++n_i)
        for (int i = 0; i < k; ++i) {
            u64 f = orc_hval(bit_a[i], keys[n_i], flat_b, flat_mode, flat_shift);
            words[f >> 6] |= (u64)1 << (f & 63);
        }
}

/* _kernels.py:225-237 */
u64 orc_contains_flat(const u64 *words, const u64 *keys, u64 n, const u64 *bit_a,
                      int k, u64 flat_b, i64 flat_mode, u64 flat_shift, uint8_t *out)
{
    u64 hits = 0;
    for (u64 n_i = 0; n_i < n; ++n_i) {
        int ok = 1;
        for (int i = 0; i < k; ++i) {
            u64 f = orc_hval(bit_a[i], keys[n_i], flat_b, flat_mode, flat_shift);
            if (((words[f >> 6] >> (f & 63)) & 1) == 0) {
                ok = 0;
                break;
            }
        }
        if (out)
            out[n_i] = (uint8_t)ok;
        hits += (u64)ok;
    }
    return hits;
}

/* io.py:126-177: 2-bit q-gram codes (A=0,C=1,G=2,T=3, lower case too, first
 * base most significant); windows touching any other byte are skipped;
 * canonical = min(code, reverse complement).  Returns the number of keys
 * written to out (capacity >= len - q + 1). */
u64 orc_encode_qgrams(const uint8_t *seq, u64 len, int q, int canonical, u64 *out)
{
    if (len < (u64)q)
        return 0;
    u64 qmask = q == 32 ? ~(u64)0 : (((u64)1 << (2 * q)) - 1);
    u64 cnt = 0, code = 0, rc = 0;
    int run = 0; /* valid bases ending at position i */
    for (u64 i = 0; i < len; ++i) {
        int v;
        switch (seq[i]) {
        case 'A': case 'a': v = 0; break;
        case 'C': case 'c': v = 1; break;
        case 'G': case 'g': v = 2; break;
        case 'T': case 't': v = 3; break;
        default: v = -1;
        }
        if (v < 0) {
            run = 0;
            continue;
        }
        code = ((code << 2) | (u64)v) & qmask; /* first base most significant */
        /* reverse complement: complement of the newest base enters on top */
        rc = (rc >> 2) | ((u64)(3 - v) << (2 * q - 2));
        if (++run < q)
            continue;
        out[cnt++] = (canonical && rc < code) ? rc : code;
    }
    return cnt;
}

/* Block-load tally (analysis.py:135-146): counts[j] = blocks with j set bits. */
void orc_block_histogram(const u64 *words, u64 num_blocks, int wpb, u64 *counts)
{
    for (u64 b = 0; b < num_blocks; ++b) {
        u64 s = 0;
        for (int w = 0; w < wpb; ++w)
            s += (u64)__builtin_popcountll(words[b * (u64)wpb + (u64)w]);
        counts[s]++;
    }
}

/* ---------------------------------------------------------------------------
 * Multi-threaded drivers for the CPU baseline.  These reproduce the
 * reference's own parallel mechanisms: read-only chunked queries on a
 * thread pool (analysis.py:96-107, cli.py:133-140) and, for single-choice
 * filters only, order-free OR insertion (the result is bit-identical to
 * stream order because OR commutes, _kernels.py:142-147).
 * ------------------------------------------------------------------------- */
typedef struct {
    const u64 *words;
    u64 *wwords;
    const u64 *keys;
    u64 n;
    u64 shard_a, shard_b, shard_shift, wps, block_b, block_shift;
    i64 shard_mode, block_mode;
    const u64 *block_a;
    int c, k, strategy, wpb;
    const u64 *bit_a, *bit_b, *bit_shift;
    const i64 *bit_mode;
    uint8_t *out;
    u64 hits;
} orc_job;

static void *orc_contains_job(void *p)
{
    orc_job *j = p;
    j->hits = orc_contains_blocks(j->words, j->keys, j->n, j->shard_a, j->shard_b,
                                  j->shard_mode, j->shard_shift, j->wps, j->block_a, j->c,
                                  j->block_b, j->block_mode, j->block_shift, j->bit_a,
                                  j->bit_b, j->bit_mode, j->bit_shift, j->k, j->strategy,
                                  j->wpb, j->out);
    return NULL;
}

static void *orc_insert_c1_job(void *p)
{
    orc_job *j = p;
    i64 *addrs = malloc(sizeof(i64) * (size_t)j->k);
    u64 *mask = malloc(sizeof(u64) * (size_t)j->wpb);
    for (u64 i = 0; i < j->n; ++i) {
        u64 x = j->keys[i];
        u64 base = orc_hval(j->shard_a, x, j->shard_b, j->shard_mode, j->shard_shift) * j->wps +
                   orc_hval(j->block_a[0], x, j->block_b, j->block_mode, j->block_shift) *
                       (u64)j->wpb;
        orc_fill_addrs(x, j->bit_a, j->bit_b, j->bit_mode, j->bit_shift, j->k, j->strategy,
                       addrs);
        memset(mask, 0, sizeof(u64) * (size_t)j->wpb);
        for (int t = 0; t < j->k; ++t)
            mask[addrs[t] >> 6] |= (u64)1 << (addrs[t] & 63);
        for (int w = 0; w < j->wpb; ++w)
            if (mask[w])
                __atomic_fetch_or(&j->wwords[base + (u64)w], mask[w], __ATOMIC_RELAXED);
    }
    free(addrs);
    free(mask);
    return NULL;
}

static u64 orc_run_jobs(int threads, u64 n, orc_job *proto, void *(*fn)(void *),
                        const u64 *keys, uint8_t *out)
{
    if (threads < 1)
        threads = 1;
    pthread_t *tid = malloc(sizeof(pthread_t) * (size_t)threads);
    orc_job *jobs = malloc(sizeof(orc_job) * (size_t)threads);
    u64 base = n / (u64)threads, extra = n % (u64)threads, start = 0;
    for (int t = 0; t < threads; ++t) {
        u64 len = base + ((u64)t < extra ? 1 : 0);
        jobs[t] = *proto;
        jobs[t].keys = keys + start;
        jobs[t].n = len;
        jobs[t].out = out ? out + start : NULL;
        start += len;
        pthread_create(&tid[t], NULL, fn, &jobs[t]);
    }
    u64 hits = 0;
    for (int t = 0; t < threads; ++t) {
        pthread_join(tid[t], NULL);
        hits += jobs[t].hits;
    }
    free(tid);
    free(jobs);
    return hits;
}

u64 orc_contains_blocks_mt(const u64 *words, const u64 *keys, u64 n,
                           u64 shard_a, u64 shard_b, i64 shard_mode, u64 shard_shift,
                           u64 wps, const u64 *block_a, int c, u64 block_b,
                           i64 block_mode, u64 block_shift, const u64 *bit_a,
                           const u64 *bit_b, const i64 *bit_mode, const u64 *bit_shift,
                           int k, int strategy, int wpb, uint8_t *out, int threads)
{
    orc_job p = {.words = words, .shard_a = shard_a, .shard_b = shard_b,
                 .shard_mode = shard_mode, .shard_shift = shard_shift, .wps = wps,
                 .block_a = block_a, .c = c, .block_b = block_b, .block_mode = block_mode,
                 .block_shift = block_shift, .bit_a = bit_a, .bit_b = bit_b,
                 .bit_mode = bit_mode, .bit_shift = bit_shift, .k = k,
                 .strategy = strategy, .wpb = wpb};
    return orc_run_jobs(threads, n, &p, orc_contains_job, keys, out);
}

void orc_insert_blocks_c1_mt(u64 *words, const u64 *keys, u64 n,
                             u64 shard_a, u64 shard_b, i64 shard_mode, u64 shard_shift,
                             u64 wps, const u64 *block_a, u64 block_b, i64 block_mode,
                             u64 block_shift, const u64 *bit_a, const u64 *bit_b,
                             const i64 *bit_mode, const u64 *bit_shift, int k,
                             int strategy, int wpb, int threads)
{
    orc_job p = {.wwords = words, .shard_a = shard_a, .shard_b = shard_b,
                 .shard_mode = shard_mode, .shard_shift = shard_shift, .wps = wps,
                 .block_a = block_a, .c = 1, .block_b = block_b, .block_mode = block_mode,
                 .block_shift = block_shift, .bit_a = bit_a, .bit_b = bit_b,
                 .bit_mode = bit_mode, .bit_shift = bit_shift, .k = k,
                 .strategy = strategy, .wpb = wpb};
    orc_run_jobs(threads, n, &p, orc_insert_c1_job, keys, NULL);
}
