// C ABI (include/bbchoc.h): filter handles, argument validation, dispatch to
// the kernels, host-buffer staging.  No exception crosses this boundary.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <condition_variable>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <unistd.h>

#include "../../include/bbchoc.h"
#include "launch.h"

using namespace bc;

namespace bc {
unsigned long long launch_count();
}

// ---------------------------------------------------------------------------------
static thread_local std::string g_err;

static int fail(int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

namespace bc {
// error entry for the other translation units (peer.cu)
int set_error(int code, const char *msg) {
    g_err = msg;
    return code;
}
}  // namespace bc

#define CUDA_TRY(expr)                                                                   \
    do {                                                                                 \
        cudaError_t e__ = (expr);                                                        \
        if (e__ != cudaSuccess)                                                          \
            return fail(e__ == cudaErrorMemoryAllocation ? BC_ENOMEM : BC_ECUDA,         \
                        "%s: %s (%s:%d)", #expr, cudaGetErrorString(e__), __FILE__,      \
                        __LINE__);                                                       \
    } while (0)

static DevHash make_dev_hash(u64 a, u64 b) {
    DevHash h;
    h.a = a;
    h.b = b;
    h.magic = 0;
    h.shift = 0;
    if (b == 1) {
        h.mode = ZERO;  // MOD_ODD with b = 1: always 0
    } else if (b & 1) {
        h.mode = MOD_ODD;
    } else if ((b & (b - 1)) == 0) {
        h.mode = SHIFT_POW2;
        h.shift = 64 - (63 - __builtin_clzll(b));  // hashing.py:73-74
    } else {
        h.mode = XOR_EVEN;
        h.shift = 32;  // u // 2, hashing.py:76
    }
    if (h.mode == MOD_ODD || h.mode == XOR_EVEN)
        h.magic = (u64)(((unsigned __int128)1 << 64) / b);
    return h;
}

// Reference cost formulas, evaluated in the same operation order as
// _kernels.py:100-109 (IEEE double, no contraction: see the build flags).
static double ref_cost(int code, double param, int j, int a, int k, int block_bits) {
    const double jf = (double)j, af = (double)a, kf = (double)k;
    const double quarter = block_bits / 4.0, half = block_bits / 2.0;
    if (code == 0) return std::pow(param, jf / quarter) + af / kf;
    if (code == 1) return param * kf * std::pow(jf / half, kf) + af;
    return kf * std::pow((jf + param * kf) / half, kf) + af;
}

struct bc_filter {
    int device = 0;
    int kind = 0;
    KParams kp{};
    DevHash *d_bits = nullptr;
    u32 *d_rank = nullptr;
    std::mutex mu;  // ordered-insert scratch
    u64 *d_owner = nullptr;
    u32 *d_lists = nullptr;
    u64 *d_lkeys = nullptr;
    u32 *d_state = nullptr;
    // completion of the last ordered launch: the scratch is per handle, so a
    // launch on another stream waits for it (one writer at a time)
    cudaEvent_t ord_done = nullptr;
    u64 chunk = 0;
    u64 slots = 0;        // claim slots per owner array
    u64 owner_words = 0;  // allocated u64 claim tags
    u64 rounds_bound = 0;
};

// ---------------------------------------------------------------------------------
extern "C" const char *bc_last_error(void) { return g_err.c_str(); }

extern "C" unsigned long long bc_launch_count(void) { return bc::launch_count(); }

extern "C" const char *bc_version(void) { return "bbchoc-b200 0.1.0 (sm_100a)"; }

extern "C" void bc_l2_release(void) { bc::l2_release_all(); }

extern "C" int bc_filter_create(const bc_filter_desc *d, bc_filter **out) {
    if (!d || !out) return fail(BC_EINVAL, "null argument");
    *out = nullptr;
    const int B = d->block_bits;
    const bool toy = (B == 8 || B == 16 || B == 32);
    if (!(toy || (B > 0 && B % 64 == 0))) return fail(BC_EINVAL, "invalid block_bits %d", B);
    if (d->kind < 0 || d->kind > 2) return fail(BC_EINVAL, "unknown kind %d", d->kind);
    if (d->k < 1 || d->k > B) return fail(BC_EINVAL, "k must be in [1, %d], got %d", B, d->k);
    if (d->strategy != 0 && d->strategy != 1)
        return fail(BC_EINVAL, "unknown strategy %d", d->strategy);
    if (d->num_blocks < 1 || d->shards < 1 || d->num_blocks % d->shards != 0)
        return fail(BC_EINVAL, "%llu blocks do not split into %llu shards",
                    (unsigned long long)d->num_blocks, (unsigned long long)d->shards);
    if (!d->bit_a || !d->bit_b) return fail(BC_EINVAL, "bit_a / bit_b must be given");
    const int c = d->choices;
    if (d->kind == BC_KIND_STANDARD) {
        if (c != 0) return fail(BC_EINVAL, "standard filters have 0 choices");
        if (d->strategy != 0 || d->shards != 1 || toy)
            return fail(BC_EINVAL, "standard filters are random, unsharded, word-multiple");
    } else if (d->kind == BC_KIND_BLOCKED) {
        if (c != 1) return fail(BC_EINVAL, "blocked filters have exactly one choice");
    } else if (c < 2 || c > BC_MAX_CHOICES) {
        return fail(BC_EINVAL, "blowchoc needs between 2 and %d choices, got %d",
                    BC_MAX_CHOICES, c);
    }
    const int wpb = B >= 64 ? B / 64 : 1;
    if (d->kind != BC_KIND_STANDARD && wpb > kMaxWpb)
        return fail(BC_EUNSUP, "block_bits %d above the supported %d", B, kMaxWpb * 64);
    if (d->kind != BC_KIND_STANDARD && d->num_blocks >= (1ull << 32))
        return fail(BC_EUNSUP, "more than 2^32 blocks");
    // bit ranges are implied by the layout (BitSelector, hashing.py:118-162):
    // random -> B for every function, distinct -> B - i, standard -> m = M*B.
    // Anything else would address bits outside a block.
    for (int i = 0; i < d->k; ++i) {
        const u64 want = d->kind == BC_KIND_STANDARD ? d->num_blocks * (u64)B
                         : d->strategy == 0          ? (u64)B
                                                     : (u64)(B - i);
        if (d->bit_b[i] != want)
            return fail(BC_EINVAL, "bit range %d is %llu, expected %llu", i,
                        (unsigned long long)d->bit_b[i], (unsigned long long)want);
    }

    bc_filter *f = new (std::nothrow) bc_filter();
    if (!f) return fail(BC_ENOMEM, "out of host memory");
    cudaGetDevice(&f->device);
    f->kind = d->kind;
    KParams &p = f->kp;
    p.k = (u32)d->k;
    p.c = (u32)(d->kind == BC_KIND_STANDARD ? 0 : c);
    p.wpb = (u32)wpb;
    p.strategy = (u32)d->strategy;
    p.block_bits = (u32)B;
    p.num_blocks = d->num_blocks;
    p.per_shard = d->num_blocks / d->shards;
    p.shard = make_dev_hash(d->shard_a, d->shards);
    p.block = make_dev_hash(0, p.per_shard);
    for (int ci = 0; ci < BC_MAX_CHOICES; ++ci) p.block_a[ci] = ci < c ? d->block_a[ci] : 0;
    if (d->kind == BC_KIND_STANDARD) {
        const u64 m = d->num_blocks * (u64)B;
        DevHash fh = make_dev_hash(0, m);
        p.flat_b = m;
        p.flat_magic = fh.magic;
        p.flat_mode = fh.mode;
        p.flat_shift = fh.shift;
    }
    std::vector<DevHash> bits(d->k);
    bool fast = d->kind != BC_KIND_STANDARD && d->strategy == 0 && B == 512 && d->k <= kMaxFastK;
    for (int i = 0; i < d->k; ++i) {
        bits[i] = make_dev_hash(d->bit_a[i], d->bit_b[i]);
        if (d->bit_b[i] != 512) fast = false;
        if (i < kMaxFastK) {
            p.bit_a_lo[i] = (u32)d->bit_a[i];
            p.bit_a_hi[i] = (u32)(d->bit_a[i] >> 32);
        }
    }
    p.fast_random = fast ? 1u : 0u;

    auto cleanup = [&](int rc) {
        bc_filter_destroy(f);
        return rc;
    };
    cudaError_t e = cudaMalloc(&f->d_bits, sizeof(DevHash) * bits.size());
    if (e != cudaSuccess) return cleanup(fail(BC_ENOMEM, "cudaMalloc: %s", cudaGetErrorString(e)));
    e = cudaMemcpy(f->d_bits, bits.data(), sizeof(DevHash) * bits.size(), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return cleanup(fail(BC_ECUDA, "cudaMemcpy: %s", cudaGetErrorString(e)));
    p.bits = f->d_bits;

    if (c >= 2) {
        // Dense ranks of the float64 costs: cost_i < cost_j  <=>  rank_i < rank_j,
        // equal costs share a rank; +inf and NaN never beat the initial +inf
        // (_kernels.py:156-170), so they get the sentinel rank.
        const int K1 = d->k + 1;
        const size_t cells = (size_t)(B + 1) * K1;
        std::vector<double> cost(cells);
        for (int j = 0; j <= B; ++j)
            for (int a = 0; a <= d->k; ++a)
                cost[(size_t)j * K1 + a] = d->cost_table
                                               ? d->cost_table[(size_t)j * K1 + a]
                                               : ref_cost(d->cost_code, d->cost_param, j, a,
                                                          d->k, B);
        std::vector<double> uniq;
        uniq.reserve(cells);
        for (double v : cost)
            if (!std::isnan(v) && !(std::isinf(v) && v > 0)) uniq.push_back(v);
        std::sort(uniq.begin(), uniq.end());
        uniq.erase(std::unique(uniq.begin(), uniq.end()), uniq.end());
        std::vector<u32> rank(cells);
        for (size_t i = 0; i < cells; ++i) {
            const double v = cost[i];
            if (std::isnan(v) || (std::isinf(v) && v > 0))
                rank[i] = 0xffffffffu;
            else
                rank[i] = (u32)(std::lower_bound(uniq.begin(), uniq.end(), v) - uniq.begin());
        }
        e = cudaMalloc(&f->d_rank, sizeof(u32) * cells);
        if (e != cudaSuccess)
            return cleanup(fail(BC_ENOMEM, "cudaMalloc: %s", cudaGetErrorString(e)));
        e = cudaMemcpy(f->d_rank, rank.data(), sizeof(u32) * cells, cudaMemcpyHostToDevice);
        if (e != cudaSuccess)
            return cleanup(fail(BC_ECUDA, "cudaMemcpy: %s", cudaGetErrorString(e)));
    }
    p.rank = f->d_rank;
    *out = f;
    return BC_OK;
}

extern "C" void bc_filter_destroy(bc_filter *f) {
    if (!f) return;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(f->device);
    cudaFree(f->d_bits);
    cudaFree(f->d_rank);
    cudaFree(f->d_owner);
    cudaFree(f->d_lists);
    cudaFree(f->d_lkeys);
    cudaFree(f->d_state);
    if (f->ord_done) cudaEventDestroy(f->ord_done);
    bc::l2_release();
    cudaSetDevice(prev);
    delete f;
}

// The library's stream-ordered scratch (cudaMallocAsync: q-gram tile offsets,
// hit counters, ticket arrays) comes from the device's default pool, whose
// release threshold is 0: every synchronisation would hand the memory back
// to the driver and the next call would map it again (~ms for tens of MB).
// Keep up to 1 GiB of it reserved instead.
static void keep_pool(int dev) {
    static std::once_flag once[64];
    if (dev < 0 || dev >= 64) return;
    std::call_once(once[dev], [dev] {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            u64 keep = 1ull << 30;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
        cudaGetLastError();
    });
}

static int check_device(bc_filter *f) {
    int dev = -1;
    cudaGetDevice(&dev);
    if (dev != f->device)
        return fail(BC_EINVAL, "filter handle belongs to device %d, current device is %d",
                    f->device, dev);
    keep_pool(dev);
    return BC_OK;
}

// Ordered-insert scratch: the claim arrays, two pending lists of `chunk`
// entries (u32 stream index + u64 key), state = {round, counter0..2}.  All
// of it is allocated into locals and published only once every allocation
// and initialisation succeeded, so a failed attempt leaves the handle
// without scratch (the next insert retries) instead of half-initialised.
static int ensure_ordered_scratch(bc_filter *f, cudaStream_t s) {
    if (f->d_owner) return BC_OK;
    const u64 M = f->kp.num_blocks;
    // Window (pending keys per round) trades rounds (grid syncs) against
    // conflicts (claims per committed key).  Measured on B200 with the
    // sliding-window kernel (bench.py --insert-mode ordered): cfg1 (M = 2^15)
    // is best at M/2 (550 Mkeys/s vs 515 at 2M, 440 at M/4); cfg3 (M = 2^23)
    // at 2^19 (1765 vs 1602 at 2^20, 442 at 2^22); cfg5 (M = 2^27) 1781 at
    // 2^18, 1896 at 2^20.
    // One-array rounds (ordered1_kernel, tools/r2_one_sweep.sh): cfg3 (c = 3)
    // 7 262 / 7 307 / 6 408 Mkeys/s at 3*2^17 / 2^19 / 3*2^18; cfg5 (c = 2)
    // 8 551 / 8 875 / 9 111.
    // Below 2^23 blocks the one-array rounds want a window of about
    // M / (2 c^2): a key loses a round when an earlier key of the window
    // shares one of its c slots, and with M/2 keys in the window most do
    // (tools/r2_window_sweep.sh, Mkeys/s at M/2, M/4, M/8, M/16: 2^20 blocks
    // c = 2: 3 970 / 6 074 / 7 004 / 5 743; c = 3: 1 576 / 2 250 / 2 798 /
    // 4 246; 2^22 blocks c = 2: 9 584 at M/8, c = 3: 6 454 at M/16).
    const u64 cc = (u64)f->kp.c * f->kp.c;
    u64 chunk = ordered_one()
                    ? std::min<u64>(std::max<u64>(M / (2 * cc), 4096),
                                    f->kp.c == 2 ? 3ull << 18 : 1ull << 19)
                    : std::min<u64>(M / 2, 1ull << 19);
    chunk = std::min<u64>(chunk, std::max<u64>(M / 2, 256));
    if (const char *e = std::getenv("BC_ORDERED_CHUNK")) chunk = std::strtoull(e, nullptr, 10);
    chunk = std::max<u64>(chunk, 256);
    chunk = std::min<u64>(chunk, 1ull << 24);
    // Claim slots: one per block up to 2^23 blocks, else 2^23 slots with the
    // blocks hashed onto them (spurious conflicts only delay commits).  The
    // claims (one u32 array of 32 MiB for ordered1_kernel) sit under a
    // persisting L2 window sized to them.  Fewer slots mean more spurious
    // conflicts, more take the L2 from the candidate blocks
    // (tools/r2_one_sweep.sh, Mkeys/s at 2^22 / 2^23 / 2^24 slots: cfg5
    // 8 810 / 8 875 / 7 909, cfg4's geometry 8 821 / 9 075 / 7 892; a 2 GiB
    // c = 3 filter 6 901 at 2^23, 6 769 at 2^24).  The two-array rounds
    // (BC_ORDERED_ONE=0, 8 bytes per slot) are best at 2^22 slots for c = 2
    // (cfg5 7 661 vs 7 117 at 2^23) and 2^23 for c >= 3 (cfg3 6 140 vs
    // 5 267).  BC_ORDERED_SLOTS overrides (0 = one per block).
    u64 slots = M;
    u64 want = (!ordered_one() && f->kp.c == 2) ? 1ull << 22 : 1ull << 23;
    if (const char *e = std::getenv("BC_ORDERED_SLOTS")) want = std::strtoull(e, nullptr, 10);
    if (want) {
        u64 pow2 = 1;
        while (pow2 < want) pow2 <<= 1;
        if (pow2 < M) slots = pow2;
    }
    // two arrays of u32 claims: the sliding-window kernel claims for round
    // r + 1 while round r's claims are being checked (the fixed-chunk kernel,
    // BC_ORDERED_WINDOW=0, uses one array of M u64 round-tagged claims)
    const u64 owner_words = ordered_owner_words(M, slots);
    u64 *owner = nullptr, *lkeys = nullptr;
    u32 *lists = nullptr, *state = nullptr;
    cudaEvent_t done = nullptr;
    cudaError_t e = cudaMalloc(&owner, sizeof(u64) * owner_words);
    if (e == cudaSuccess) e = cudaMalloc(&lists, sizeof(u32) * 2 * chunk);
    if (e == cudaSuccess) e = cudaMalloc(&lkeys, sizeof(u64) * 2 * chunk);
    if (e == cudaSuccess) e = cudaMalloc(&state, sizeof(u32) * 16);
    if (e == cudaSuccess) e = cudaMemsetAsync(owner, 0xff, sizeof(u64) * owner_words, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(state, 0, sizeof(u32) * 16, s);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&done, cudaEventDisableTiming);
    if (e != cudaSuccess) {
        cudaFree(owner);
        cudaFree(lists);
        cudaFree(lkeys);
        cudaFree(state);
        if (done) cudaEventDestroy(done);
        return fail(e == cudaErrorMemoryAllocation ? BC_ENOMEM : BC_ECUDA,
                    "ordered-insert scratch: %s", cudaGetErrorString(e));
    }
    f->d_lists = lists;
    f->d_lkeys = lkeys;
    f->d_state = state;
    f->ord_done = done;
    f->chunk = chunk;
    f->slots = slots;
    f->owner_words = owner_words;
    f->rounds_bound = 0;
    f->d_owner = owner;  // published last: the "scratch ready" flag
    return BC_OK;
}

// Ordered launches on a handle run one at a time even from several streams:
// the caller's stream first waits for the previous launch (its scratch), and
// the launch is recorded as the new previous one.  Call with f->mu held.
static int ordered_begin(bc_filter *f, cudaStream_t s) {
    CUDA_TRY(cudaStreamWaitEvent(s, f->ord_done, 0));
    return BC_OK;
}

static int ordered_end(bc_filter *f, cudaStream_t s) {
    CUDA_TRY(cudaEventRecord(f->ord_done, s));
    return BC_OK;
}

// Every round commits at least one key, so rounds <= keys: re-arm the round
// tags long before the 32-bit counter could wrap.
static int ordered_rearm(bc_filter *f, u64 n, cudaStream_t s) {
    if (f->rounds_bound + n >= (1ull << 31)) {
        CUDA_TRY(cudaMemsetAsync(f->d_owner, 0xff, sizeof(u64) * f->owner_words, s));
        CUDA_TRY(cudaMemsetAsync(f->d_state, 0, sizeof(u32) * 8, s));
        f->rounds_bound = 0;
    }
    return BC_OK;
}

// Region-partitioned single-choice inserts (partition_insert.cu) are opt-in:
// on B200 the bucket scatter currently costs more than it saves (cfg2: 2.2 ms
// vs 1.75 ms direct).  BC_PARTITION_MIN_KEYS=<n> enables them
// for batches of at least n keys.
static const u64 kPartitionMinKeys = []() -> u64 {
    const char *e = std::getenv("BC_PARTITION_MIN_KEYS");
    return e ? std::strtoull(e, nullptr, 10) : ~0ull;
}();

static int insert_device(bc_filter *f, u64 *words, const u64 *keys, u64 n, int mode,
                         cudaStream_t s) {
    if (n == 0) return BC_OK;
    if (f->kind == BC_KIND_STANDARD) {
        CUDA_TRY(launch_flat(OP_INSERT, f->kp, words, keys, n, nullptr, nullptr, s));
        return BC_OK;
    }
    if (f->kp.c == 1) {  // OR commutes: any order is the reference's order
        if (partition_supported(f->kp) && n >= kPartitionMinKeys) {
            // region-partitioned: bucket by 64 KiB filter region, OR in shared memory
            const u64 per = std::min<u64>(n, 1ull << 27);
            void *scratch = nullptr;
            CUDA_TRY(cudaMallocAsync(&scratch, partition_scratch_bytes(f->kp, per), s));
            cudaError_t e = cudaSuccess;
            for (u64 off = 0; off < n && e == cudaSuccess; off += per)
                e = launch_partitioned_insert(f->kp, words, keys + off, std::min(per, n - off),
                                              scratch, s);
            cudaFreeAsync(scratch, s);
            CUDA_TRY(e);
            return BC_OK;
        }
        CUDA_TRY(launch_blocks(OP_INSERT, f->kp, words, keys, n, nullptr, nullptr, s));
        return BC_OK;
    }
    if (mode == BC_INSERT_RELAXED) {
        // keep at most M/2 keys in flight (FPR within ~3%): one
        // persistent launch whose grid holds <= M/2 keys (256 per CTA) at a time,
        // or, for filters under 512 blocks, launches of M/2 keys each
        // BC_RELAXED_INFLIGHT_PCT (experiments only): keys in flight as a
        // percentage of M instead of the 50% the tolerance is stated for
        static const u64 pct = [] {
            const char *e = std::getenv("BC_RELAXED_INFLIGHT_PCT");
            return e ? std::max<u64>(1, std::strtoull(e, nullptr, 10)) : 50ull;
        }();
        const u64 per = std::max<u64>(1, f->kp.num_blocks * pct / 100);
        if (per >= 256) {
            KParams kp = f->kp;
            kp.max_ctas = (u32)std::min<u64>(per / 256, 0xffffffffu);
            CUDA_TRY(launch_blocks(OP_INSERT, kp, words, keys, n, nullptr, nullptr, s));
            return BC_OK;
        }
        for (u64 off = 0; off < n; off += per)
            CUDA_TRY(launch_blocks(OP_INSERT, f->kp, words, keys + off, std::min(per, n - off),
                                   nullptr, nullptr, s));
        return BC_OK;
    }
    std::lock_guard<std::mutex> lk(f->mu);
    int rc = ensure_ordered_scratch(f, s);
    if (rc == BC_OK) rc = ordered_begin(f, s);
    if (rc) return rc;
    if (ordered_ticket_supported(f->kp)) {
        // small filters: a dataflow over per-block tickets (ordered_ticket.cu)
        cudaError_t e = launch_ordered_ticket(f->kp, words, keys, n, s);
        if (e != cudaSuccess) rc = fail(BC_ECUDA, "ordered ticket insert: %s", cudaGetErrorString(e));
        const int rc2 = ordered_end(f, s);
        return rc ? rc : rc2;
    }
    for (u64 off = 0; off < n && rc == BC_OK; off += (1ull << 30)) {
        const u64 len = std::min<u64>(1ull << 30, n - off);
        rc = ordered_rearm(f, len, s);
        if (rc) break;
        cudaError_t e = launch_ordered(f->kp, words, keys + off, len, f->chunk, f->d_owner,
                                       f->slots, f->d_lists, f->d_lkeys, f->d_state, s);
        if (e != cudaSuccess)
            rc = fail(BC_ECUDA, "ordered insert: %s", cudaGetErrorString(e));
        f->rounds_bound += len;
    }
    const int rc2 = ordered_end(f, s);
    return rc ? rc : rc2;
}

extern "C" int bc_insert(bc_filter *f, uint64_t *d_words, const uint64_t *d_keys, uint64_t n,
                         int mode, void *stream) {
    if (!f) return fail(BC_EINVAL, "null filter");
    if (n && (!d_words || !d_keys)) return fail(BC_EINVAL, "null words or keys");
    if (mode != BC_INSERT_ORDERED && mode != BC_INSERT_RELAXED)
        return fail(BC_EINVAL, "unknown insert mode %d", mode);
    if (int rc = check_device(f)) return rc;
    return insert_device(f, d_words, d_keys, n, mode, (cudaStream_t)stream);
}

static int contains_device(bc_filter *f, const u64 *words, const u64 *keys, u64 n, u8 *out,
                           unsigned long long *hits, cudaStream_t s) {
    if (n == 0) return BC_OK;
    if (f->kind == BC_KIND_STANDARD)
        CUDA_TRY(launch_flat(OP_CONTAINS, f->kp, const_cast<u64 *>(words), keys, n, out, hits, s));
    else
        CUDA_TRY(launch_blocks(OP_CONTAINS, f->kp, const_cast<u64 *>(words), keys, n, out, hits,
                               s));
    return BC_OK;
}

extern "C" int bc_contains(bc_filter *f, const uint64_t *d_words, const uint64_t *d_keys,
                           uint64_t n, uint8_t *d_out, unsigned long long *d_hits, void *stream) {
    if (!f) return fail(BC_EINVAL, "null filter");
    if (n && (!d_words || !d_keys)) return fail(BC_EINVAL, "null words or keys");
    if (int rc = check_device(f)) return rc;
    return contains_device(f, d_words, d_keys, n, d_out, d_hits, (cudaStream_t)stream);
}

// ---- q-grams ------------------------------------------------------------------------
static u64 qgram_windows(u64 len, int q) { return len >= (u64)q ? len - (u64)q + 1 : 0; }

extern "C" int bc_encode_qgrams(const uint8_t *d_seq, uint64_t len, int q, int canonical,
                                uint64_t record_len, uint64_t *d_keys,
                                unsigned long long *d_count, void *stream) {
    if (q < 1 || q > 32) return fail(BC_EINVAL, "q must be in [1, 32], got %d", q);
    cudaStream_t s = (cudaStream_t)stream;
    const u64 nwin = qgram_windows(len, q);
    if (nwin == 0) {
        if (d_count) CUDA_TRY(cudaMemsetAsync(d_count, 0, sizeof(*d_count), s));
        return BC_OK;
    }
    if (!d_seq || !d_keys) return fail(BC_EINVAL, "null sequence or key buffer");
    const u64 ntiles = (nwin + kQgramTile - 1) / kQgramTile;
    u64 *tiles = nullptr;
    CUDA_TRY(cudaMallocAsync((void **)&tiles, sizeof(u64) * ntiles, s));
    const RecSpec rec{record_len, 0};
    cudaError_t e = launch_qgram_offsets(d_seq, len, q, rec, tiles, ntiles, d_count, s);
    if (e == cudaSuccess) e = launch_qgram_encode(d_seq, len, q, canonical, rec, tiles, d_keys, s);
    cudaFreeAsync(tiles, s);
    CUDA_TRY(e);
    return BC_OK;
}

// Materialise the keys of a window slice (for the geometries no fused kernel
// covers: non-512-bit blocks, the distinct strategy with c >= 2, standard
// filters).  The caller walks the sequence in slices of kEncodeSlice windows
// (consecutive inserts equal one insert; lookups write at the running answer
// offset), so at most kEncodeSlice keys are ever materialised.
static constexpr u64 kEncodeSlice = 1ull << 26;

static int encode_tmp(const u8 *seq, u64 len, int q, int canonical, RecSpec rec, u64 **keys,
                      u64 *n, cudaStream_t s) {
    const u64 nwin = qgram_windows(len, q);
    *keys = nullptr;
    *n = 0;
    if (nwin == 0) return BC_OK;
    unsigned long long *d_cnt = nullptr;
    u64 *tiles = nullptr;
    const u64 ntiles = (nwin + kQgramTile - 1) / kQgramTile;
    CUDA_TRY(cudaMallocAsync((void **)keys, sizeof(u64) * nwin, s));
    cudaError_t e = cudaMallocAsync((void **)&d_cnt, sizeof(*d_cnt), s);
    if (e == cudaSuccess) e = cudaMallocAsync((void **)&tiles, sizeof(u64) * ntiles, s);
    if (e == cudaSuccess) e = launch_qgram_offsets(seq, len, q, rec, tiles, ntiles, d_cnt, s);
    if (e == cudaSuccess) e = launch_qgram_encode(seq, len, q, canonical, rec, tiles, *keys, s);
    unsigned long long h_cnt = 0;
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(&h_cnt, d_cnt, sizeof h_cnt, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (tiles) cudaFreeAsync(tiles, s);
    if (d_cnt) cudaFreeAsync(d_cnt, s);
    if (e != cudaSuccess) {
        cudaFreeAsync(*keys, s);
        *keys = nullptr;
        return fail(BC_ECUDA, "q-gram encode: %s", cudaGetErrorString(e));
    }
    *n = h_cnt;
    return BC_OK;
}

// Record spec of the slice starting at window w of a sequence.
static RecSpec slice_rec(u64 record_len, u64 w) {
    return RecSpec{record_len, record_len ? w % record_len : 0};
}

static int add_count(unsigned long long *d_count, u64 n, cudaStream_t s) {
    if (!d_count || n == 0) return BC_OK;
    // d_count was zeroed on the stream; add the host-known total
    unsigned long long hn = 0;
    CUDA_TRY(cudaMemcpyAsync(&hn, d_count, sizeof hn, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    hn += n;
    CUDA_TRY(cudaMemcpyAsync(d_count, &hn, sizeof hn, cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    return BC_OK;
}

extern "C" int bc_insert_qgrams(bc_filter *f, uint64_t *d_words, const uint8_t *d_seq,
                                uint64_t len, int q, int canonical, uint64_t record_len,
                                int mode, unsigned long long *d_count, void *stream) {
    if (!f) return fail(BC_EINVAL, "null filter");
    if (q < 1 || q > 32) return fail(BC_EINVAL, "q must be in [1, 32], got %d", q);
    if (mode != BC_INSERT_ORDERED && mode != BC_INSERT_RELAXED)
        return fail(BC_EINVAL, "unknown insert mode %d", mode);
    if (int rc = check_device(f)) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    const u64 nwin = qgram_windows(len, q);
    if (d_count) CUDA_TRY(cudaMemsetAsync(d_count, 0, sizeof(*d_count), s));
    if (nwin == 0) return BC_OK;
    if (!d_words || !d_seq) return fail(BC_EINVAL, "null words or sequence");
    const bool blocks512 = f->kind != BC_KIND_STANDARD && f->kp.wpb == 8;
    if (blocks512 && (f->kp.c == 1 || mode == BC_INSERT_RELAXED)) {
        // c == 1: one launch (OR commutes).  relaxed: windows in slices of M/2.
        const u64 per = f->kp.c == 1 ? nwin : std::max<u64>(1, f->kp.num_blocks / 2);
        for (u64 w = 0; w < nwin; w += per) {
            const u64 nw = std::min(per, nwin - w);
            CUDA_TRY(launch_qgram_blocks(OP_INSERT, f->kp, d_words, d_seq + w, nw + q - 1, q,
                                         canonical, slice_rec(record_len, w), nullptr, nullptr,
                                         nullptr, d_count, s));
        }
        return BC_OK;
    }
    if (blocks512 && ordered_tiles_supported(f->kp)) {
        // exact stream order, keys encoded on the fly from the sequence
        // (window index = priority): no key array
        std::lock_guard<std::mutex> lk(f->mu);
        int rc = ensure_ordered_scratch(f, s);
        if (rc == BC_OK) rc = ordered_begin(f, s);
        if (rc) return rc;
        if (ordered_ticket_supported(f->kp)) {
            cudaError_t e = launch_ordered_ticket_qgrams(f->kp, d_words, d_seq, nwin, q, canonical,
                                                         slice_rec(record_len, 0), d_count, s);
            if (e != cudaSuccess)
                rc = fail(BC_ECUDA, "ordered ticket q-gram insert: %s", cudaGetErrorString(e));
            const int rc2 = ordered_end(f, s);
            return rc ? rc : rc2;
        }
        for (u64 w = 0; w < nwin && rc == BC_OK; w += (1ull << 30)) {
            const u64 nw = std::min<u64>(1ull << 30, nwin - w);
            rc = ordered_rearm(f, nw, s);
            if (rc) break;
            cudaError_t e = launch_ordered_qgrams(f->kp, d_words, d_seq + w, nw, q, canonical,
                                                  slice_rec(record_len, w), f->chunk, f->d_owner,
                                                  f->slots, f->d_lists, f->d_lkeys, f->d_state,
                                                  d_count, s);
            if (e != cudaSuccess)
                rc = fail(BC_ECUDA, "ordered q-gram insert: %s", cudaGetErrorString(e));
            f->rounds_bound += nw;
        }
        const int rc2 = ordered_end(f, s);
        return rc ? rc : rc2;
    }
    // other geometries: bounded slices of materialised keys
    u64 total = 0;
    for (u64 w = 0; w < nwin; w += kEncodeSlice) {
        const u64 nw = std::min(kEncodeSlice, nwin - w);
        u64 *keys = nullptr, n = 0;
        int rc = encode_tmp(d_seq + w, nw + q - 1, q, canonical, slice_rec(record_len, w), &keys,
                            &n, s);
        if (rc == BC_OK) rc = insert_device(f, d_words, keys, n, mode, s);
        if (keys) cudaFreeAsync(keys, s);
        if (rc) return rc;
        total += n;
    }
    return add_count(d_count, total, s);
}

extern "C" int bc_contains_qgrams(bc_filter *f, const uint64_t *d_words, const uint8_t *d_seq,
                                  uint64_t len, int q, int canonical, uint64_t record_len,
                                  uint8_t *d_out, unsigned long long *d_count,
                                  unsigned long long *d_hits, void *stream) {
    if (!f) return fail(BC_EINVAL, "null filter");
    if (q < 1 || q > 32) return fail(BC_EINVAL, "q must be in [1, 32], got %d", q);
    if (int rc = check_device(f)) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    const u64 nwin = qgram_windows(len, q);
    if (nwin == 0) {
        if (d_count) CUDA_TRY(cudaMemsetAsync(d_count, 0, sizeof(*d_count), s));
        return BC_OK;
    }
    if (!d_words || !d_seq) return fail(BC_EINVAL, "null words or sequence");
    if (f->kind != BC_KIND_STANDARD && f->kp.wpb == 8) {
        const u64 ntiles = (nwin + kQgramTile - 1) / kQgramTile;
        u64 *tiles = nullptr;
        const bool need_off = d_out != nullptr || d_count != nullptr;
        if (need_off) {
            CUDA_TRY(cudaMallocAsync((void **)&tiles, sizeof(u64) * ntiles, s));
            cudaError_t e = launch_qgram_offsets(d_seq, len, q, RecSpec{record_len, 0}, tiles,
                                                 ntiles, d_count, s);
            if (e != cudaSuccess) {
                cudaFreeAsync(tiles, s);
                CUDA_TRY(e);
            }
        }
        cudaError_t e = launch_qgram_blocks(OP_CONTAINS, f->kp, const_cast<u64 *>(d_words), d_seq,
                                            len, q, canonical, RecSpec{record_len, 0}, tiles,
                                            d_out, d_hits, nullptr, s);
        if (tiles) cudaFreeAsync(tiles, s);
        CUDA_TRY(e);
        return BC_OK;
    }
    if (d_count) CUDA_TRY(cudaMemsetAsync(d_count, 0, sizeof(*d_count), s));
    u64 total = 0;
    for (u64 w = 0; w < nwin; w += kEncodeSlice) {
        const u64 nw = std::min(kEncodeSlice, nwin - w);
        u64 *keys = nullptr, n = 0;
        int rc = encode_tmp(d_seq + w, nw + q - 1, q, canonical, slice_rec(record_len, w), &keys,
                            &n, s);
        if (rc == BC_OK)
            rc = contains_device(f, d_words, keys, n, d_out ? d_out + total : nullptr, d_hits, s);
        if (keys) cudaFreeAsync(keys, s);
        if (rc) return rc;
        total += n;
    }
    return add_count(d_count, total, s);
}

// ---- analysis / routing ---------------------------------------------------------------
extern "C" int bc_block_histogram(const uint64_t *d_words, uint64_t num_blocks, int block_bits,
                                  unsigned long long *d_counts, void *stream) {
    const bool toy = (block_bits == 8 || block_bits == 16 || block_bits == 32);
    if (!(toy || (block_bits > 0 && block_bits % 64 == 0)))
        return fail(BC_EINVAL, "invalid block_bits %d", block_bits);
    if (num_blocks && (!d_words || !d_counts)) return fail(BC_EINVAL, "null words or counts");
    CUDA_TRY(launch_histogram(d_words, num_blocks, block_bits, d_counts, (cudaStream_t)stream));
    return BC_OK;
}

extern "C" int bc_route(bc_filter *f, const uint64_t *d_keys, uint64_t n, uint64_t *d_shard,
                        void *stream) {
    if (!f) return fail(BC_EINVAL, "null filter");
    if (n && (!d_keys || !d_shard)) return fail(BC_EINVAL, "null keys or output");
    if (int rc = check_device(f)) return rc;
    CUDA_TRY(launch_eval_hash(f->kp.shard, d_keys, n, d_shard, (cudaStream_t)stream));
    return BC_OK;
}

extern "C" int bc_eval_hash(uint64_t a, uint64_t b, const uint64_t *d_keys, uint64_t n,
                            uint64_t *d_out, void *stream) {
    if (b < 1) return fail(BC_EINVAL, "hash range must be >= 1, got %llu", (unsigned long long)b);
    if (n && (!d_keys || !d_out)) return fail(BC_EINVAL, "null keys or output");
    CUDA_TRY(launch_eval_hash(make_dev_hash(a, b), d_keys, n, d_out, (cudaStream_t)stream));
    return BC_OK;
}

extern "C" int bc_pcg64_fill(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
                             uint64_t inc_lo, uint64_t offset, uint64_t n, uint64_t and_mask,
                             uint64_t or_mask, uint64_t *d_out, void *stream) {
    if (n && !d_out) return fail(BC_EINVAL, "null output");
    if (!(inc_lo & 1)) return fail(BC_EINVAL, "PCG64 increment must be odd");
    CUDA_TRY(launch_pcg64_fill(state_hi, state_lo, inc_hi, inc_lo, offset, n, and_mask, or_mask,
                               d_out, (cudaStream_t)stream));
    return BC_OK;
}

// ---- CLI query output -----------------------------------------------------------------
namespace {
// Threads for the host-side text work (query TSV formatting, key parsing):
// BC_PARSE_THREADS, default min(16, cores); 1 = serial.
unsigned host_text_threads() {
    static const unsigned t = [] {
        if (const char *e = std::getenv("BC_PARSE_THREADS")) return (unsigned)std::max(1, std::atoi(e));
        return std::min(16u, std::max(1u, std::thread::hardware_concurrency()));
    }();
    return t;
}

const struct DigitPairs {
    char d[200];
    DigitPairs() {
        for (int i = 0; i < 100; ++i) {
            d[2 * i] = (char)('0' + i / 10);
            d[2 * i + 1] = (char)('0' + i % 10);
        }
    }
} g_pairs;

// "<key>\t<0|1>\n" for keys [i0, i1) at o; returns the end.
char *format_range(const uint64_t *keys, const uint8_t *ans, uint64_t i0, uint64_t i1, char *o) {
    for (uint64_t i = i0; i < i1; ++i) {
        uint64_t v = keys[i];
        char buf[20];
        int p = 20;
        while (v >= 100) {
            const unsigned r = (unsigned)(v % 100);
            v /= 100;
            p -= 2;
            std::memcpy(buf + p, g_pairs.d + 2 * r, 2);
        }
        if (v >= 10) {
            p -= 2;
            std::memcpy(buf + p, g_pairs.d + 2 * v, 2);
        } else {
            buf[--p] = (char)('0' + v);
        }
        std::memcpy(o, buf + p, 20 - p);
        o += 20 - p;
        o[0] = '\t';
        o[1] = ans[i] ? '1' : '0';
        o[2] = '\n';
        o += 3;
    }
    return o;
}

// bytes format_range writes for keys [i0, i1)
uint64_t format_bytes(const uint64_t *keys, uint64_t i0, uint64_t i1) {
    static const uint64_t p10[20] = {1ull,
                                     10ull,
                                     100ull,
                                     1000ull,
                                     10000ull,
                                     100000ull,
                                     1000000ull,
                                     10000000ull,
                                     100000000ull,
                                     1000000000ull,
                                     10000000000ull,
                                     100000000000ull,
                                     1000000000000ull,
                                     10000000000000ull,
                                     100000000000000ull,
                                     1000000000000000ull,
                                     10000000000000000ull,
                                     100000000000000000ull,
                                     1000000000000000000ull,
                                     10000000000000000000ull};
    uint64_t total = 0;
    for (uint64_t i = i0; i < i1; ++i) {
        const uint64_t v = keys[i];
        // digits from the bit length (1233 / 4096 ~ log10 2), corrected by one compare
        const unsigned t = ((64u - (unsigned)__builtin_clzll(v | 1)) * 1233u) >> 12;
        total += t + ((v | 1) < p10[t] ? 0u : 1u) + 3u;
    }
    return total;
}
}  // namespace

extern "C" int bc_format_answers(const uint64_t *h_keys, const uint8_t *h_answers, uint64_t n,
                                 char *h_out, uint64_t out_cap, uint64_t *written) {
    if (!written) return fail(BC_EINVAL, "null byte count");
    *written = 0;
    if (n == 0) return BC_OK;
    if (!h_keys || !h_answers || !h_out) return fail(BC_EINVAL, "null keys, answers or output");
    if (out_cap / 23 < n) return fail(BC_EINVAL, "output buffer below 23 bytes per key");
    // large batches: a length pass gives every thread's output offset, then
    // each formats its keys straight into place
    const unsigned T = (unsigned)std::min<uint64_t>(host_text_threads(), n >> 17);
    if (T < 2) {
        *written = (uint64_t)(format_range(h_keys, h_answers, 0, n, h_out) - h_out);
        return BC_OK;
    }
    std::vector<uint64_t> at(T + 1, 0);
    {
        std::vector<std::thread> th;
        for (unsigned t = 0; t < T; ++t)
            th.emplace_back([&, t] { at[t + 1] = format_bytes(h_keys, n * t / T, n * (t + 1) / T); });
        for (auto &x : th) x.join();
    }
    for (unsigned t = 0; t < T; ++t) at[t + 1] += at[t];
    {
        std::vector<std::thread> th;
        for (unsigned t = 0; t < T; ++t)
            th.emplace_back([&, t] {
                format_range(h_keys, h_answers, n * t / T, n * (t + 1) / T, h_out + at[t]);
            });
        for (auto &x : th) x.join();
    }
    *written = at[T];
    return BC_OK;
}

// ---- text key ingestion ---------------------------------------------------------------
namespace {
inline bool is_space(char c) {
    return c == ' ' || c == '\t' || c == '\r' || c == '\v' || c == '\f' || c == '\n';
}

// One stripped, non-empty line -> value; false if int() would reject it or the
// value is outside [0, 2^64).
bool parse_line(const char *b, const char *e, u64 *v) {
    bool neg = false;
    if (*b == '+' || *b == '-') {
        neg = *b == '-';
        ++b;
    }
    if (b == e) return false;
    u64 acc = 0;
    bool prev_digit = false;
    for (const char *c = b; c < e; ++c) {
        if (*c == '_') {  // only between two digits
            if (!prev_digit || c + 1 == e || c[1] < '0' || c[1] > '9') return false;
            prev_digit = false;
            continue;
        }
        if (*c < '0' || *c > '9') return false;
        const u64 d = (u64)(*c - '0');
        if (acc > (~0ull - d) / 10) return false;  // >= 2^64
        acc = acc * 10 + d;
        prev_digit = true;
    }
    if (neg && acc != 0) return false;  // negative
    *v = acc;
    return true;
}
}  // namespace

static int parse_keys_serial(const char *h_text, uint64_t len, uint64_t *h_keys, uint64_t cap,
                             uint64_t *consumed, uint64_t *lines, uint64_t *n_keys);

// Large blocks are parsed by several threads: the text is cut at line ends
// into one segment per thread, a first pass counts each segment's lines and
// keys (memchr + strip), a second parses every segment straight into its
// place in h_keys.  Anything the serial parser would not run through to the
// end of the block -- more keys than cap, a rejected line -- is left to it, so
// the outputs and the error are the serial parser's in every case.
// BC_PARSE_THREADS (default min(16, cores); 1 = serial).
static bool parse_keys_parallel(const char *h_text, uint64_t len, uint64_t *h_keys, uint64_t cap,
                                uint64_t *consumed, uint64_t *lines, uint64_t *n_keys) {
    const u64 kMinSeg = 1ull << 20;
    const unsigned T = (unsigned)std::min<u64>(host_text_threads(), len / kMinSeg);
    if (T < 2) return false;
    // whole lines only: [0, stop) ends after the last '\n'
    const char *last = static_cast<const char *>(memrchr(h_text, '\n', (size_t)len));
    if (!last) return false;
    const u64 stop = (u64)(last - h_text) + 1;
    std::vector<u64> cut(T + 1, stop);
    cut[0] = 0;
    for (unsigned t = 1; t < T; ++t) {
        const u64 at = std::max(cut[t - 1], stop * t / T);
        const char *nl = at < stop ? static_cast<const char *>(
                                         std::memchr(h_text + at, '\n', (size_t)(stop - at)))
                                   : nullptr;
        cut[t] = nl ? (u64)(nl - h_text) + 1 : stop;
    }
    std::vector<u64> nkeys(T, 0), nlines(T, 0);
    auto each_line = [&](unsigned t, auto &&on_line) {
        const char *p = h_text + cut[t], *end = h_text + cut[t + 1];
        while (p < end) {
            const char *nl = static_cast<const char *>(std::memchr(p, '\n', (size_t)(end - p)));
            const char *b = p, *e = nl;
            while (b < e && is_space(*b)) ++b;
            while (e > b && is_space(e[-1])) --e;
            if (!on_line(b, e)) return false;
            p = nl + 1;
        }
        return true;
    };
    {
        std::vector<std::thread> th;
        for (unsigned t = 0; t < T; ++t)
            th.emplace_back([&, t] {
                u64 k = 0, l = 0;
                each_line(t, [&](const char *b, const char *e) {
                    k += b < e;
                    ++l;
                    return true;
                });
                nkeys[t] = k;
                nlines[t] = l;
            });
        for (auto &x : th) x.join();
    }
    u64 total = 0, total_lines = 0;
    std::vector<u64> at(T, 0);
    for (unsigned t = 0; t < T; ++t) {
        at[t] = total;
        total += nkeys[t];
        total_lines += nlines[t];
    }
    if (total > cap) return false;  // the serial parser stops at cap keys
    std::atomic<bool> bad{false};
    {
        std::vector<std::thread> th;
        for (unsigned t = 0; t < T; ++t)
            th.emplace_back([&, t] {
                u64 *out = h_keys + at[t];
                const bool ok = each_line(t, [&](const char *b, const char *e) {
                    if (b == e) return true;
                    u64 v;
                    if (!parse_line(b, e, &v)) return false;
                    *out++ = v;
                    return !bad.load(std::memory_order_relaxed);
                });
                if (!ok) bad.store(true, std::memory_order_relaxed);
            });
        for (auto &x : th) x.join();
    }
    if (bad.load()) return false;  // the serial parser words the error
    *consumed = stop;
    *lines = total_lines;
    *n_keys = total;
    return true;
}

extern "C" int bc_parse_keys_text(const char *h_text, uint64_t len, uint64_t *h_keys,
                                  uint64_t cap, uint64_t *consumed, uint64_t *lines,
                                  uint64_t *n_keys) {
    if (!consumed || !lines || !n_keys) return fail(BC_EINVAL, "null output counters");
    *consumed = *lines = *n_keys = 0;
    if (len && !h_text) return fail(BC_EINVAL, "null text");
    if (cap && !h_keys) return fail(BC_EINVAL, "null key buffer");
    if (parse_keys_parallel(h_text, len, h_keys, cap, consumed, lines, n_keys)) return BC_OK;
    *consumed = *lines = *n_keys = 0;
    return parse_keys_serial(h_text, len, h_keys, cap, consumed, lines, n_keys);
}

static int parse_keys_serial(const char *h_text, uint64_t len, uint64_t *h_keys, uint64_t cap,
                             uint64_t *consumed, uint64_t *lines, uint64_t *n_keys) {
    const char *p = h_text, *end = h_text + len;
    u64 n = 0, line = 0;
    while (p < end && n < cap) {
        const char *nl = static_cast<const char *>(std::memchr(p, '\n', (size_t)(end - p)));
        if (!nl) break;  // partial line: the caller carries it
        const char *b = p, *e = nl;
        while (b < e && is_space(*b)) ++b;
        while (e > b && is_space(e[-1])) --e;
        if (b < e) {
            u64 v;
            if (!parse_line(b, e, &v)) {
                *consumed = (u64)(p - h_text);
                *lines = line;
                *n_keys = n;
                return fail(BC_EINVAL, "line %llu of the chunk is not a 64-bit key",
                            (unsigned long long)line);
            }
            h_keys[n++] = v;
        }
        ++line;
        p = nl + 1;
    }
    *consumed = (u64)(p - h_text);
    *lines = line;
    *n_keys = n;
    return BC_OK;
}

// FASTA lines -> records joined with a separator byte (reference io.py:226-242,
// _read_fasta: lines stripped of surrounding whitespace, header lines close the
// record in progress, blank lines skipped, sequence before the first header is
// an error).  One memchr + memcpy per line.
extern "C" int bc_fasta_join(const char *h_text, uint64_t len, int at_eof, uint8_t sep,
                             uint32_t *state, uint8_t *h_out, uint64_t out_len_in,
                             uint64_t *out_len, uint64_t *rec_ends, uint64_t rec_cap,
                             uint64_t *n_recs, uint64_t *consumed) {
    if (!state || !out_len || !n_recs || !consumed) return fail(BC_EINVAL, "null output");
    if ((len && !h_text) || !h_out) return fail(BC_EINVAL, "null buffer");
    bool seen = (*state & 1u) != 0, open = (*state & 2u) != 0;
    const char *p = h_text, *end = h_text + len;
    u64 o = out_len_in, nr = 0;
    *out_len = o;
    *n_recs = 0;
    *consumed = 0;
    // an open record carried in h_out[0, out_len_in) must hold at least one base
    if (open && o == 0) return fail(BC_EINVAL, "open record without bytes");
    while (p < end) {
        const char *nl = static_cast<const char *>(std::memchr(p, '\n', (size_t)(end - p)));
        if (!nl) {
            if (!at_eof) break;  // partial line: the caller carries it
            nl = end;
        }
        const char *b = p, *e = nl;
        while (b < e && is_space(*b)) ++b;
        while (e > b && is_space(e[-1])) --e;
        if (b < e) {
            if (*b == '>') {
                if (open) {
                    if (nr >= rec_cap) break;  // table full: this line is not consumed
                    rec_ends[nr++] = o;
                    open = false;
                }
                seen = true;
            } else {
                if (!seen) return fail(BC_EINVAL, "FASTA input does not start with a header line");
                if (!open) {
                    if (o) h_out[o++] = sep;  // between records only
                    open = true;
                }
                std::memcpy(h_out + o, b, (size_t)(e - b));
                o += (u64)(e - b);
            }
        }
        p = nl < end ? nl + 1 : end;
    }
    if (at_eof && p == end && open && nr < rec_cap) {
        rec_ends[nr++] = o;
        open = false;
    }
    *state = (seen ? 1u : 0u) | (open ? 2u : 0u);
    *out_len = o;
    *n_recs = nr;
    *consumed = (u64)(p - h_text);
    return BC_OK;
}

// ---- parallel host copies -------------------------------------------------------------
// Pageable caller buffers are staged through pinned memory with memcpy; one
// thread copies ~14 GB/s, a quarter of the PCIe Gen5 link, so the copies of a
// chunk are split over a small persistent pool (BC_COPY_THREADS, default
// min(8, cores / 2); 1 disables).
namespace {
class CopyPool {
   public:
    static CopyPool &get() {
        static CopyPool pool;
        return pool;
    }

    void copy(void *dst, const void *src, size_t n) {
        const size_t kMin = 1 << 20;  // below this one thread is faster
        const int parts = (int)std::min<size_t>(workers_.size() + 1, std::max<size_t>(1, n / kMin));
        if (parts <= 1 || getpid() != pid_) {  // a forked child has no workers
            std::memcpy(dst, src, n);
            return;
        }
        const size_t per = ((n + parts - 1) / parts + 63) & ~size_t(63);  // parts * per >= n
        {
            std::lock_guard<std::mutex> lk(mu_);
            for (int i = 1; i < parts; ++i) {
                const size_t a = std::min(n, per * i), b = std::min(n, per * (i + 1));
                if (b > a) {
                    jobs_.push_back({static_cast<char *>(dst) + a,
                                     static_cast<const char *>(src) + a, b - a});
                    ++pending_;
                }
            }
        }
        cv_.notify_all();
        std::memcpy(dst, src, std::min(n, per));  // the caller's share
        std::unique_lock<std::mutex> lk(mu_);
        done_.wait(lk, [&] { return pending_ == 0; });
    }

   private:
    struct Job {
        char *dst;
        const char *src;
        size_t n;
    };

    CopyPool() : pid_(getpid()) {
        int t = 0;
        if (const char *e = std::getenv("BC_COPY_THREADS")) t = std::atoi(e) - 1;
        else t = (int)std::min(8u, std::max(1u, std::thread::hardware_concurrency() / 2)) - 1;
        for (int i = 0; i < t; ++i) workers_.emplace_back([this] { run(); });
    }

    ~CopyPool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto &w : workers_) w.join();
    }

    void run() {
        for (;;) {
            Job j;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return stop_ || !jobs_.empty(); });
                if (stop_ && jobs_.empty()) return;
                j = jobs_.back();
                jobs_.pop_back();
            }
            std::memcpy(j.dst, j.src, j.n);
            std::lock_guard<std::mutex> lk(mu_);
            if (--pending_ == 0) done_.notify_all();
        }
    }

    std::vector<std::thread> workers_;
    std::vector<Job> jobs_;
    std::mutex mu_;
    std::condition_variable cv_, done_;
    int pending_ = 0;
    bool stop_ = false;
    const pid_t pid_;
};

void host_copy(void *dst, const void *src, size_t n) { CopyPool::get().copy(dst, src, n); }
}  // namespace

// ---- host-buffer entry points ---------------------------------------------------------
// Per-device staging: two pinned key buffers, two pinned answer buffers, two
// device key/answer buffers and two copy streams, so the copy of chunk i+1
// (and the answers of chunk i-1) overlap the kernel of chunk i, while the
// kernels themselves run in order on the caller's stream.
namespace {
constexpr u64 kStageKeys = 1ull << 22;  // 32 MiB of keys per buffer

struct Staging {
    std::mutex mu;
    bool ready = false;
    u64 *h_keys[2] = {nullptr, nullptr};
    u8 *h_out[2] = {nullptr, nullptr};
    u64 *d_keys[2] = {nullptr, nullptr};
    u8 *d_out[2] = {nullptr, nullptr};
    cudaStream_t cs[2] = {nullptr, nullptr};
    cudaEvent_t h2d[2], kdone[2], done[2];
};

std::mutex g_stage_mu;
std::map<int, Staging *> g_stage;

Staging *staging_for(int dev) {
    std::lock_guard<std::mutex> lk(g_stage_mu);
    auto it = g_stage.find(dev);
    if (it != g_stage.end()) return it->second;
    Staging *st = new Staging();
    g_stage[dev] = st;
    return st;
}

int staging_init(Staging *st) {
    if (st->ready) return BC_OK;
    for (int b = 0; b < 2; ++b) {
        CUDA_TRY(cudaHostAlloc((void **)&st->h_keys[b], sizeof(u64) * kStageKeys,
                               cudaHostAllocDefault));
        CUDA_TRY(cudaHostAlloc((void **)&st->h_out[b], kStageKeys, cudaHostAllocDefault));
        CUDA_TRY(cudaMalloc((void **)&st->d_keys[b], sizeof(u64) * kStageKeys));
        CUDA_TRY(cudaMalloc((void **)&st->d_out[b], kStageKeys));
        CUDA_TRY(cudaStreamCreateWithFlags(&st->cs[b], cudaStreamNonBlocking));
        CUDA_TRY(cudaEventCreateWithFlags(&st->h2d[b], cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&st->kdone[b], cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&st->done[b], cudaEventDisableTiming));
        CUDA_TRY(cudaEventRecord(st->done[b], st->cs[b]));
    }
    st->ready = true;
    return BC_OK;
}

bool is_pinned(const void *p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}
}  // namespace

static int host_pipeline(bc_filter *f, u64 *words, const u64 *h_keys, u64 n, int op, int mode,
                         u8 *h_out, unsigned long long *h_hits, cudaStream_t s) {
    Staging *st = staging_for(f->device);
    std::lock_guard<std::mutex> lk(st->mu);
    if (int rc = staging_init(st)) return rc;
    const bool keys_pinned = is_pinned(h_keys);
    const bool out_pinned = h_out != nullptr && is_pinned(h_out);
    unsigned long long *d_hits = nullptr;
    if (h_hits) {
        CUDA_TRY(cudaMallocAsync((void **)&d_hits, sizeof(*d_hits), s));
        CUDA_TRY(cudaMemsetAsync(d_hits, 0, sizeof(*d_hits), s));
    }
    // the copy streams must not start before earlier work on `s`
    cudaEvent_t start;
    CUDA_TRY(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
    struct EventGuard {
        cudaEvent_t e;
        ~EventGuard() { cudaEventDestroy(e); }
    } start_guard{start};
    CUDA_TRY(cudaEventRecord(start, s));
    for (int b = 0; b < 2; ++b) CUDA_TRY(cudaStreamWaitEvent(st->cs[b], start, 0));

    struct Pending {
        u64 off = 0, len = 0;
        bool live = false;
    } pend[2];
    int rc = BC_OK;
    u64 chunk_i = 0;
    // at least four chunks for mid-size batches, so copies overlap kernels
    const u64 chunk = std::min(kStageKeys, std::max<u64>(1ull << 18, (n + 3) / 4));
    for (u64 off = 0; off < n && rc == BC_OK; off += chunk, ++chunk_i) {
        const int b = (int)(chunk_i & 1);
        const u64 len = std::min(chunk, n - off);
        // The device buffers of slot b are reused in stream order (copy stream
        // b queues behind its previous D2H, which waited for that chunk's
        // kernel); only the host staging buffers need the host to wait.
        if (!keys_pinned || (h_out && !out_pinned))
            CUDA_TRY(cudaEventSynchronize(st->done[b]));  // staging slot b is free again
        if (pend[b].live && h_out && !out_pinned)
            host_copy(h_out + pend[b].off, st->h_out[b], pend[b].len);
        pend[b].live = false;
        const u64 *src = h_keys + off;
        if (!keys_pinned) {
            host_copy(st->h_keys[b], src, sizeof(u64) * len);
            src = st->h_keys[b];
        }
        CUDA_TRY(cudaMemcpyAsync(st->d_keys[b], src, sizeof(u64) * len, cudaMemcpyHostToDevice,
                                 st->cs[b]));
        CUDA_TRY(cudaEventRecord(st->h2d[b], st->cs[b]));
        CUDA_TRY(cudaStreamWaitEvent(s, st->h2d[b], 0));
        if (op == OP_INSERT)
            rc = insert_device(f, words, st->d_keys[b], len, mode, s);
        else
            rc = contains_device(f, words, st->d_keys[b], len, h_out ? st->d_out[b] : nullptr,
                                 d_hits, s);
        if (rc) break;
        CUDA_TRY(cudaEventRecord(st->kdone[b], s));
        CUDA_TRY(cudaStreamWaitEvent(st->cs[b], st->kdone[b], 0));
        if (h_out) {
            u8 *dst = out_pinned ? h_out + off : st->h_out[b];
            CUDA_TRY(cudaMemcpyAsync(dst, st->d_out[b], len, cudaMemcpyDeviceToHost, st->cs[b]));
            pend[b] = {off, len, true};
        }
        CUDA_TRY(cudaEventRecord(st->done[b], st->cs[b]));
    }
    for (int b = 0; b < 2; ++b) {
        CUDA_TRY(cudaEventSynchronize(st->done[b]));
        if (pend[b].live && h_out && !out_pinned)
            host_copy(h_out + pend[b].off, st->h_out[b], pend[b].len);
    }
    if (d_hits) {
        unsigned long long v = 0;
        CUDA_TRY(cudaMemcpyAsync(&v, d_hits, sizeof v, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaFreeAsync(d_hits, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        *h_hits += v;
    }
    CUDA_TRY(cudaStreamSynchronize(s));
    return rc;
}

extern "C" int bc_insert_peers(bc_filter *f, uint64_t *const *h_parts, int nparts,
                               const uint64_t *d_keys, uint64_t n, uint64_t keys_in_flight,
                               void *stream) {
    if (!f) return fail(BC_EINVAL, "null filter");
    if (!h_parts || nparts < 1 || nparts > kMaxParts)
        return fail(BC_EINVAL, "nparts must be in [1, %d]", kMaxParts);
    if (n && !d_keys) return fail(BC_EINVAL, "null keys");
    for (int r = 0; r < nparts; ++r) {
        if (!h_parts[r]) return fail(BC_EINVAL, "null replica pointer %d", r);
        if (reinterpret_cast<uintptr_t>(h_parts[r]) % 64)
            return fail(BC_EINVAL, "replica %d is not 64-byte aligned", r);
    }
    if (f->kind == BC_KIND_STANDARD || f->kp.c < 2 || f->kp.c > 4 || !f->kp.fast_random ||
        f->kp.wpb != 8)
        return fail(BC_EUNSUP,
                    "partitioned inserts need 2..4 choices, 512-bit blocks, random strategy");
    if (int rc = check_device(f)) return rc;
    if (n == 0) return BC_OK;
    KParams kp = f->kp;
    // keys in flight: 256 per CTA (relaxed512 tiles); the caller's share of
    // the M/2 the relaxed tolerance is stated for
    const u64 inflight = keys_in_flight ? keys_in_flight : std::max<u64>(1, kp.num_blocks / 2);
    kp.max_ctas = (u32)std::max<u64>(1, std::min<u64>(inflight / 256, 0xffffffffu));
    CUDA_TRY(launch_relaxed_peers(kp, h_parts, nparts, d_keys, n, (cudaStream_t)stream));
    return BC_OK;
}

extern "C" int bc_insert_host(bc_filter *f, uint64_t *d_words, const uint64_t *h_keys,
                              uint64_t n, int mode, void *stream) {
    if (!f) return fail(BC_EINVAL, "null filter");
    if (n && (!d_words || !h_keys)) return fail(BC_EINVAL, "null words or keys");
    if (mode != BC_INSERT_ORDERED && mode != BC_INSERT_RELAXED)
        return fail(BC_EINVAL, "unknown insert mode %d", mode);
    if (int rc = check_device(f)) return rc;
    if (n == 0) return BC_OK;
    return host_pipeline(f, d_words, h_keys, n, OP_INSERT, mode, nullptr, nullptr,
                         (cudaStream_t)stream);
}

extern "C" int bc_contains_host(bc_filter *f, const uint64_t *d_words, const uint64_t *h_keys,
                                uint64_t n, uint8_t *h_out, unsigned long long *h_hits,
                                void *stream) {
    if (!f) return fail(BC_EINVAL, "null filter");
    if (n && (!d_words || !h_keys)) return fail(BC_EINVAL, "null words or keys");
    if (int rc = check_device(f)) return rc;
    if (n == 0) return BC_OK;
    return host_pipeline(f, const_cast<u64 *>(d_words), h_keys, n, OP_CONTAINS, 0, h_out,
                         h_hits, (cudaStream_t)stream);
}
