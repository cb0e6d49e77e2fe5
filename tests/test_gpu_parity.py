"""Parity of the CUDA path (through the C ABI) with the reference.

* against the reference's own golden vectors (tests/golden): bit arrays,
  lookup answers, histograms, q-gram keys, the DNA case;
* against the CPU oracle (oracle/, pinned to the same vectors) on seeded
  inputs too large for committed fixtures;
* size-independent properties at BASELINE sizes (no false negatives,
  idempotence, monotonicity, histogram conservation).
"""

import hashlib
import os

import numpy as np
import pytest
import torch

import paper_2501_18977_b200 as bb
from oracle import oracle as orc

pytestmark = pytest.mark.gpu

CASES = [
    "std_k7", "blk_rand_k7", "blk_dist_k7", "bc2_rand_k7", "bc2_dist_k7", "bc3_rand_k7",
    "bc2_rand_b16", "bc2_dist_b16", "bc3_k12_20k", "bc2_k6_t4", "blk_k9_t8", "bc3_dist_k10",
    "bc4_k8", "bc8_k5", "bc2_mix", "bc3_la", "bc2_exp13", "bc2_b64", "bc2_b128", "bc2_b1024",
    "blk_b8", "bc3_b32_dist", "bc2_dist_k40", "std_k10_odd", "bc2_overfill",
    "cfg1", "cfg2_small", "cfg3_small", "cfg5_small_k11",
]


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def config_of(case):
    cfg = dict(case["config"])
    if isinstance(cfg.get("cost"), dict):
        c = cfg["cost"]
        cfg["cost"] = bb.CostModel(c["kind"], c["param"], c["k"])
    return bb.FilterConfig(**cfg)


def probes_of(case):
    keys = bb.even_keys(case["n_insert"], case["insert_seed"])
    pos = keys[: max(1, case["n_insert"] // 2)]
    return keys, np.concatenate([pos, bb.odd_keys(case["n_neg"], case["neg_seed"])])


@pytest.mark.parametrize("name", CASES)
def test_ordered_build_and_lookup_match_reference(golden, name):
    meta, arr = golden
    case = meta[name]
    f = bb.Filter.from_config(config_of(case))
    keys, probes = probes_of(case)
    f.insert_many(keys)
    words = f.storage.words
    if f"{name}__words" in arr:
        np.testing.assert_array_equal(words, arr[f"{name}__words"])
    assert sha(words) == case["words_sha256"]
    out = f.contains_many(probes).astype(np.uint8)
    assert sha(out) == case["out_sha256"]
    assert f.count_hits(probes) == case["hits_pos"] + case["hits_neg"]
    if f.kind != "standard":
        hist = bb.block_load_histogram(f)
        assert sha(hist.counts.astype(np.int64)) == case["hist_sha256"]
    assert f.inserted == keys.shape[0]


@pytest.mark.parametrize("name", ["cfg1", "cfg2_small", "bc3_k12_20k", "bc2_k6_t4",
                                  "bc2_dist_k7", "bc2_rand_b16", "std_k10_odd"])
def test_device_tensor_inputs(golden, name):
    """CUDA-tensor keys stay on the device and give the same answers."""
    meta, _ = golden
    case = meta[name]
    f = bb.Filter.from_config(config_of(case))
    keys, probes = probes_of(case)
    f.insert_many(torch.from_numpy(keys).cuda())
    assert sha(f.storage.words) == case["words_sha256"]
    out = f.contains_many(torch.from_numpy(probes).cuda())
    assert out.is_cuda and out.dtype == torch.bool
    assert sha(out.cpu().numpy().astype(np.uint8)) == case["out_sha256"]
    assert f.count_hits(torch.from_numpy(probes).cuda()) == case["hits_pos"] + case["hits_neg"]


@pytest.mark.parametrize("name", ["cfg1", "bc3_k12_20k", "bc2_k6_t4", "bc3_dist_k10",
                                  "bc8_k5", "bc2_b1024", "cfg3_small", "cfg5_small_k11"])
def test_relaxed_build_tolerance(golden, name):
    """Relaxed multi-choice inserts against the exact-order build of the same
    stream (itself pinned to the reference's words), with SURVEY §8(a)'s
    tolerances written here: zero false negatives; |log2 FPR_relaxed -
    log2 FPR_exact| <= 0.1 + 3 sigma over 2^24 device-generated negatives;
    mean block load within 1 bit; load variance within 15% (plus 3 sigma of
    the variance estimate over the filter's M blocks); and, for filters
    of at least 2^15 blocks (config 1 and up, where the tolerance is stated),
    the unbinned load-histogram total variation <= 0.05."""
    import math

    meta, _ = golden
    case = meta[name]
    keys, _ = probes_of(case)
    exact = bb.Filter.from_config(config_of(case))
    exact.insert_many(keys)
    assert sha(exact.storage.words) == case["words_sha256"]
    f = bb.Filter.from_config(config_of(case), insert_mode="relaxed")
    f.insert_many(keys)
    assert f.contains_many(keys).all()
    neg = bb.odd_keys(1 << 24, 12, device="cuda")
    fp_e, fp_r = exact.count_hits(neg), f.count_hits(neg)
    sigma = math.sqrt(1 / max(fp_e, 1) + 1 / max(fp_r, 1)) / math.log(2)
    assert abs(math.log2(max(fp_r, 1) / max(fp_e, 1))) <= 0.1 + 3 * sigma, (fp_e, fp_r)
    h_r, h_e = bb.block_load_histogram(f), bb.block_load_histogram(exact)
    assert abs(h_r.mean_load - h_e.mean_load) <= 1.0, (h_r.mean_load, h_e.mean_load)
    # 15% plus 3 sigma of the variance estimate itself over M blocks
    # (sqrt(2 / M) relative): a 57-block filter's variance is not resolvable
    # to 15%, a config-1 filter's (2^15 blocks) is to within 2.3 points
    tol = 0.15 + 3 * math.sqrt(2.0 / f.num_blocks)
    assert abs(h_r.variance / h_e.variance - 1) <= tol, (h_r.variance, h_e.variance, tol)
    if f.num_blocks >= 1 << 15:
        tv = bb.histogram_distance(h_r.counts, h_e.counts)
        assert tv <= 0.05, tv


def test_relaxed_equals_ordered_for_single_choice(golden):
    meta, _ = golden
    case = meta["cfg2_small"]
    f = bb.Filter.from_config(config_of(case), insert_mode="relaxed")
    keys, _ = probes_of(case)
    f.insert_many(keys)
    assert sha(f.storage.words) == case["words_sha256"]


def test_lookups_on_oracle_built_words_are_bit_identical():
    """Lookups on a bit array built elsewhere (the oracle) give identical answers."""
    for kind, c, k in [("blocked", 1, 12), ("blowchoc", 2, 14), ("blowchoc", 3, 16)]:
        o = orc.make_filter(kind, k=k, choices=c, size_bits=k * 2**16, seed=3)
        o.insert_many(orc.even_keys(2**16, 4))
        f = bb.Filter.from_config(bb.FilterConfig(kind=kind, k=k, choices=c,
                                                  size_bits=k * 2**16, seed=3),
                                  words=o.words)
        probes = np.concatenate([orc.even_keys(2**15, 4), orc.odd_keys(2**18, 5)])
        np.testing.assert_array_equal(f.contains_many(probes), o.contains_many(probes))


@pytest.mark.parametrize("kind,c,k,shards", [
    ("blocked", 1, 1, 1), ("blocked", 1, 3, 1), ("blocked", 1, 4, 1), ("blocked", 1, 9, 4),
    ("blocked", 1, 16, 1), ("blocked", 1, 17, 1), ("blocked", 1, 24, 2), ("blocked", 1, 40, 1),
    ("blowchoc", 2, 3, 1), ("blowchoc", 2, 11, 2), ("blowchoc", 4, 20, 1),
])
def test_lookup_kernels_every_k(kind, c, k, shards):
    """Inserts and lookups over the k range: compile-time-k lookup kernels
    (4 <= k <= 16), the runtime-k fallback and sharded layouts, against the
    oracle on the same seeded keys; ragged batch tails included."""
    n = 3 * 2**13 + 5
    o = orc.make_filter(kind, k=k, choices=c, size_bits=k * n, seed=7 + k, shards=shards)
    keys = orc.even_keys(n, 8)
    o.insert_many(keys)
    f = bb.Filter.from_config(bb.FilterConfig(kind=kind, k=k, choices=c, size_bits=k * n,
                                              seed=7 + k, shards=shards))
    f.insert_many(keys)
    np.testing.assert_array_equal(f.storage.words, o.words)
    probes = np.concatenate([keys[::3], orc.odd_keys(2**16 + 3, 9)])
    np.testing.assert_array_equal(f.contains_many(probes), o.contains_many(probes))


def test_cfg2_full_size_bit_identical():
    """BASELINE config 2 at full size: 2^26 keys, k=12, 12 bits/key; the GPU
    bit array equals the oracle's (threaded OR build, itself pinned to the
    reference's cfg2_small digest)."""
    n = 2**26
    cfg = bb.FilterConfig(kind="blocked", k=12, size_bits=12 * n, seed=1)
    keys = bb.even_keys(n, 11)
    f = bb.Filter.from_config(cfg)
    f.insert_many(torch.from_numpy(keys).cuda())
    o = orc.make_filter("blocked", k=12, size_bits=12 * n, seed=1)
    o.insert_many_mt(keys, threads=8)
    np.testing.assert_array_equal(f.storage.words, o.words)
    probes = np.concatenate([keys[::2], bb.odd_keys(n // 2, 12)])
    got = f.contains_many(torch.from_numpy(probes).cuda()).cpu().numpy()
    np.testing.assert_array_equal(got, o.contains_many(probes, threads=8))


def test_cfg3_properties_full_size():
    """Config 3 geometry (c=3, k=16, 512 MiB): relaxed build of 2^28 keys has
    no false negatives on a sample and an FPR near the reference's 4.84e-4."""
    n = 2**28
    cfg = bb.FilterConfig(kind="blowchoc", k=16, choices=3, size_bits=16 * n, seed=1)
    f = bb.Filter.from_config(cfg, insert_mode="relaxed")
    gen = torch.Generator(device="cuda").manual_seed(7)
    keys = (torch.randint(-2**63, 2**63 - 1, (n,), device="cuda", dtype=torch.int64,
                          generator=gen) & ~1)
    f.insert_many(keys)
    sample = keys[:: 97]
    assert f.count_hits(sample) == sample.numel()
    neg = torch.randint(-2**63, 2**63 - 1, (2**26,), device="cuda", dtype=torch.int64,
                        generator=gen) | 1
    fpr = f.count_hits(neg) / neg.numel()
    assert 3.5e-4 < fpr < 6.5e-4
    hist = bb.block_load_histogram(f)
    assert hist.counts.sum() == f.num_blocks
    assert hist.total_set_bits == f.storage.total_set_bits()


@pytest.mark.parametrize("name,c,k,size_bits,n", [
    # config 3 geometry: 512 MiB, M = 2^23 (one claim slot per block)
    ("cfg3", 3, 16, 16 * 2**28, 2**23),
    # config 5 geometry: 8 GiB, M = 2^27 blocks hashed onto 2^23 claim slots
    ("cfg5", 2, 11, 2**36, 2**22),
    # the ticket dataflow's largest default: 3 * 2^17 blocks
    ("ticket_max_c2", 2, 14, 3 * 2**26, 2**23),
    ("ticket_max_c3", 3, 16, 3 * 2**26, 2**23),
    # the smallest filters on the claim rounds: identity claim slots, window M / (2 c^2)
    ("claims_min_c2", 2, 14, 512 * (3 * 2**17 + 1), 2**23),
    ("claims_min_c3", 3, 16, 512 * (3 * 2**17 + 1), 2**23),
    ("claims_2p21_c3", 3, 16, 2**30, 2**23),
])
def test_exact_order_full_geometry_matches_oracle(name, c, k, size_bits, n):
    """Exact-order builds on the full-size filters of configs 3 and 5 (claim
    rounds), at the ticket dataflow's largest default sizes and just above
    them (only the key count is reduced so the sequential oracle finishes in
    seconds):
    bit-identical words, and identical answers on a mixed probe set."""
    cfg = bb.FilterConfig(kind="blowchoc", k=k, choices=c, size_bits=size_bits, seed=1)
    keys = bb.even_keys(n, 11)
    f = bb.Filter.from_config(cfg, insert_mode="ordered")
    f.insert_many(torch.from_numpy(keys).cuda())
    o = orc.make_filter("blowchoc", k=k, choices=c, size_bits=size_bits, seed=1)
    o.insert_many(keys)
    got = f.storage.d_words.cpu().numpy()
    assert np.array_equal(got, o.words), f"{name}: exact-order words differ from the oracle"
    probes = np.concatenate([keys[::5], bb.odd_keys(2**20, 12)])
    ans = f.contains_many(torch.from_numpy(probes).cuda()).cpu().numpy()
    np.testing.assert_array_equal(ans, o.contains_many(probes, threads=8))


def test_exact_order_full_size_split_and_reinsert():
    """Config 3 at full size (2^28 keys, exact order): building in two calls
    gives the same bits as one call (stream order is the only input), and
    inserting the stream again changes nothing (every key is then a no-op
    under the reference's rule, _kernels.py:156-160)."""
    n = 2**28
    cfg = bb.FilterConfig(kind="blowchoc", k=16, choices=3, size_bits=16 * n, seed=1)
    keys = bb.even_keys(n, 11, device="cuda")
    f = bb.Filter.from_config(cfg, insert_mode="ordered")
    f.insert_many(keys)
    one = f.storage.d_words.clone()
    g = bb.Filter.from_config(cfg, insert_mode="ordered")
    h = 3 * n // 7
    g.insert_many(keys[:h])
    g.insert_many(keys[h:])
    assert torch.equal(g.storage.d_words, one)
    f.insert_many(keys)
    assert torch.equal(f.storage.d_words, one)
    assert f.count_hits(keys[::101]) == keys[::101].numel()


def test_relaxed_vs_exact_order_cfg5_full_size():
    """Config 5 at full size (8 GiB, k = 11, 1.2 x 2^32 keys): the relaxed
    build against the bit-exact build of the same stream, with the relaxed
    tolerances of SURVEY §8(a) written here: no false negatives, FPR within
    0.1 in log2 plus 3 sigma, mean block load within 1 bit, load variance
    within 15%, histogram total variation <= 0.05."""
    import math

    from paper_2501_18977_b200.analysis import histogram_distance

    n = int(1.2 * 2**32)
    cfg = bb.FilterConfig(kind="blowchoc", k=11, choices=2, size_bits=2**36, seed=1)
    keys = bb.even_keys(n, 11, device="cuda")
    neg = bb.odd_keys(2**26, 12, device="cuda")
    res = {}
    for mode in ("ordered", "relaxed"):
        f = bb.Filter.from_config(cfg, insert_mode=mode)
        f.insert_many(keys)
        assert f.count_hits(keys[::997]) == keys[::997].numel(), f"{mode}: false negatives"
        res[mode] = (f.count_hits(neg), bb.block_load_histogram(f))
        del f
        torch.cuda.empty_cache()
    (fp_e, h_e), (fp_r, h_r) = res["ordered"], res["relaxed"]
    sigma = math.sqrt(1 / fp_e + 1 / fp_r) / math.log(2)  # stderr of the log2 ratio
    assert abs(math.log2(fp_r / fp_e)) <= 0.1 + 3 * sigma, (fp_e, fp_r)
    assert abs(h_r.mean_load - h_e.mean_load) <= 1.0
    assert abs(h_r.variance / h_e.variance - 1) <= 0.15
    assert histogram_distance(h_r.counts, h_e.counts) <= 0.05


def test_dna_full_genome_fused_equals_composition():
    """Config 4 scale: a seeded 1.2e9-bp genome.  The fused canonical 31-mer
    insert equals insert_many(encode_qgrams(genome)) bit for bit (one choice:
    order-free), and fused count-only lookups of 10^6 reads with 1%
    substitutions equal the materialised lookups; the true-read k-mer hit
    rate is near 0.99^31 = 0.732."""
    L, R, RL = 1_200_000_000, 10**6, 150
    g = torch.Generator(device="cuda").manual_seed(4)
    lut = torch.tensor(list(b"ACGT"), dtype=torch.uint8, device="cuda")
    codes = torch.randint(0, 4, (L,), device="cuda", dtype=torch.uint8, generator=g)
    genome = lut[codes.long()]
    start = torch.randint(0, L - RL, (R, 1), device="cuda", dtype=torch.int64, generator=g)
    c = codes[start + torch.arange(RL, device="cuda")]
    del codes
    sub = torch.rand((R, RL), device="cuda", generator=g) < 0.01
    shift = torch.randint(1, 4, (R, RL), device="cuda", dtype=torch.uint8, generator=g)
    reads = lut[torch.where(sub, (c + shift) % 4, c).long()]  # (R, RL): one record per row
    enc = bb.QGramEncoder(q=31, canonical=True)
    cfg = bb.FilterConfig(kind="blocked", k=14, size_bits=14 * (L - 30), seed=1)
    fused = bb.Filter.from_config(cfg)
    assert fused.insert_qgrams(enc, genome) == L - 30
    comp = bb.Filter.from_config(cfg)
    keys = bb.encode_qgrams(enc, genome)
    assert keys.numel() == L - 30
    comp.insert_many(keys)
    del keys
    assert torch.equal(fused.storage.d_words, comp.storage.d_words)
    hits = fused.count_qgram_hits(enc, reads)
    rk = bb.encode_qgrams(enc, reads)
    assert rk.numel() == R * (RL - 30)
    assert hits == comp.count_hits(rk)
    assert 0.72 < hits / rk.numel() < 0.75


# -- edge cases ------------------------------------------------------------------------

@pytest.mark.parametrize("kind,c", [("standard", None), ("blocked", 1), ("blowchoc", 2),
                                    ("blowchoc", 3)])
def test_empty_and_ragged_batches(kind, c):
    cfg = bb.FilterConfig(kind=kind, k=8, n_capacity=5000, choices=c, seed=9)
    f = bb.Filter.from_config(cfg)
    o = orc.make_filter(kind, k=8, n_capacity=5000, choices=c, seed=9)
    f.insert_many(np.empty(0, dtype=np.uint64))
    assert f.contains_many(np.empty(0, dtype=np.uint64)).shape == (0,)
    assert f.count_hits(np.empty(0, dtype=np.uint64)) == 0
    keys = bb.even_keys(4097, 3)
    for lo, hi in [(0, 1), (1, 256), (256, 257), (257, 1000), (1000, 4097)]:
        f.insert_many(keys[lo:hi])
        o.insert_many(keys[lo:hi])
    np.testing.assert_array_equal(f.storage.words, o.words)
    for n in (1, 2, 255, 256, 257, 1023):
        p = bb.odd_keys(n, n)
        np.testing.assert_array_equal(f.contains_many(p), o.contains_many(p))


def test_idempotent_and_monotone():
    f = bb.Filter.from_config(bb.FilterConfig(kind="blowchoc", k=8, n_capacity=10_000, seed=5))
    keys = bb.even_keys(10_000, 9)
    f.insert_many(keys)
    bits = f.storage.total_set_bits()
    f.insert_many(keys)
    assert f.storage.total_set_bits() == bits
    probes = bb.odd_keys(50_000, 3)
    seen = f.contains_many(probes)
    f.insert_many(bb.even_keys(10_000, 10))
    assert (f.contains_many(probes) | ~seen).all()


def test_host_edits_reach_the_device():
    f = bb.Filter.from_config(bb.FilterConfig(kind="blocked", k=4, n_capacity=100))
    assert f.load() == 0.0
    f.storage.words[:] = ~np.uint64(0)
    assert f.load() == 1.0
    assert f.contains_many(bb.odd_keys(100, 1)).all()


def test_scalar_api_roundtrip():
    for kind, c, strategy in [("standard", None, "random"), ("blocked", 1, "distinct"),
                              ("blowchoc", 3, "random"), ("blowchoc", 2, "distinct")]:
        f = bb.Filter.from_config(bb.FilterConfig(kind=kind, k=5, n_capacity=500, choices=c,
                                                  strategy=strategy, seed=3))
        keys = bb.even_keys(100, 7).tolist()
        for x in keys:
            f.insert(x)
            assert f.lookup(x)
        assert all(x in f for x in keys)


def test_split_bits_across_choices_is_negative():
    f = bb.Filter.from_config(bb.FilterConfig(kind="blowchoc", k=2, size_bits=64, choices=2,
                                              block_bits=16, seed=21))
    addrs = sorted(f.bit_selector.select(77))
    blocks = f.candidate_blocks(77)
    if len(addrs) >= 2 and blocks[0] != blocks[1]:
        f.storage.set_bits(blocks[0], addrs[:1])
        f.storage.set_bits(blocks[1], addrs[1:])
        assert not f.lookup(77)


def test_eval_hash_many_and_routing(golden):
    _, arr = golden
    a, b, x, h = arr["hash__a"], arr["hash__b"], arr["hash__x"], arr["hash__h"]
    for bv in np.unique(b)[:40]:
        sel = b == bv
        for av in np.unique(a[sel])[:2]:
            s2 = sel & (a == av)
            got = bb.eval_hash_many(bb.HashSpec(a=int(av), b=int(bv)), x[s2])
            np.testing.assert_array_equal(got, h[s2])
    f = bb.Filter.from_config(bb.FilterConfig(kind="blowchoc", k=6, n_capacity=5000,
                                              shards=4, seed=61))
    keys = bb.even_keys(3000, 1)
    np.testing.assert_array_equal(f.route_many(keys), [f.shard_of(int(v)) for v in keys])


def test_eval_hash_modulus_paths():
    """The device remainder (single-multiply Barrett) for odd
    and even ranges from 3 to 2^64 - 1, against Python's exact integers --
    random keys plus keys that put a*x just below, on and above multiples
    of b."""
    rng = np.random.default_rng(8)
    ranges = [3, 5, 6, 1000, 1_572_864, 32_812_500, (1 << 30) - 2, (1 << 30) - 1,
              (1 << 30) + 1, (1 << 30) + 2, 3 << 40, (1 << 63) + 7, (1 << 64) - 1]
    ranges += [int(v) for v in rng.integers(3, 1 << 30, 20)]
    for b in ranges:
        if b & (b - 1) == 0:
            continue
        for a in (0x9E3779B97F4A7C15, int(rng.integers(1, 2**63)) * 2 + 1):
            a |= 1 << 63 | 1
            x = [int(v) for v in rng.integers(0, 2**64, 2000, dtype=np.uint64)]
            ainv = pow(a, -1, 1 << 64)
            for t in (1, 2, 3, 7):  # a*x = t*b + {-1, 0, 1} (mod 2^64)
                for d in (-1, 0, 1):
                    x.append(((t * b + d) % (1 << 64)) * ainv % (1 << 64))
            x += [0, 1, (1 << 64) - 1, 1 << 63]
            keys = np.array(x, dtype=np.uint64)
            got = bb.eval_hash_many(bb.HashSpec(a=a, b=b), keys)
            want = []
            for v in x:
                ax = a * v % (1 << 64)
                if b % 2 == 0:
                    ax ^= ax >> 32
                want.append(ax % b)
            np.testing.assert_array_equal(got, np.array(want, dtype=np.uint64), err_msg=str(b))


def test_sharded_build_equals_sequential():
    cfg = bb.FilterConfig(kind="blowchoc", k=7, n_capacity=20_000, choices=3, shards=8, seed=4)
    keys = bb.even_keys(20_000, 5)
    a = bb.build_sequential(cfg, keys)
    b = bb.build_sharded(cfg, [keys[:7000], keys[7000:]])
    np.testing.assert_array_equal(a.storage.words, b.storage.words)
    o = orc.make_filter("blowchoc", k=7, n_capacity=20_000, choices=3, shards=8, seed=4)
    o.insert_many(keys)
    np.testing.assert_array_equal(a.storage.words, o.words)


def test_estimate_fpr_and_histogram_vs_oracle():
    cfg = bb.FilterConfig(kind="blowchoc", k=10, n_capacity=50_000, choices=2, seed=2)
    f = bb.Filter.from_config(cfg)
    keys = bb.even_keys(50_000, 3)
    f.insert_many(keys)
    o = orc.make_filter("blowchoc", k=10, n_capacity=50_000, choices=2, seed=2)
    o.insert_many(keys)
    np.testing.assert_array_equal(bb.block_load_histogram(f).counts,
                                  o.block_histogram().astype(np.int64))
    neg = bb.odd_keys(2**20, 8)
    est = bb.estimate_fpr(f, neg)
    assert est.false_positives == int(o.contains_many(neg).sum())
    est2 = bb.estimate_fpr(f, n_queries=2**20, chunk_size=2**18)
    assert est2.n_queries == 2**20


# -- q-grams ---------------------------------------------------------------------------

def test_qgram_kats(golden):
    meta, arr = golden
    for kat in meta["qgram_kats"]:
        got = bb.encode_qgrams(bb.QGramEncoder(kat["q"], kat["canonical"]), kat["seq"])
        assert got.tolist() == [int(v) for v in kat["keys"]]
    for case in meta["qgrams"]:
        i = case["idx"]
        enc = bb.QGramEncoder(case["q"], case["canonical"])
        got = bb.encode_qgrams(enc, arr[f"qg__{i}__seq"].tobytes())
        np.testing.assert_array_equal(got, arr[f"qg__{i}__keys"])


def test_qgram_long_sequence_vs_oracle():
    rng = np.random.default_rng(11)
    seq = np.frombuffer(b"ACGTacgtN", dtype=np.uint8)[
        rng.choice(9, size=300_001, p=[0.24] * 4 + [0.01] * 4 + [0.0])].copy()
    seq[rng.random(seq.shape[0]) < 0.001] = ord("N")
    seq = seq.tobytes()
    for q in (1, 7, 31, 32):
        for canonical in (True, False):
            got = bb.encode_qgrams(bb.QGramEncoder(q, canonical), seq)
            np.testing.assert_array_equal(got, orc.encode_qgrams(seq, q, canonical))


def test_dna_case(golden):
    """Fused q-gram insert / lookup == the reference's two-pass composition."""
    meta, arr = golden
    d = meta["dna"]
    enc = bb.QGramEncoder(31, True)
    genome = arr["dna__genome"].tobytes()
    cfg = bb.FilterConfig(kind="blowchoc", k=14, choices=2, size_bits=14 * (d["L"] - 30), seed=1)
    f = bb.Filter.from_config(cfg)
    assert f.insert_qgrams(enc, genome) == d["n_keys"]   # ordered: materialises keys
    assert sha(f.storage.words) == d["words_sha256"]
    reads = arr["dna__reads"].tobytes()
    per_read = [reads[i * 150:(i + 1) * 150] for i in range(len(reads) // 150)]
    hits = [int(f.contains_qgrams(enc, r).sum()) for r in per_read]
    assert hits == d["read_hits"]
    assert [f.count_qgram_hits(enc, r) for r in per_read[:50]] == d["read_hits"][:50]
    # all reads at once, separated so no window spans two reads
    joined = bb.join_records(per_read)
    ans = f.contains_qgrams(enc, joined)
    sl = bb.record_slices(per_read, 31)
    assert [int(ans[a:b].sum()) for a, b in sl] == d["read_hits"]
    assert f.count_qgram_hits(enc, joined) == sum(d["read_hits"])


def test_fused_qgram_insert_single_choice_and_relaxed():
    rng = np.random.default_rng(3)
    genome = np.frombuffer(b"ACGT", dtype=np.uint8)[rng.integers(0, 4, 400_000)].tobytes()
    enc = bb.QGramEncoder(31, True)
    keys = orc.encode_qgrams(genome, 31)
    # c = 1: fused path is bit-identical
    cfg = bb.FilterConfig(kind="blocked", k=12, size_bits=12 * len(keys), seed=2)
    f = bb.Filter.from_config(cfg)
    assert f.insert_qgrams(enc, genome) == keys.shape[0]
    o = orc.make_filter("blocked", k=12, size_bits=12 * len(keys), seed=2)
    o.insert_many(keys)
    np.testing.assert_array_equal(f.storage.words, o.words)
    # c = 2 relaxed: no false negatives for any genome k-mer
    cfg2 = bb.FilterConfig(kind="blowchoc", k=14, choices=2, size_bits=14 * len(keys), seed=2)
    g = bb.Filter.from_config(cfg2, insert_mode="relaxed")
    g.insert_qgrams(enc, genome)
    assert g.contains_qgrams(enc, genome).all()
    assert g.count_qgram_hits(enc, genome) == keys.shape[0]


@pytest.mark.parametrize("seed", [0, 11, 12, 5, 2**40 + 7])
def test_device_key_streams_equal_numpy(seed):
    """even_keys / odd_keys generated on the GPU (PCG64 jump-ahead) are
    bit-identical to the reference's numpy streams, at any offset."""
    for n in (1, 63, 64, 65, 4097, 100_003):
        np.testing.assert_array_equal(bb.even_keys(n, seed, device="cuda").cpu().numpy(),
                                      bb.even_keys(n, seed))
        np.testing.assert_array_equal(bb.odd_keys(n, seed, device="cuda").cpu().numpy(),
                                      bb.odd_keys(n, seed))
    full = bb.even_keys(300_000, seed)
    for off in (1, 77, 4096, 123_456):
        got = bb.even_keys(1000, seed, device="cuda", offset=off).cpu().numpy()
        np.testing.assert_array_equal(got, full[off:off + 1000])


def test_estimate_fpr_device_stream_matches_host():
    cfg = bb.FilterConfig(kind="blowchoc", k=8, n_capacity=100_000, choices=2, seed=3)
    f = bb.Filter.from_config(cfg)
    f.insert_many(bb.even_keys(100_000, 4))
    est = bb.estimate_fpr(f, n_queries=3 * 2**18 + 5, chunk_size=2**18, seed=99)
    host = sum(f.count_hits(bb.odd_keys(min(2**18, 3 * 2**18 + 5 - a), bb.derive_seed(99, i)))
               for i, a in enumerate(range(0, 3 * 2**18 + 5, 2**18)))
    assert est.false_positives == host


def test_partitioned_single_choice_insert_bit_identical(golden, tmp_path):
    """The opt-in region-partitioned insert (BC_PARTITION_MIN_KEYS) gives the
    reference's bit array (run in a subprocess: the knob is read at load)."""
    import subprocess
    import sys

    meta, _ = golden
    case = meta["cfg2_small"]
    script = (
        "import hashlib, numpy as np, torch, paper_2501_18977_b200 as bb\n"
        f"cfg = bb.FilterConfig(kind='blocked', k=12, size_bits=12 * 2**20, seed=1)\n"
        "f = bb.Filter.from_config(cfg)\n"
        f"f.insert_many(torch.from_numpy(bb.even_keys({case['n_insert']}, {case['insert_seed']})).cuda())\n"
        "print(hashlib.sha256(f.storage.words.tobytes()).hexdigest())\n")
    env = dict(os.environ, BC_PARTITION_MIN_KEYS="1")
    out = subprocess.run([sys.executable, "-c", script], env=env, capture_output=True, text=True,
                         cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert out.returncode == 0, out.stderr
    assert out.stdout.strip().splitlines()[-1] == case["words_sha256"]



def _run_with_env(script, **env):
    import subprocess
    import sys

    out = subprocess.run([sys.executable, "-c", script], env=dict(os.environ, **env),
                         capture_output=True, text=True,
                         cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert out.returncode == 0, out.stderr
    return out.stdout.strip().splitlines()[-1]


@pytest.mark.parametrize("persist", ["0", "1"])
def test_l2_window_does_not_change_results(golden, persist):
    """Filters launched with or without the L2-persisting window (BC_L2_PERSIST,
    read at load, hence the subprocess) give the reference's bits and answers;
    bc_l2_release between calls is harmless."""
    meta, _ = golden
    case = meta["cfg2_small"]
    script = (
        "import hashlib, numpy as np, torch, paper_2501_18977_b200 as bb\n"
        "from paper_2501_18977_b200 import _native\n"
        f"cfg = bb.FilterConfig(**{dict(case['config'])!r})\n"
        "f = bb.Filter.from_config(cfg)\n"
        f"keys = bb.even_keys({case['n_insert']}, {case['insert_seed']})\n"
        "f.insert_many(torch.from_numpy(keys).cuda())\n"
        "_native.lib().bc_l2_release()\n"
        f"probes = np.concatenate([keys[:max(1, {case['n_insert']} // 2)], "
        f"bb.odd_keys({case['n_neg']}, {case['neg_seed']})])\n"
        "out = f.contains_many(torch.from_numpy(probes).cuda()).cpu().numpy().astype(np.uint8)\n"
        "print(hashlib.sha256(f.storage.words.tobytes()).hexdigest(), "
        "hashlib.sha256(out.tobytes()).hexdigest())\n")
    words, answers = _run_with_env(script, BC_L2_PERSIST=persist).split()
    assert words == case["words_sha256"]
    assert answers == case["out_sha256"]


def test_unpipelined_relaxed_insert_within_tolerance(golden):
    """BC_RELAXED_PIPE=0 (the plain two-phase tile) meets the same relaxed
    tolerances as the default pipelined kernel."""
    meta, _ = golden
    case = meta["bc3_k12_20k"]
    script = (
        "import numpy as np, torch, paper_2501_18977_b200 as bb\n"
        "from paper_2501_18977_b200.filters import CostModel\n"
        f"cfg = bb.FilterConfig(**{dict(case['config'])!r})\n"
        "f = bb.Filter.from_config(cfg, insert_mode='relaxed')\n"
        f"keys = bb.even_keys({case['n_insert']}, {case['insert_seed']})\n"
        "f.insert_many(keys)\n"
        "assert f.contains_many(keys).all()\n"
        f"print(f.count_hits(bb.odd_keys({case['n_neg']}, {case['neg_seed']})))\n")
    hits = int(_run_with_env(script, BC_RELAXED_PIPE="0"))
    ref = case["hits_neg"]
    assert abs(hits - ref) <= 0.1 * ref + 3 * np.sqrt(2.0 * max(ref, 1)) + 1


@pytest.mark.parametrize("name", ["cfg1", "bc3_k12_20k", "bc2_k6_t4", "bc8_k5"])
def test_ordered_build_in_several_calls(golden, name):
    """Exact-order inserts split over several calls (ragged sizes, the claim
    state carried between launches) give the reference's bit array."""
    meta, _ = golden
    case = meta[name]
    f = bb.Filter.from_config(config_of(case))
    keys, _ = probes_of(case)
    n = keys.shape[0]
    cuts = [0, 1, 257, n // 3, n // 3 + 1, (2 * n) // 3, n]
    for a, b in zip(cuts[:-1], cuts[1:]):
        f.insert_many(keys[a:b])
    assert sha(f.storage.words) == case["words_sha256"]
    assert f.inserted == n


@pytest.mark.parametrize("kind,c,strategy,bb_bits", [
    ("standard", None, "random", 512), ("blocked", 1, "random", 512),
    ("blowchoc", 2, "random", 512), ("blowchoc", 3, "distinct", 512),
    ("blowchoc", 2, "random", 128), ("blocked", 1, "random", 16),
])
def test_extreme_keys(kind, c, strategy, bb_bits):
    """Edge keys (0, 1, 2^32 +- 1, 2^63, 2^64 - 1, all-ones halves) and their
    neighbours inserted and looked up: bits and answers equal the oracle's."""
    edge = [0, 1, 2, 2**32 - 1, 2**32, 2**32 + 1, 2**63 - 1, 2**63, 2**63 + 1,
            2**64 - 2, 2**64 - 1, 0xFFFFFFFF00000000, 0x00000000FFFFFFFF,
            0x5555555555555555, 0xAAAAAAAAAAAAAAAA]
    keys = np.array(edge, dtype=np.uint64)
    kw = dict(kind=kind, k=7, size_bits=4096, seed=99, strategy=strategy,
              block_bits=bb_bits)
    if c is not None:
        kw["choices"] = c
    o = orc.make_filter(kind, k=7, choices=c, strategy=strategy, block_bits=bb_bits,
                        size_bits=4096, seed=99)
    o.insert_many(keys[::2])
    f = bb.Filter.from_config(bb.FilterConfig(**kw))
    f.insert_many(keys[::2])
    np.testing.assert_array_equal(f.storage.words, o.words)
    np.testing.assert_array_equal(f.contains_many(keys), o.contains_many(keys))
    assert f.contains_many(keys[::2]).all()


@pytest.mark.parametrize("one", ["1", "0"])
@pytest.mark.parametrize("slots", ["64", "4096"])
def test_ordered_build_with_hashed_claim_slots(golden, slots, one):
    """Exact-order inserts with the claim tags hashed onto few slots
    (BC_ORDERED_SLOTS, read when the scratch is allocated): spurious
    conflicts only delay commits, the bits stay the reference's.  With 64
    slots the build takes hundreds of rounds, so the one-array kernel's 8-bit
    round tag wraps (the in-kernel clear of the claims).  Both claim-round
    kernels: one array of epoch-tagged claims (default) and two reset-on-win
    arrays (BC_ORDERED_ONE=0)."""
    meta, _ = golden
    case = meta["bc3_k12_20k"]
    script = (
        "import hashlib, numpy as np, paper_2501_18977_b200 as bb\n"
        f"cfg = bb.FilterConfig(**{dict(case['config'])!r})\n"
        "f = bb.Filter.from_config(cfg)\n"
        f"keys = bb.even_keys({case['n_insert']}, {case['insert_seed']})\n"
        "f.insert_many(keys[:7000]); f.insert_many(keys[7000:])\n"
        "print(hashlib.sha256(f.storage.words.tobytes()).hexdigest())\n")
    assert _run_with_env(script, BC_ORDERED_SLOTS=slots, BC_ORDERED_TICKET="0",
                         BC_ORDERED_ONE=one) == case["words_sha256"]


GRID = {"BC_ORDERED_TICKET": "0"}  # exact inserts on the grid-wide claim rounds


@pytest.mark.parametrize("name,env", [("cfg2_small", {"BC_LOOKUP_PIPE": "0"}),
                                      ("bc3_k12_20k", {**GRID, "BC_ORDERED_WINDOW": "0"}),
                                      ("cfg1", {**GRID, "BC_ORDERED_WINDOW": "0"}),
                                      ("bc3_k12_20k", {**GRID, "BC_ORDERED_TILES": "0"}),
                                      ("cfg1", {**GRID, "BC_ORDERED_TILES": "0"}),
                                      ("cfg1", GRID), ("bc3_k12_20k", GRID),
                                      ("cfg1", {**GRID, "BC_ORDERED_ONE": "0"}),
                                      ("bc3_k12_20k", {**GRID, "BC_ORDERED_ONE": "0"}),
                                      ("cfg3_small", {**GRID, "BC_ORDERED_ONE": "0"}),
                                      ("cfg1", {**GRID, "BC_ORDERED_REL_BITS": "10"}),
                                      ("cfg3_small", {**GRID, "BC_ORDERED_REL_BITS": "6"}),
                                      ("bc2_k6_t4", {**GRID, "BC_ORDERED_REL_BITS": "3"}),
                                      ("bc4_k8", GRID), ("cfg3_small", GRID),
                                      ("bc8_k5", GRID), ("bc2_k6_t4", GRID),
                                      ("cfg1", {"BC_TICKET_INFLIGHT_PCT": "3"}),
                                      ("cfg1", {"BC_TICKET_CHUNK": "100000"}),
                                      ("bc3_k12_20k", {"BC_TICKET_CHUNK": "777",
                                                       "BC_TICKET_INFLIGHT_PCT": "1000"}),
                                      ("cfg5_small_k11", {"BC_TICKET_CHUNK": "65536"})])
def test_fallback_kernels_match_reference(golden, name, env):
    """The kernel variants kept behind switches (unpipelined single-choice
    lookups, the grid-wide exact inserts that small filters no longer use,
    the two-array claim rounds, the one-array rounds with a claim range of a
    few keys only (BC_ORDERED_REL_BITS: most keys are out of range of the
    round's base and wait without a claim), fixed-chunk exact inserts, exact
    inserts that commit one thread per key)
    and the ticket exact insert with narrow / wide in-flight windows and
    several ticket sets per call still give the reference's bits and
    answers."""
    meta, _ = golden
    case = meta[name]
    script = (
        "import hashlib, numpy as np, paper_2501_18977_b200 as bb\n"
        f"cfg = bb.FilterConfig(**{dict(case['config'])!r})\n"
        "f = bb.Filter.from_config(cfg)\n"
        f"keys = bb.even_keys({case['n_insert']}, {case['insert_seed']})\n"
        "f.insert_many(keys)\n"
        f"probes = np.concatenate([keys[:max(1, {case['n_insert']} // 2)], "
        f"bb.odd_keys({case['n_neg']}, {case['neg_seed']})])\n"
        "out = f.contains_many(probes).astype(np.uint8)\n"
        "print(hashlib.sha256(f.storage.words.tobytes()).hexdigest(), "
        "hashlib.sha256(out.tobytes()).hexdigest())\n")
    words, answers = _run_with_env(script, **env).split()
    assert words == case["words_sha256"]
    assert answers == case["out_sha256"]


def test_foreign_cuda_arrays_stay_on_device(golden):
    """Keys given as non-torch CUDA arrays (__cuda_array_interface__ or
    DLPack, as CuPy / Numba provide) are used in place and answered on the
    device, like CUDA tensors."""
    meta, _ = golden
    case = meta["cfg1"]
    keys, probes = probes_of(case)
    t_keys = torch.from_numpy(keys).cuda()
    t_probes = torch.from_numpy(probes).cuda()

    class CAI:
        def __init__(self, t):
            self.t = t
            self.__cuda_array_interface__ = t.__cuda_array_interface__

    class DL:
        def __init__(self, t):
            self.t = t

        def __dlpack__(self, stream=None):
            return self.t.__dlpack__()

        def __dlpack_device__(self):
            return self.t.__dlpack_device__()

    for wrap in (CAI, DL):
        f = bb.Filter.from_config(config_of(case))
        f.insert_many(wrap(t_keys))
        assert sha(f.storage.words) == case["words_sha256"]
        out = f.contains_many(wrap(t_probes))
        assert isinstance(out, torch.Tensor) and out.is_cuda
        assert sha(out.cpu().numpy().astype(np.uint8)) == case["out_sha256"]
        assert f.count_hits(wrap(t_probes)) == case["hits_pos"] + case["hits_neg"]


@pytest.mark.parametrize("canonical", [True, False])
def test_qgram_read_matrix_records(canonical):
    """A 2-D reads matrix (fixed-length records, no separators): encode,
    fused insert and fused lookup equal the per-read composition through the
    oracle; no window crosses a row (also with the relaxed insert's slicing,
    whose slices start mid-record)."""
    rng = np.random.default_rng(12)
    reads = rng.choice(np.frombuffer(b"ACGTacgtN", np.uint8), size=(397, 151),
                       p=[0.124] * 8 + [0.008])
    q = 31
    enc = bb.QGramEncoder(q, canonical=canonical)
    want = np.concatenate([orc.encode_qgrams(r.tobytes(), q, canonical) for r in reads])
    got = bb.encode_qgrams(enc, reads)
    np.testing.assert_array_equal(got, want)
    got_t = bb.encode_qgrams(enc, torch.from_numpy(reads).cuda())
    assert got_t.is_cuda
    np.testing.assert_array_equal(got_t.cpu().numpy(), want)
    np.testing.assert_array_equal(bb.encode_qgrams(enc, reads.reshape(-1), record_len=151),
                                  want)

    for kind, c, mode in (("blocked", 1, "ordered"), ("blowchoc", 2, "ordered"),
                          ("blowchoc", 2, "relaxed")):
        cfg = bb.FilterConfig(kind=kind, k=9, choices=c, n_capacity=3000, seed=4)
        f = bb.Filter.from_config(cfg, insert_mode=mode)
        assert f.insert_qgrams(enc, reads) == want.size
        if mode == "ordered":
            o = orc.make_filter(kind, k=9, choices=c, n_capacity=3000, seed=4)
            o.insert_many(want)
            np.testing.assert_array_equal(f.storage.words, o.words)
        assert f.contains_many(want).all()
        probe = rng.choice(np.frombuffer(b"ACGT", np.uint8), size=(50, 151))
        pk = np.concatenate([want[:500]] + [orc.encode_qgrams(r.tobytes(), q, canonical)
                                            for r in probe])
        both = np.concatenate([reads[:5], probe])
        pw = np.concatenate([orc.encode_qgrams(r.tobytes(), q, canonical) for r in both])
        np.testing.assert_array_equal(f.contains_qgrams(enc, both), f.contains_many(pw))
        assert f.count_qgram_hits(enc, both) == int(f.contains_many(pw).sum())
        del pk
    with pytest.raises(ValueError):
        bb.encode_qgrams(enc, reads, record_len=150)


@pytest.mark.parametrize("n", [1, 7, 4097, 131_075, 393_219, 1_048_579, 3_145_733,
                               (1 << 22) + 11, 3 * (1 << 22) + 5])
def test_host_buffers_awkward_lengths(n):
    """Pageable numpy keys and answers of awkward lengths (staged through
    pinned chunks by the parallel host copy) give the device path's bits and
    answers."""
    cfg = bb.FilterConfig(kind="blowchoc", k=9, choices=2, size_bits=10 * max(n, 1000), seed=3)
    keys = bb.even_keys(n, 5)
    probes = np.concatenate([keys[::2], bb.odd_keys(n, 6)])
    f = bb.Filter.from_config(cfg)
    g = bb.Filter.from_config(cfg)
    f.insert_many(keys)                                   # host path
    g.insert_many(torch.from_numpy(keys).cuda())          # device path
    assert torch.equal(f.storage.d_words, g.storage.d_words)
    want = g.contains_many(torch.from_numpy(probes).cuda()).cpu().numpy()
    np.testing.assert_array_equal(f.contains_many(probes), want)
    np.testing.assert_array_equal(f.contains_many(probes[1:]), want[1:])  # unaligned start
    assert f.count_hits(probes) == int(want.sum())


def test_concurrent_host_inserts_into_separate_filters():
    """Several threads insert pageable numpy streams into their own filters at
    once (shared per-device staging and copy pool): each filter equals its
    sequentially built twin."""
    from concurrent.futures import ThreadPoolExecutor

    cfgs = [bb.FilterConfig(kind=kind, k=k, choices=c, size_bits=12 * (1 << 21), seed=s)
            for s, (kind, k, c) in enumerate([("blocked", 12, 1), ("blowchoc", 14, 2),
                                              ("blowchoc", 16, 3), ("standard", 9, None)])]
    streams = [bb.even_keys((1 << 21) + 17 * i, 40 + i) for i in range(len(cfgs))]

    def build(i):
        f = bb.Filter.from_config(cfgs[i])
        f.insert_many(streams[i][: len(streams[i]) // 3])
        f.insert_many(streams[i][len(streams[i]) // 3:])
        return f.storage.d_words.clone()

    with ThreadPoolExecutor(len(cfgs)) as pool:
        got = list(pool.map(build, range(len(cfgs))))
    for i, cfg in enumerate(cfgs):
        g = bb.Filter.from_config(cfg)
        g.insert_many(torch.from_numpy(streams[i]).cuda())
        assert torch.equal(got[i], g.storage.d_words), cfg


def test_concurrent_lookups_from_threads(golden):
    """The reference's query pool (cli.py:133-140) calls contains_many from
    several threads on one filter: same answers as one call."""
    from concurrent.futures import ThreadPoolExecutor

    meta, _ = golden
    case = meta["cfg1"]
    f = bb.Filter.from_config(config_of(case))
    keys, probes = probes_of(case)
    f.insert_many(keys)
    parts = np.array_split(probes, 8)
    with ThreadPoolExecutor(8) as pool:
        got = np.concatenate(list(pool.map(f.contains_many, parts)))
    assert sha(got.astype(np.uint8)) == case["out_sha256"]
    g = bb.Filter.from_config(config_of(case))  # handle created under contention
    g.storage.load_words(f.storage.words)
    with ThreadPoolExecutor(8) as pool:
        counts = list(pool.map(g.count_hits, parts))
    assert sum(counts) == case["hits_pos"] + case["hits_neg"]


@pytest.mark.parametrize("env", [{"BC_TICKET_CHUNK": "1000"}, {"BC_ORDERED_TICKET": "0"},
                                 {"BC_ORDERED_TICKET": "0", "BC_ORDERED_ONE": "0"},
                                 {"BC_ORDERED_TICKET": "0", "BC_ORDERED_REL_BITS": "7"}])
def test_fused_exact_qgram_insert_in_ticket_sets_and_claim_rounds(env):
    """The fused exact-order q-gram insert of a reads matrix (fixed-length
    records) split into many ticket sets (each set's stream resumes mid-record)
    and on the grid-wide claim rounds equals the oracle's stream-order insert
    of encode_qgrams."""
    script = (
        "import numpy as np, paper_2501_18977_b200 as bb\n"
        "from oracle import oracle as orc\n"
        "rng = np.random.default_rng(21)\n"
        "reads = rng.choice(np.frombuffer(b'ACGTacgtN', np.uint8), size=(211, 97),\n"
        "                   p=[0.124] * 8 + [0.008])\n"
        "enc = bb.QGramEncoder(21, canonical=True)\n"
        "want = np.concatenate([orc.encode_qgrams(r.tobytes(), 21, True) for r in reads])\n"
        "f = bb.Filter.from_config(bb.FilterConfig(kind='blowchoc', k=9, choices=3,\n"
        "                                          n_capacity=4000, seed=5))\n"
        "assert f.insert_qgrams(enc, reads) == want.size\n"
        "o = orc.make_filter('blowchoc', k=9, choices=3, n_capacity=4000, seed=5)\n"
        "o.insert_many(want)\n"
        "print(bool(np.array_equal(f.storage.words, o.words)), want.size)\n")
    ok, n = _run_with_env(script, **env).split()
    assert ok == "True" and int(n) > 10000


@pytest.mark.parametrize("env", [{}, {"BC_ORDERED_REL_BITS": "10"}, {"BC_ORDERED_ONE": "0"}])
def test_fused_exact_qgram_insert_across_a_long_invalid_run(env):
    """A sequence with 300,000 non-ACGT bytes in the middle, inserted by the
    fused exact-order claim rounds: the stream cursor crosses the run without
    admitting a key, so the claim base lags far behind the next valid windows
    (out of claim range when the range is narrowed to 2^10); the words equal
    the oracle's stream-order insert of encode_qgrams."""
    script = (
        "import numpy as np, paper_2501_18977_b200 as bb\n"
        "from oracle import oracle as orc\n"
        "rng = np.random.default_rng(5)\n"
        "a = rng.choice(np.frombuffer(b'ACGT', np.uint8), size=40000)\n"
        "b = rng.choice(np.frombuffer(b'ACGT', np.uint8), size=50000)\n"
        "seq = np.concatenate([a, np.full(300000, ord('N'), np.uint8), b]).tobytes()\n"
        "enc = bb.QGramEncoder(25, canonical=True)\n"
        "want = orc.encode_qgrams(seq, 25, True)\n"
        "cfg = dict(kind='blowchoc', k=10, choices=2, n_capacity=want.size, seed=8)\n"
        "f = bb.Filter.from_config(bb.FilterConfig(**cfg))\n"
        "assert f.insert_qgrams(enc, seq) == want.size\n"
        "o = orc.make_filter(**cfg)\n"
        "o.insert_many(want)\n"
        "print(bool(np.array_equal(f.storage.words, o.words)), want.size)\n")
    ok, n = _run_with_env(script, BC_ORDERED_TICKET="0", **env).split()
    assert ok == "True" and int(n) == 40000 - 24 + 50000 - 24


def test_insert_qgram_batches_equals_one_insert_per_batch():
    """insert_qgram_batches (counts read once at the end) against
    insert_qgrams per batch, exact order: same words, same total."""
    rng = np.random.default_rng(17)
    recs = [rng.choice(np.frombuffer(b"ACGTN", np.uint8), size=int(n), p=[0.245] * 4 + [0.02])
            for n in rng.integers(10, 5000, 40)]
    batches = [bb.join_records([r.tobytes() for r in recs[i:i + 7]]) for i in range(0, 40, 7)]
    enc = bb.QGramEncoder(19, canonical=True)
    cfg = bb.FilterConfig(kind="blowchoc", k=8, choices=2, n_capacity=120_000, seed=3)
    a, b = bb.Filter.from_config(cfg), bb.Filter.from_config(cfg)
    total = sum(a.insert_qgrams(enc, x) for x in batches)
    assert b.insert_qgram_batches(enc, iter(batches)) == total == a.inserted == b.inserted
    np.testing.assert_array_equal(a.storage.words, b.storage.words)
    assert bb.Filter.from_config(cfg).insert_qgram_batches(enc, []) == 0
