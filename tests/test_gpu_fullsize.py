"""Full-size parity of BASELINE configs 3, 4 and 5 against the reference.

The exact-order (bit-exact, the ``Filter`` default) GPU builds of the full
workloads are compared with digests the reference itself produced on the same
key streams (tests/golden/make_fullsize.py, numba, in the build container):

* cfg3: 2^28 keys ``even_keys(2^28, 11)`` into the 512 MiB c = 3 filter;
* cfg4: the canonical 31-mers of a 1.2e9-bp genome (``synthetic_genome``:
  base i = "ACGT"[w_i >> 62] of the PCG64 word stream of seed 4) into the
  2 GB c = 2 filter, through the fused sequence path (no key array);
* cfg5: 1.2 x 2^32 keys ``even_keys(., 11)`` into the 8 GiB c = 2 filter
  (k = 11), also pinned at the design load (2^32 keys).

Each fixture also pins lookups on the final bit array: the false-positive
count over ``odd_keys(2^24, 12)`` and the answers to its first 2^20 keys.

The relaxed (atomic) builds are then checked against these exact builds with
the tolerances of SURVEY §8(a), written in the tests: zero false negatives,
|log2 FPR_relaxed - log2 FPR_exact| <= 0.1 + 3 sigma over >= 2^24
device-generated negatives, mean block load within 1 bit, load variance
within 15%, unbinned load-histogram total variation <= 0.05.
"""

import hashlib
import json
import math
import os

import numpy as np
import pytest
import torch

import paper_2501_18977_b200 as bb
from paper_2501_18977_b200 import _native
from paper_2501_18977_b200.analysis import histogram_distance

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
N_NEG = 1 << 24


def fixture(cfgno):
    path = os.path.join(GOLDEN, f"fullsize_cfg{cfgno}.json")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated (tests/golden/make_fullsize.py)")
    with open(path) as fh:
        return json.load(fh)


def sha_device(t: torch.Tensor) -> str:
    """sha256 of a device tensor's bytes, copied to the host in 1 GiB pieces."""
    h = hashlib.sha256()
    b = t.view(torch.uint8)
    step = 1 << 30
    for a in range(0, b.numel(), step):
        h.update(b[a:a + step].cpu().numpy().tobytes())
    return h.hexdigest()


def lookup_pins(f, fx):
    neg = bb.odd_keys(N_NEG, 12, device="cuda")
    assert f.count_hits(neg) == fx["neg_keys"]["false_positives"]
    ans = f.contains_many(neg[: 1 << 20]).cpu().numpy().astype(np.uint8)
    assert hashlib.sha256(ans.tobytes()).hexdigest() == \
        fx["neg_keys"]["answers_sha256_first_2p20"]
    return neg


def relaxed_within_tolerance(relaxed, fp_exact, h_exact, neg, pos_sample):
    """SURVEY §8(a) relaxed-mode tolerances against the exact build."""
    assert relaxed.count_hits(pos_sample) == pos_sample.numel(), "relaxed: false negatives"
    fp_r = relaxed.count_hits(neg)
    sigma = math.sqrt(1 / fp_exact + 1 / fp_r) / math.log(2)  # stderr of the log2 ratio
    assert abs(math.log2(fp_r / fp_exact)) <= 0.1 + 3 * sigma, (fp_exact, fp_r)
    h_r = bb.block_load_histogram(relaxed)
    assert abs(h_r.mean_load - h_exact.mean_load) <= 1.0, (h_r.mean_load, h_exact.mean_load)
    assert abs(h_r.variance / h_exact.variance - 1) <= 0.15, (h_r.variance, h_exact.variance)
    tv = histogram_distance(h_r.counts, h_exact.counts)
    assert tv <= 0.05, tv


def test_cfg3_full_size_exact_order_equals_reference():
    fx = fixture(3)
    cfg = bb.FilterConfig(**fx["filter"])
    keys = bb.even_keys(fx["n_keys"], 11, device="cuda")
    f = bb.Filter.from_config(cfg)  # insert_mode "ordered": the reference's stream order
    f.insert_many(keys)
    assert sha_device(f.storage.d_words) == fx["words_sha256"]
    neg = lookup_pins(f, fx)
    # relaxed build of the same stream within the stated tolerance
    fp_e, h_e = fx["neg_keys"]["false_positives"], bb.block_load_histogram(f)
    assert h_e.total_set_bits == fx["set_bits"]
    del f
    r = bb.Filter.from_config(cfg, insert_mode="relaxed")
    r.insert_many(keys)
    relaxed_within_tolerance(r, fp_e, h_e, neg, keys[::61])


def test_cfg4_full_genome_fused_exact_order_equals_reference():
    """Config 4: the fused exact-order q-gram insert (keys encoded inside the
    claim-round kernel from the sequence, one cooperative launch per 2^30
    windows, no key array) equals the reference's
    insert_many(encode_qgrams(genome)) bit for bit."""
    fx = fixture(4)
    g = fx["genome"]
    genome = bb.synthetic_genome(g["length"], g["seed"], device="cuda")
    enc = bb.QGramEncoder(g["q"], g["canonical"])
    cfg = bb.FilterConfig(**fx["filter"])
    f = bb.Filter.from_config(cfg)
    l0 = _native.launch_count()
    assert f.insert_qgrams(enc, genome) == fx["n_keys"]
    torch.cuda.synchronize()
    # fused: the claim-round kernel alone (no encode / count / scan launches)
    assert _native.launch_count() - l0 == (fx["n_keys"] + (1 << 30) - 1) >> 30
    assert sha_device(f.storage.d_words) == fx["words_sha256"]
    neg = lookup_pins(f, fx)
    fp_e, h_e = fx["neg_keys"]["false_positives"], bb.block_load_histogram(f)
    del f
    r = bb.Filter.from_config(cfg, insert_mode="relaxed")
    r.insert_qgrams(enc, genome)
    assert r.count_qgram_hits(enc, genome[: 1 << 24]) == (1 << 24) - g["q"] + 1
    relaxed_within_tolerance(r, fp_e, h_e, neg, bb.encode_qgrams(enc, genome[-(1 << 22):]))


def test_cfg5_full_size_exact_order_equals_reference():
    fx = fixture(5)
    cfg = bb.FilterConfig(**fx["filter"])
    n = fx["n_keys"]
    keys = bb.even_keys(n, 11, device="cuda")
    f = bb.Filter.from_config(cfg)
    mark = int(next(iter(fx["marks"])))
    f.insert_many(keys[:mark])
    assert sha_device(f.storage.d_words) == fx["marks"][str(mark)]
    f.insert_many(keys[mark:])
    assert sha_device(f.storage.d_words) == fx["words_sha256"]
    neg = lookup_pins(f, fx)
    fp_e, h_e = fx["neg_keys"]["false_positives"], bb.block_load_histogram(f)
    del f
    torch.cuda.empty_cache()
    r = bb.Filter.from_config(cfg, insert_mode="relaxed")
    r.insert_many(keys)
    relaxed_within_tolerance(r, fp_e, h_e, neg, keys[::997])


def test_cfg1_relaxed_vs_exact_2p24_negatives(golden):
    """Config 1 at full size: relaxed vs exact with 2^24 negatives and the
    unbinned histogram distance (M = 2^15 blocks)."""
    meta, _ = golden
    case = meta["cfg1"]
    cfg = bb.FilterConfig(**case["config"])
    keys = torch.from_numpy(bb.even_keys(case["n_insert"], case["insert_seed"])).cuda()
    exact = bb.Filter.from_config(cfg)
    exact.insert_many(keys)
    assert hashlib.sha256(exact.storage.words.tobytes()).hexdigest() == case["words_sha256"]
    neg = bb.odd_keys(N_NEG, 12, device="cuda")
    fp_e, h_e = exact.count_hits(neg), bb.block_load_histogram(exact)
    r = bb.Filter.from_config(cfg, insert_mode="relaxed")
    r.insert_many(keys)
    relaxed_within_tolerance(r, fp_e, h_e, neg, keys)
