"""Pin the CPU oracle to the reference: every golden vector must be reproduced
exactly before the oracle is trusted as the checker for the CUDA path."""

import hashlib
import math

import numpy as np
import pytest

from oracle import oracle as orc


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _oracle_filter(meta_case):
    cfg = dict(meta_case["config"])
    cost = cfg.pop("cost", None)
    code, param = 0, None
    if cost is not None:
        code, param = ("exp", "mix", "la").index(cost["kind"]), cost["param"]
    return orc.make_filter(cost_code=code, cost_param=param, **cfg)


def test_hash_kats(golden):
    _, arr = golden
    L = orc.lib()
    for a, b, x, h in zip(arr["hash__a"].tolist(), arr["hash__b"].tolist(),
                          arr["hash__x"].tolist(), arr["hash__h"].tolist()):
        mode, s = orc.hash_branch(b)
        assert L.orc_hash(a, x, b, mode, s) == h
        assert orc.hash_value(a, x, b) == h


def test_reference_hash_kats_restated():
    # test_hashing.py:48-57
    assert orc.hash_value(3, 7, 5) == 1
    assert orc.hash_value(1, 2**63, 512) == 256
    assert orc.hash_value(1, 5, 10) == 5


def test_cost_values_bit_exact(golden):
    meta, arr = golden
    L = orc.lib()
    for i, spec in enumerate(meta["costs"]):
        tab = arr[f"cost__{i}"]
        code = ("exp", "mix", "la").index(spec["kind"])
        for j in range(spec["B"] + 1):
            for a in range(spec["k"] + 1):
                got = L.orc_cost_value(j, a, spec["k"], code, spec["param"], spec["B"])
                assert got == tab[j, a] or (math.isnan(got) and math.isnan(tab[j, a]))


def test_qgram_kats(golden):
    meta, arr = golden
    for kat in meta["qgram_kats"]:
        got = orc.encode_qgrams(kat["seq"], kat["q"], kat["canonical"])
        assert got.tolist() == [int(v) for v in kat["keys"]]
    for case in meta["qgrams"]:
        i = case["idx"]
        seq = arr[f"qg__{i}__seq"].tobytes()
        got = orc.encode_qgrams(seq, case["q"], case["canonical"])
        np.testing.assert_array_equal(got, arr[f"qg__{i}__keys"])


@pytest.mark.parametrize("name", [
    "std_k7", "blk_rand_k7", "blk_dist_k7", "bc2_rand_k7", "bc2_dist_k7", "bc3_rand_k7",
    "bc2_rand_b16", "bc2_dist_b16", "bc3_k12_20k", "bc2_k6_t4", "blk_k9_t8", "bc3_dist_k10",
    "bc4_k8", "bc8_k5", "bc2_mix", "bc3_la", "bc2_exp13", "bc2_b64", "bc2_b128", "bc2_b1024",
    "blk_b8", "bc3_b32_dist", "bc2_dist_k40", "std_k10_odd", "bc2_overfill",
    "cfg1", "cfg2_small", "cfg3_small", "cfg5_small_k11",
])
def test_filter_cases(golden, name):
    meta, arr = golden
    case = meta[name]
    f = _oracle_filter(case)
    assert f.num_blocks == case["num_blocks"]
    assert str(f.shard_a) == case["shard_a"]
    assert [str(v) for v in f.block_a.tolist()] == case["block_a"]
    assert [str(v) for v in f.bit_a.tolist()] == case["bit_a"]
    keys = orc.even_keys(case["n_insert"], case["insert_seed"])
    f.insert_many(keys)
    assert sha(f.words) == case["words_sha256"]
    if f"{name}__words" in arr:
        np.testing.assert_array_equal(f.words, arr[f"{name}__words"])
    pos = keys[: max(1, case["n_insert"] // 2)]
    probes = np.concatenate([pos, orc.odd_keys(case["n_neg"], case["neg_seed"])])
    out = f.contains_many(probes).astype(np.uint8)
    assert sha(out) == case["out_sha256"]
    assert int(out[: pos.shape[0]].sum()) == case["hits_pos"] == pos.shape[0]
    if f.kind != "standard":
        hist = f.block_histogram().astype(np.int64)
        assert sha(hist) == case["hist_sha256"]
        # threaded lookup == sequential lookup
        out_mt = f.contains_many(probes, threads=4).astype(np.uint8)
        np.testing.assert_array_equal(out_mt, out)


def test_threaded_c1_insert_is_bit_identical(golden):
    meta, _ = golden
    case = meta["cfg2_small"]
    f = _oracle_filter(case)
    f.insert_many_mt(orc.even_keys(case["n_insert"], case["insert_seed"]), threads=4)
    assert sha(f.words) == case["words_sha256"]


def test_dna_case(golden):
    meta, arr = golden
    d = meta["dna"]
    genome = arr["dna__genome"].tobytes()
    keys = orc.encode_qgrams(genome, 31, True)
    assert keys.shape[0] == d["n_keys"] and sha(keys) == d["keys_sha256"]
    f = orc.make_filter("blowchoc", k=14, choices=2, size_bits=14 * (d["L"] - 30), seed=1)
    assert f.num_blocks == d["num_blocks"]
    f.insert_many(keys)
    assert sha(f.words) == d["words_sha256"]
    reads = arr["dna__reads"].tobytes()
    hits = [int(f.contains_many(orc.encode_qgrams(reads[i * 150:(i + 1) * 150], 31)).sum())
            for i in range(len(reads) // 150)]
    assert hits == d["read_hits"]
