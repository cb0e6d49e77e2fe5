"""Host-side logic (no GPU): configuration, sizing, cost models, hash
parameter derivation against the reference's golden vectors, and the C ABI
library's exports."""

import ctypes
import math
import os
import re

import numpy as np
import pytest

import paper_2501_18977_b200 as bb
from paper_2501_18977_b200 import _native
from paper_2501_18977_b200.filters import cost_table

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# -- sizing / config (reference test_filters.py:25-41, 109-147) ----------------------

def test_size_for_examples():
    assert bb.size_for(10**6, 10) == (14_427_136, 28_178)
    assert bb.size_for(512, 1) == (1024, 2)
    assert bb.size_for(2000, 1, shards=4)[1] == 8
    with pytest.raises(bb.ConfigError):
        bb.size_for(0, 10)
    with pytest.raises(bb.ConfigError):
        bb.size_for(10, 0)


def test_config_rejects_bad_combinations():
    bad = [dict(kind="standard", k=10, n_capacity=10, strategy="distinct"),
           dict(kind="blowchoc", k=600, n_capacity=10),
           dict(kind="blowchoc", k=4, n_capacity=10, choices=9),
           dict(kind="blocked", k=4, n_capacity=10, choices=2),
           dict(kind="standard", k=4, n_capacity=10, shards=2),
           dict(kind="blocked", k=4, n_capacity=10, size_bits=4096),
           dict(kind="blocked", k=4),
           dict(kind="blocked", k=4, n_capacity=10, block_bits=48),
           dict(kind="weird", k=4, n_capacity=10)]
    for kw in bad:
        with pytest.raises(bb.ConfigError):
            bb.FilterConfig(**kw).validated()


def test_config_defaults():
    cfg = bb.FilterConfig(kind="blowchoc", k=9, n_capacity=10).validated()
    assert cfg.choices == 2 and cfg.cost == bb.CostModel("exp", bb.GOLDEN_BETA, 9)
    assert bb.FilterConfig(kind="blocked", k=9, n_capacity=10).validated().choices == 1
    assert bb.FilterConfig(kind="standard", k=9, n_capacity=10).validated().choices == 0
    m, blocks = bb.FilterConfig(kind="blocked", k=4, size_bits=10_000).validated().sizing()
    assert (blocks, m) == (20, 10_240)


def test_baseline_geometry():
    """SURVEY §8 geometry table for the five BASELINE configs."""
    cases = [(dict(kind="blowchoc", k=14, choices=2, size_bits=16 * 2**20), 32_768, 1),
             (dict(kind="blocked", k=12, size_bits=12 * 2**26), 1_572_864, 2),
             (dict(kind="blowchoc", k=16, choices=3, size_bits=16 * 2**28), 8_388_608, 1),
             (dict(kind="blowchoc", k=14, choices=2, size_bits=14 * (1_200_000_000 - 30)),
              32_812_500, 2),
             (dict(kind="blowchoc", k=11, choices=2, size_bits=2**36), 134_217_728, 1)]
    for kw, blocks, mode in cases:
        _, nb = bb.FilterConfig(**kw).validated().sizing()
        assert nb == blocks
        assert bb.hash_branch(nb)[0] == mode


# -- cost models (reference test_filters.py:46-80) -------------------------------------

def test_cost_anchors():
    assert bb.cost_exp(128, 0, 7, bb.GOLDEN_BETA) == pytest.approx(bb.GOLDEN_BETA)
    assert bb.cost_exp(0, 0, 7, bb.GOLDEN_BETA) == 1.0
    assert bb.cost_mix(128, 3, 7, 1.0) == 7 * 0.5**7 + 3 == 3.0546875
    assert bb.cost_la(200, 2, 7, 3.5) == pytest.approx(7 * (224.5 / 256) ** 7 + 2)
    for j in range(0, 513, 64):
        for a in (0, 2, 7):
            assert bb.cost_la(j, a, 7, 0.0) == bb.cost_mix(j, a, 7, 1.0)
    with pytest.raises(bb.ConfigError):
        bb.CostModel(kind="exp", param=0.0, k=4)
    with pytest.raises(bb.ConfigError):
        bb.CostModel(kind="mix", param=-1.0, k=4)


def test_cost_table_matches_reference_kernel_formula(golden):
    """The table handed to the C ABI equals the reference's float64 costs."""
    meta, arr = golden
    for i, spec in enumerate(meta["costs"]):
        tab = cost_table(spec["kind"], spec["param"], spec["k"], spec["B"])
        np.testing.assert_array_equal(tab, arr[f"cost__{i}"])


def test_rank_table_order_preserving(golden):
    """Dense ranks (what the kernels compare) preserve every < and == of the
    float64 costs, so the argmin with strict < is unchanged."""
    meta, arr = golden
    for i in range(len(meta["costs"])):
        tab = arr[f"cost__{i}"].ravel()
        uniq = np.unique(tab)
        rank = np.searchsorted(uniq, tab)
        idx = np.random.default_rng(i).integers(0, tab.shape[0], size=(20_000, 2))
        a, b = tab[idx[:, 0]], tab[idx[:, 1]]
        ra, rb = rank[idx[:, 0]], rank[idx[:, 1]]
        assert np.array_equal(a < b, ra < rb) and np.array_equal(a == b, ra == rb)


def test_overload_fpr():
    assert bb.overload_fpr(1.0, 10) == pytest.approx(2.0**-10)
    assert bb.overload_fpr(0.0, 10) == 0.0


# -- hashing (reference test_hashing.py) ------------------------------------------------

def test_hash_kats(golden):
    _, arr = golden
    for a, b, x, h in zip(arr["hash__a"].tolist(), arr["hash__b"].tolist(),
                          arr["hash__x"].tolist(), arr["hash__h"].tolist()):
        assert bb.eval_hash(bb.HashSpec(a=a, b=b), x) == h


def test_make_hash_invariants():
    for seed in range(20):
        h = bb.make_hash(bb.SplitMix64(seed), 512)
        assert h.a % 2 == 1 and h.a >= 2**63
    assert math.gcd(bb.make_hash(bb.SplitMix64(7), 6).a, 6) == 1
    with pytest.raises(ValueError):
        bb.make_hash(bb.SplitMix64(1), 0)


def test_adjust_distinct_kats(golden):
    meta, _ = golden
    assert bb.adjust_distinct([5, 5, 4]) == [4, 5, 6]
    assert bb.adjust_distinct([0, 0, 0]) == [0, 1, 2]
    for case in meta["distinct"]:
        assert bb.adjust_distinct(case["raws"]) == case["out"]


def test_parameter_derivation_matches_reference(golden):
    """Same seed -> same h0 / block / bit multipliers as the reference."""
    meta, _ = golden
    for name, case in meta.items():
        if not isinstance(case, dict) or "config" not in case:
            continue
        cfg = dict(case["config"])
        if isinstance(cfg.get("cost"), dict):
            c = cfg["cost"]
            cfg["cost"] = bb.CostModel(c["kind"], c["param"], c["k"])
        v = bb.FilterConfig(**cfg).validated()
        _, nb = v.sizing()
        assert nb == case["num_blocks"], name
        rng = bb.SplitMix64(v.seed)
        assert str(bb.make_hash(rng, v.shards).a) == case["shard_a"], name
        if v.kind == "standard":
            bits = [bb.make_hash(rng, nb * v.block_bits).a for _ in range(v.k)]
        else:
            blocks = [bb.make_hash(rng, nb // v.shards).a for _ in range(v.choices)]
            assert [str(a) for a in blocks] == case["block_a"], name
            bits = [s.a for s in bb.BitSelector.draw(rng, v.strategy, v.k, v.block_bits).specs]
        assert [str(a) for a in bits] == case["bit_a"], name


# -- the C ABI library ---------------------------------------------------------------------

def _header_symbols():
    with open(os.path.join(ROOT, "include", "bbchoc.h")) as fh:
        text = fh.read()
    return set(re.findall(r"^\s*(?:[\w\s\*]+?)\b(bc_\w+)\s*\(", text, flags=re.M))


def test_library_exports_every_declared_symbol():
    L = _native.lib()
    declared = _header_symbols()
    assert declared == set(_native.EXPORTS)
    for name in declared:
        assert hasattr(L, name), name
    assert b"sm_100a" in L.bc_version()


def test_abi_argument_errors_without_gpu():
    L = _native.lib()
    assert L.bc_insert(None, None, None, 0, 0, None) == _native.BC_EINVAL
    assert L.bc_contains(None, None, None, 0, None, None, None) == _native.BC_EINVAL
    assert b"null filter" in L.bc_last_error()
    assert L.bc_eval_hash(3, 0, None, 0, None, None) == _native.BC_EINVAL
    assert L.bc_encode_qgrams(None, 10, 33, 1, 0, None, None, None) == _native.BC_EINVAL
    assert L.bc_block_histogram(None, 1, 48, None, None) == _native.BC_EINVAL
    d = _native.BcFilterDesc()
    d.kind, d.k, d.choices, d.block_bits, d.num_blocks, d.shards = 2, 4, 9, 512, 8, 1
    arr = (ctypes.c_uint64 * 4)(3, 5, 7, 9)
    d.bit_a = arr
    d.bit_b = arr
    h = ctypes.c_void_p()
    assert L.bc_filter_create(ctypes.byref(d), ctypes.byref(h)) == _native.BC_EINVAL
    assert b"choices" in L.bc_last_error()
    # bit ranges must match the layout: random -> B (here 3 != 512)
    d.choices = 2
    assert L.bc_filter_create(ctypes.byref(d), ctypes.byref(h)) == _native.BC_EINVAL
    assert b"bit range 0" in L.bc_last_error()
    d.kind, d.choices, d.block_bits = 1, 1, 8
    assert L.bc_filter_create(ctypes.byref(d), ctypes.byref(h)) == _native.BC_EINVAL


def test_partition_by_shard_is_stable():
    from paper_2501_18977_b200.sharding import partition_by_shard

    keys = np.arange(20, dtype=np.uint64)
    shard = np.array([i % 3 for i in range(20)], dtype=np.uint64)
    parts = partition_by_shard(keys, shard, 3)
    assert [p.tolist() for p in parts] == [list(range(s, 20, 3)) for s in range(3)]


def test_config_validation_matches_reference_fixture():
    """FilterConfig.validated / sizing against the reference's own outcomes on
    1500 seeded parameter sets (tests/golden/config_cases.json, written by
    make_golden.py): the same error class and message, or the same
    normalised choices, seed and sizing."""
    import json
    import os

    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                        "config_cases.json")
    with open(path) as fh:
        cases = json.load(fh)
    assert len(cases) == 1500
    for case in cases:
        want = case["result"]
        try:
            c = bb.FilterConfig(**case["config"]).validated()
            got = {"ok": True, "choices": c.choices, "seed": c.seed, "sizing": list(c.sizing())}
        except Exception as exc:  # noqa: BLE001
            got = {"ok": False, "error": type(exc).__name__, "message": str(exc)}
        assert got == want, case["config"]


def test_hash_derivation_matches_reference_fixture():
    """Shard, block and bit multipliers/ranges derived from the seed equal the
    reference's for 300 seeded configurations (tests/golden/spec_cases.json,
    written by make_golden.py from the reference)."""
    import json
    import os

    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "spec_cases.json")
    with open(path) as fh:
        cases = json.load(fh)
    assert len(cases) == 300
    for case in cases:
        f = bb.Filter.from_config(bb.FilterConfig(**case["config"]))
        assert [f.shard_spec.a, f.shard_spec.b] == case["shard"], case["config"]
        assert [[h.a, h.b] for h in f.block_specs] == case["blocks"], case["config"]
        assert [[h.a, h.b] for h in f.bit_specs] == case["bits"], case["config"]
