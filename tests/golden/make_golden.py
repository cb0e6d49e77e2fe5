"""Generate the golden vectors that pin the oracle (and the CUDA path) to the
reference implementation.

Runs ONLY in the build container, where the reference is importable from
/root/reference/pkg/src (numba JIT).  Its outputs are committed under
tests/golden/ and are what the tests read; nothing at test time touches
/root/reference.

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

Every case drives the reference through its public API
(Filter.from_config / insert_many / contains_many / storage.words,
encode_qgrams, eval_hash, cost_*), i.e. exactly the calls the drop-in
replaces.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, REF)

from blowchoc import (  # noqa: E402
    CostModel, Filter, FilterConfig, GOLDEN_BETA, HashSpec, QGramEncoder,
    block_load_histogram, cost_exp, cost_la, cost_mix, encode_qgrams, eval_hash,
    even_keys, odd_keys,
)
from blowchoc.hashing import adjust_distinct  # noqa: E402


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# (name, FilterConfig kwargs, n_insert, insert seed, n_probe_neg, neg seed, store_words)
FILTER_CASES = [
    # the eight variants of the reference's batch==scalar test (test_kernels.py:9-36)
    ("std_k7", dict(kind="standard", k=7, n_capacity=400, seed=31), 400, 37, 400, 47, True),
    ("blk_rand_k7", dict(kind="blocked", k=7, n_capacity=400, seed=31), 400, 37, 400, 47, True),
    ("blk_dist_k7", dict(kind="blocked", k=7, n_capacity=400, strategy="distinct", seed=31),
     400, 37, 400, 47, True),
    ("bc2_rand_k7", dict(kind="blowchoc", k=7, n_capacity=400, choices=2, seed=31),
     400, 37, 400, 47, True),
    ("bc2_dist_k7", dict(kind="blowchoc", k=7, n_capacity=400, choices=2, strategy="distinct",
                         seed=31), 400, 37, 400, 47, True),
    ("bc3_rand_k7", dict(kind="blowchoc", k=7, n_capacity=400, choices=3, seed=31),
     400, 37, 400, 47, True),
    ("bc2_rand_b16", dict(kind="blowchoc", k=2, n_capacity=400, choices=2, block_bits=16,
                          seed=31), 400, 37, 400, 47, True),
    ("bc2_dist_b16", dict(kind="blowchoc", k=2, n_capacity=400, choices=2, block_bits=16,
                          strategy="distinct", seed=31), 400, 37, 400, 47, True),
    # test_kernels.py:51-59 and :62-73
    ("bc3_k12_20k", dict(kind="blowchoc", k=12, n_capacity=20_000, choices=3, seed=53),
     20_000, 59, 20_000, 60, True),
    ("bc2_k6_t4", dict(kind="blowchoc", k=6, n_capacity=5000, choices=2, shards=4, seed=61),
     5000, 67, 2000, 71, True),
    # wider coverage: other widths, choice counts, cost models, shards
    ("blk_k9_t8", dict(kind="blocked", k=9, n_capacity=30_000, shards=8, seed=5),
     30_000, 6, 30_000, 7, True),
    ("bc3_dist_k10", dict(kind="blowchoc", k=10, n_capacity=8000, choices=3,
                          strategy="distinct", seed=9), 8000, 10, 8000, 11, True),
    ("bc4_k8", dict(kind="blowchoc", k=8, n_capacity=8000, choices=4, seed=12),
     9000, 13, 8000, 14, True),
    ("bc8_k5", dict(kind="blowchoc", k=5, n_capacity=4000, choices=8, seed=15),
     5000, 16, 4000, 17, True),
    ("bc2_mix", dict(kind="blowchoc", k=9, n_capacity=8000, choices=2,
                     cost=CostModel("mix", 1.0, 9), seed=18), 9000, 19, 8000, 20, True),
    ("bc3_la", dict(kind="blowchoc", k=7, n_capacity=8000, choices=3,
                    cost=CostModel("la", 3.5, 7), seed=21), 9000, 22, 8000, 23, True),
    ("bc2_exp13", dict(kind="blowchoc", k=6, n_capacity=6000, choices=2,
                       cost=CostModel("exp", 1.3, 6), seed=24), 7000, 25, 6000, 26, True),
    ("bc2_b64", dict(kind="blowchoc", k=4, n_capacity=3000, choices=2, block_bits=64,
                     seed=27), 3000, 28, 3000, 29, True),
    ("bc2_b128", dict(kind="blowchoc", k=5, n_capacity=3000, choices=2, block_bits=128,
                      seed=30), 3000, 31, 3000, 32, True),
    ("bc2_b1024", dict(kind="blowchoc", k=12, n_capacity=3000, choices=2, block_bits=1024,
                       seed=33), 3000, 34, 3000, 35, True),
    ("blk_b8", dict(kind="blocked", k=2, n_capacity=300, block_bits=8, seed=36),
     300, 37, 300, 38, True),
    ("bc3_b32_dist", dict(kind="blowchoc", k=3, n_capacity=500, choices=3, block_bits=32,
                          strategy="distinct", seed=39), 500, 40, 500, 41, True),
    ("bc2_dist_k40", dict(kind="blowchoc", k=40, n_capacity=2000, choices=2,
                          strategy="distinct", seed=42), 2000, 43, 2000, 44, True),
    ("std_k10_odd", dict(kind="standard", k=10, size_bits=512 * 777, seed=45),
     20_000, 46, 20_000, 47, True),
    ("bc2_overfill", dict(kind="blowchoc", k=8, n_capacity=3000, choices=2, seed=48),
     9000, 49, 5000, 50, True),
    # BASELINE configs at full (cfg1) or reduced size; words pinned by digest
    ("cfg1", dict(kind="blowchoc", k=14, choices=2, size_bits=16 * 2**20, seed=1),
     2**20, 11, 2**20, 12, False),
    ("cfg2_small", dict(kind="blocked", k=12, size_bits=12 * 2**20, seed=1),
     2**20, 11, 2**20, 12, False),
    ("cfg3_small", dict(kind="blowchoc", k=16, choices=3, size_bits=16 * 2**18, seed=1),
     2**18, 11, 2**18, 12, False),
    ("cfg5_small_k11", dict(kind="blowchoc", k=11, choices=2, size_bits=16 * 2**18, seed=1),
     2**18 + 2**18 // 5, 11, 2**18, 12, False),
]


def filter_cases(store: dict, meta: dict) -> None:
    for name, kw, n_ins, s_ins, n_neg, s_neg, store_words in FILTER_CASES:
        cfg = FilterConfig(**kw)
        f = Filter.from_config(cfg)
        keys = even_keys(n_ins, s_ins)
        f.insert_many(keys)
        pos = keys[: max(1, n_ins // 2)]
        neg = odd_keys(n_neg, s_neg)
        probes = np.concatenate([pos, neg])
        out = f.contains_many(probes).astype(np.uint8)
        hist = block_load_histogram(f)
        v = cfg.validated()
        meta[name] = dict(
            config={k_: (val if not isinstance(val, CostModel) else
                         dict(kind=val.kind, param=val.param, k=val.k))
                    for k_, val in kw.items()},
            n_insert=n_ins, insert_seed=s_ins, n_neg=n_neg, neg_seed=s_neg,
            num_blocks=f.num_blocks, choices=v.choices,
            shard_a=str(f.shard_spec.a),
            block_a=[str(h.a) for h in f.block_specs],
            bit_a=[str(s.a) for s in f.bit_specs],
            bit_b=[s.b for s in f.bit_specs],
            words_sha256=sha(f.storage.words),
            out_sha256=sha(out), hits_pos=int(out[: pos.shape[0]].sum()),
            hits_neg=int(out[pos.shape[0]:].sum()),
            hist_sha256=sha(hist.counts.astype(np.int64)),
            mean_load=hist.mean_load, variance=hist.variance,
        )
        if store_words:
            store[f"{name}__words"] = f.storage.words.copy()
            store[f"{name}__out"] = np.packbits(out)
        print(f"{name}: blocks={f.num_blocks} hits_neg={meta[name]['hits_neg']}", flush=True)


def hash_kats(store: dict) -> None:
    rng = np.random.default_rng(2024)
    a_list, b_list, x_list, h_list = [], [], [], []
    bs = ([1, 3, 5, 7, 511, 513, 1_572_864, 32_812_500, 39450, 1000, 6, 10, 2**20 - 3] +
          [2**e for e in range(0, 40)] +
          [int(v) for v in rng.integers(1, 2**40, 60)] +
          [int(v) * 2 for v in rng.integers(1, 2**30, 40)] +
          [512 - i for i in range(64)])
    for b in bs:
        for _ in range(16):
            a = int(rng.integers(0, 2**63, dtype=np.uint64)) * 2 + 1
            x = int(rng.integers(0, 2**64, dtype=np.uint64))
            a_list.append(a)
            b_list.append(b)
            x_list.append(x)
            h_list.append(eval_hash(HashSpec(a=a, b=b), x))
    # edge keys
    for b in (3, 512, 1_572_864, 32_812_500):
        for x in (0, 1, 2**63, 2**64 - 1, 2**64 - 2, 2**32, 2**32 - 1):
            a = 2**64 - 1
            a_list.append(a)
            b_list.append(b)
            x_list.append(x)
            h_list.append(eval_hash(HashSpec(a=a, b=b), x))
    store["hash__a"] = np.array(a_list, dtype=np.uint64)
    store["hash__b"] = np.array(b_list, dtype=np.uint64)
    store["hash__x"] = np.array(x_list, dtype=np.uint64)
    store["hash__h"] = np.array(h_list, dtype=np.uint64)


def distinct_kats(meta: dict) -> None:
    rng = np.random.default_rng(77)
    cases = []
    for B in (8, 16, 32, 512):
        for _ in range(40):
            k = int(rng.integers(1, min(B, 24) + 1))
            raws = [int(rng.integers(0, B - i)) for i in range(k)]
            cases.append(dict(B=B, raws=raws, out=adjust_distinct(raws)))
    meta["distinct"] = cases


def cost_tables(store: dict, meta: dict) -> None:
    specs = [("exp", GOLDEN_BETA, 14, 512), ("exp", GOLDEN_BETA, 16, 512),
             ("exp", 1.3, 6, 512), ("mix", 1.0, 9, 512), ("la", 3.5, 7, 512),
             ("exp", GOLDEN_BETA, 2, 16), ("mix", 2.0, 12, 1024)]
    meta["costs"] = []
    for i, (kind, param, k, B) in enumerate(specs):
        fn = dict(exp=cost_exp, mix=cost_mix, la=cost_la)[kind]
        tab = np.array([[fn(j, a, k, param, B) for a in range(k + 1)] for j in range(B + 1)],
                       dtype=np.float64)
        store[f"cost__{i}"] = tab
        meta["costs"].append(dict(kind=kind, param=param, k=k, B=B))


def qgram_kats(store: dict, meta: dict) -> None:
    rng = np.random.default_rng(99)
    alphabet = np.frombuffer(b"ACGTacgtNnRX>", dtype=np.uint8)
    meta["qgrams"] = []
    i = 0
    for q in (1, 2, 3, 5, 8, 15, 16, 17, 31, 32):
        for canonical in (True, False):
            for density in (0.0, 0.02, 0.3):
                L = int(rng.integers(0, 400))
                seq = rng.choice(alphabet[:8], size=L)
                bad = rng.random(L) < density
                seq[bad] = rng.choice(alphabet[8:], size=int(bad.sum()))
                seqb = seq.astype(np.uint8).tobytes()
                keys = encode_qgrams(QGramEncoder(q=q, canonical=canonical), seqb)
                store[f"qg__{i}__seq"] = np.frombuffer(seqb, dtype=np.uint8)
                store[f"qg__{i}__keys"] = keys
                meta["qgrams"].append(dict(q=q, canonical=canonical, idx=i))
                i += 1
    # the reference's own KATs (test_io.py:156-193)
    meta["qgram_kats"] = [
        dict(q=2, canonical=False, seq="ACGT", keys=[1, 6, 11]),
        dict(q=2, canonical=True, seq="GT", keys=[1]),
        dict(q=3, canonical=False, seq="ACNGT", keys=[]),
        dict(q=2, canonical=False, seq="ac", keys=[1]),
        dict(q=2, canonical=False, seq="A", keys=[]),
        dict(q=32, canonical=False, seq="T" * 32, keys=[2**64 - 1]),
        dict(q=2, canonical=True, seq="AT", keys=[3]),
    ]
    for kat in meta["qgram_kats"]:
        got = encode_qgrams(QGramEncoder(q=kat["q"], canonical=kat["canonical"]), kat["seq"])
        assert got.tolist() == kat["keys"], kat
        kat["keys"] = [str(v) for v in kat["keys"]]


def dna_case(store: dict, meta: dict) -> None:
    """cfg4 shape at 1e5 bp: synthetic genome, canonical 31-mers, c=2 k=14."""
    rng = np.random.default_rng(4)
    L = 100_000
    genome = np.frombuffer(b"ACGT", dtype=np.uint8)[rng.integers(0, 4, L)].tobytes()
    enc = QGramEncoder(q=31, canonical=True)
    keys = encode_qgrams(enc, genome)
    cfg = FilterConfig(kind="blowchoc", k=14, choices=2, size_bits=14 * (L - 30), seed=1)
    f = Filter.from_config(cfg)
    f.insert_many(keys)
    # reads of 150 bp with 1% substitutions, plus reads from an unrelated genome
    reads = []
    for _ in range(200):
        s = int(rng.integers(0, L - 150))
        r = bytearray(genome[s: s + 150])
        for p in np.nonzero(rng.random(150) < 0.01)[0]:
            r[p] = b"ACGT"[(b"ACGT".index(r[p]) + int(rng.integers(1, 4))) % 4]
        reads.append(bytes(r))
    other = np.frombuffer(b"ACGT", dtype=np.uint8)[rng.integers(0, 4, 150 * 200)].tobytes()
    reads += [other[i * 150: (i + 1) * 150] for i in range(200)]
    hits = [int(f.contains_many(encode_qgrams(enc, r)).sum()) for r in reads]
    store["dna__genome"] = np.frombuffer(genome, dtype=np.uint8)
    store["dna__reads"] = np.frombuffer(b"".join(reads), dtype=np.uint8)
    meta["dna"] = dict(L=L, genome_seed=4, keys_sha256=sha(keys), n_keys=int(keys.shape[0]),
                       num_blocks=f.num_blocks, words_sha256=sha(f.storage.words),
                       read_hits=hits, reads_sha256=hashlib.sha256(b"".join(reads)).hexdigest())


def bwch_files() -> None:
    """BWCH v1 files written by the reference's write_filter (io.py:60-72)."""
    from blowchoc import write_filter

    out = os.path.join(OUT, "bwch")
    os.makedirs(out, exist_ok=True)
    cases = {
        "blocked_pinned": (FilterConfig(kind="blocked", k=4, size_bits=2 * 512, seed=0x1234),
                           None),
        "blowchoc_mix": (FilterConfig(kind="blowchoc", k=6, n_capacity=300, choices=3,
                                      cost=CostModel("mix", 2.5, 6), seed=99, shards=2), 300),
        "standard": (FilterConfig(kind="standard", k=5, n_capacity=200, seed=5,
                                  block_bits=128), 200),
        "distinct": (FilterConfig(kind="blowchoc", k=7, n_capacity=250, choices=2,
                                  strategy="distinct", seed=3, block_bits=64), 250),
    }
    meta = {}
    for name, (cfg, n) in cases.items():
        f = Filter.from_config(cfg)
        if n is None:  # the reference's own pinned-layout case (test_io.py:70-86)
            f.storage.set_bits(0, {0, 1})
            f.storage.set_bits(1, {64})
        else:
            f.insert_many(even_keys(n, 8))
        p = os.path.join(out, name + ".bwch")
        write_filter(f, p)
        with open(p, "rb") as fh:
            meta[name] = dict(n=n, sha256=hashlib.sha256(fh.read()).hexdigest())
    with open(os.path.join(out, "index.json"), "w") as fh:
        json.dump(meta, fh, indent=1)


def config_cases() -> None:
    """FilterConfig.validated / sizing outcomes of the reference on seeded
    random (mostly invalid) parameter sets: error class and message, or the
    normalised choices / seed and the sizing (config_cases.json)."""
    import random

    rng = random.Random(5)
    grid = dict(kind=["standard", "blocked", "blowchoc", "bogus"], k=[0, 1, 7, 600],
                n_capacity=[None, 0, 1000, 123457], size_bits=[None, 0, 5000, 99991],
                choices=[None, 0, 1, 2, 3, 9], strategy=["random", "distinct", "x"],
                relative_size=[1.0, 0.0, 1.3], shards=[0, 1, 4, 7],
                seed=[0, 2**70 + 3, -5], block_bits=[512, 64, 100, 16, 1024])
    tame = dict(kind=["standard", "blocked", "blowchoc", "blowchoc"], k=[1, 7, 12, 16],
                choices=[None, 2, 3, 8], strategy=["random", "random", "distinct"],
                shards=[1, 1, 4, 7], seed=[0, 1, 2**70 + 3], block_bits=[512, 512, 64, 1024])
    cases = []
    for i in range(1500):
        if i % 3:  # mostly plausible configurations, sized one way or the other
            kw = {name: rng.choice(v) for name, v in tame.items()}
            if rng.random() < 0.5:
                kw["n_capacity"] = rng.randrange(1, 10**7)
                kw["relative_size"] = rng.choice([1.0, 0.8, 1.25])
            else:
                kw["size_bits"] = rng.randrange(1, 10**9)
        else:
            kw = {name: rng.choice(v) for name, v in grid.items()}
        try:
            c = FilterConfig(**kw).validated()
            res = {"ok": True, "choices": c.choices, "seed": c.seed, "sizing": list(c.sizing())}
        except Exception as exc:  # noqa: BLE001 -- the class and message are the fixture
            res = {"ok": False, "error": type(exc).__name__, "message": str(exc)}
        cases.append({"config": kw, "result": res})
    with open(os.path.join(OUT, "config_cases.json"), "w") as fh:
        json.dump(cases, fh, separators=(",", ":"))


def spec_cases() -> None:
    """Hash parameters the reference derives (Filter._derive_hashes,
    filters.py:252-263) for seeded configurations: shard, block and bit
    multipliers and ranges (spec_cases.json)."""
    import random

    rng = random.Random(11)
    cases = []
    for _ in range(300):
        kind = rng.choice(["standard", "blocked", "blowchoc", "blowchoc"])
        kw = dict(kind=kind, k=rng.randrange(1, 24), seed=rng.randrange(0, 2**64),
                  n_capacity=rng.randrange(1, 10**6))
        if kind == "blowchoc":
            kw["choices"] = rng.randrange(2, 9)
        if kind != "standard":
            kw["shards"] = rng.choice([1, 1, 2, 3, 8])
            kw["strategy"] = rng.choice(["random", "distinct"])
            kw["block_bits"] = rng.choice([512, 512, 64, 256, 1024])
        f = Filter.from_config(FilterConfig(**kw))
        cases.append({
            "config": kw,
            "shard": [f.shard_spec.a, f.shard_spec.b],
            "blocks": [[h.a, h.b] for h in f.block_specs],
            "bits": [[h.a, h.b] for h in f.bit_specs],
        })
    with open(os.path.join(OUT, "spec_cases.json"), "w") as fh:
        json.dump(cases, fh, separators=(",", ":"))


def main() -> None:
    spec_cases()
    config_cases()
    bwch_files()
    store: dict = {}
    meta: dict = {}
    hash_kats(store)
    distinct_kats(meta)
    cost_tables(store, meta)
    qgram_kats(store, meta)
    dna_case(store, meta)
    filter_cases(store, meta)
    np.savez_compressed(os.path.join(OUT, "golden.npz"), **store)
    with open(os.path.join(OUT, "golden.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
