"""Exercise every kernel of libbbchoc on small inputs (for compute-sanitizer):

    compute-sanitizer --tool memcheck python tools/sanitize_smoke.py
    compute-sanitizer --tool racecheck python tools/sanitize_smoke.py

Checks results against the CPU oracle so a silent corruption also fails."""

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2501_18977_b200 as bb  # noqa: E402
from oracle import oracle as orc  # noqa: E402


def check(kind, c, strategy="random", B=512, k=7, n=3000, shards=1, mode="ordered"):
    cfg = bb.FilterConfig(kind=kind, k=k, n_capacity=n, choices=c, strategy=strategy,
                          block_bits=B, shards=shards, seed=5)
    f = bb.Filter.from_config(cfg, insert_mode=mode)
    o = orc.make_filter(kind, k=k, n_capacity=n, choices=c, strategy=strategy, block_bits=B,
                        shards=shards, seed=5)
    keys = bb.even_keys(n, 1)
    f.insert_many(torch.from_numpy(keys).cuda())
    o.insert_many(keys)
    probes = np.concatenate([keys[:500], bb.odd_keys(777, 2)])
    got = f.contains_many(torch.from_numpy(probes).cuda()).cpu().numpy()
    if mode == "ordered" or c in (None, 1):
        assert np.array_equal(f.storage.words, o.words), (kind, c, strategy, B)
        assert np.array_equal(got, o.contains_many(probes)), (kind, c, strategy, B)
    else:
        assert got[:500].all()
    bb.block_load_histogram(f)
    f.count_hits(probes)


def main():
    for kind, c in (("standard", None), ("blocked", 1), ("blowchoc", 2), ("blowchoc", 3)):
        check(kind, c)
    check("blowchoc", 2, mode="relaxed")
    check("blowchoc", 4, strategy="distinct")
    check("blowchoc", 2, B=16, k=2)
    check("blowchoc", 3, B=1024, k=12, shards=4)
    check("blocked", 1, strategy="distinct", shards=2)
    enc = bb.QGramEncoder(31)
    rng = np.random.default_rng(3)
    genome = np.frombuffer(b"ACGTN", dtype=np.uint8)[rng.choice(5, 20_000,
                                                                p=[.24] * 4 + [.04])].tobytes()
    for kind, c, mode in (("blocked", 1, "ordered"), ("blowchoc", 2, "relaxed"),
                          ("blowchoc", 2, "ordered")):
        f = bb.Filter.from_config(bb.FilterConfig(kind=kind, k=9, n_capacity=20_000, choices=c,
                                                  seed=2), insert_mode=mode)
        f.insert_qgrams(enc, genome)
        assert f.contains_qgrams(enc, genome).all()
        f.count_qgram_hits(enc, genome)
    np.testing.assert_array_equal(bb.encode_qgrams(enc, genome), orc.encode_qgrams(genome, 31))
    np.testing.assert_array_equal(bb.even_keys(1000, 3, device="cuda").cpu().numpy(),
                                  bb.even_keys(1000, 3))
    bb.eval_hash_many(bb.HashSpec(a=2**63 + 1, b=1000), bb.even_keys(1000, 4))
    torch.cuda.synchronize()
    print("sanitize smoke ok")


if __name__ == "__main__":
    main()
