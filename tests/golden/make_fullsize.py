"""Full-size golden digests of the reference's stream-order builds for
BASELINE configs 3, 4 (c = 2) and 5.

Runs ONLY in the build container, where the reference is importable from
/root/reference/pkg/src (numba JIT); writes tests/golden/fullsize_cfg{N}.json,
which the -m gpu tests compare the exact-order GPU builds against.  Nothing
at test time touches /root/reference.

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_fullsize.py 3|4|5

Every build goes through the reference's public API (Filter.from_config,
insert_many, contains_many, storage.words, encode_qgrams) on the key
streams the bench and the GPU tests generate on the device:

* cfg3 / cfg5: ``even_keys(n, 11)`` (analysis.py:34-37), drawn in chunks of
  the same numpy PCG64 stream (a full-range uint64 draw consumes exactly
  one 64-bit output per key, so chunked draws equal one draw);
* cfg4: a 1.2e9-bp genome whose base i is ``"ACGT"[w_i >> 62]`` for the
  i-th 64-bit word of ``default_rng(GENOME_SEED).integers(0, 2**64,
  uint64)``; its canonical 31-mers are encoded with the reference's
  ``encode_qgrams`` in chunks overlapping by q - 1 bases (every window is
  valid, so the chunks' windows are exactly the genome's, in order) and
  inserted in stream order.

Recorded: sha256 of the words (cfg5 also after the first 2^32 keys, the
design load), and lookup pins on the final bit array: the false-positive
count over ``odd_keys(2^24, 12)`` and the sha256 of the answers to its first
2^20 keys.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, REF)

from blowchoc import Filter, FilterConfig, QGramEncoder, encode_qgrams, odd_keys  # noqa: E402

CHUNK = 1 << 26
GENOME_SEED = 4
GENOME_LEN = 1_200_000_000
Q = 31
N_NEG = 1 << 24

CASES = {
    3: dict(cfg=dict(kind="blowchoc", k=16, choices=3, size_bits=16 * 2**28, seed=1),
            n=2**28, marks=()),
    4: dict(cfg=dict(kind="blowchoc", k=14, choices=2, size_bits=14 * (GENOME_LEN - Q + 1),
                     seed=1), n=GENOME_LEN - Q + 1, marks=()),
    5: dict(cfg=dict(kind="blowchoc", k=11, choices=2, size_bits=2**36, seed=1),
            n=int(1.2 * 2**32), marks=(2**32,)),
}


def log(msg: str) -> None:
    print(f"[{time.strftime('%H:%M:%S')}] {msg}", flush=True)


def sha(a: np.ndarray) -> str:
    h = hashlib.sha256()
    v = np.ascontiguousarray(a).view(np.uint8)
    step = 1 << 30
    for i in range(0, v.shape[0], step):
        h.update(v[i:i + step])
    return h.hexdigest()


def key_chunks(n: int, seed: int):
    """even_keys(n, seed) in CHUNK-sized pieces of the same stream."""
    rng = np.random.default_rng(seed)
    done = 0
    while done < n:
        m = min(CHUNK, n - done)
        yield rng.integers(0, 2**64, size=m, dtype=np.uint64) & ~np.uint64(1)
        done += m


def genome_chunks(length: int, seed: int, overlap: int):
    """The PCG64-word genome as ASCII, in CHUNK-base pieces overlapping by
    ``overlap`` bases."""
    rng = np.random.default_rng(seed)
    alphabet = np.frombuffer(b"ACGT", dtype=np.uint8)
    tail = np.empty(0, dtype=np.uint8)
    done = 0
    while done < length:
        m = min(CHUNK, length - done)
        w = rng.integers(0, 2**64, size=m, dtype=np.uint64)
        bases = alphabet[(w >> np.uint64(62)).astype(np.intp)]
        yield np.concatenate([tail, bases])
        tail = bases[-overlap:] if overlap else np.empty(0, dtype=np.uint8)
        done += m


def main(cfgno: int) -> None:
    case = CASES[cfgno]
    f = Filter.from_config(FilterConfig(**case["cfg"]))
    words = f.storage.words
    log(f"cfg{cfgno}: {words.nbytes / 2**20:.0f} MiB filter, {case['n']} keys")
    res = {"config": cfgno, "filter": case["cfg"], "n_keys": case["n"], "marks": {}}
    t0 = time.time()
    done = 0
    if cfgno == 4:
        enc = QGramEncoder(Q, True)
        res["genome"] = dict(length=GENOME_LEN, seed=GENOME_SEED, q=Q, canonical=True,
                             base_rule="ACGT[(pcg64 uint64 word i) >> 62]")
        for seq in genome_chunks(GENOME_LEN, GENOME_SEED, Q - 1):
            keys = encode_qgrams(enc, seq.tobytes())
            f.insert_many(keys)
            done += keys.shape[0]
            log(f"  {done} k-mers ({done / (time.time() - t0) / 1e6:.2f} M/s)")
    else:
        marks = list(case["marks"])
        for keys in key_chunks(case["n"], 11):
            if marks and done + keys.shape[0] > marks[0]:
                cut = marks[0] - done
                f.insert_many(keys[:cut])
                res["marks"][str(marks[0])] = sha(words)
                log(f"  mark {marks[0]}: {res['marks'][str(marks[0])]}")
                f.insert_many(keys[cut:])
                marks.pop(0)
            else:
                f.insert_many(keys)
            done += keys.shape[0]
            log(f"  {done} keys ({done / (time.time() - t0) / 1e6:.2f} M/s)")
    assert done == case["n"], (done, case["n"])
    res["insert_seconds"] = round(time.time() - t0, 1)
    res["words_sha256"] = sha(words)
    neg = odd_keys(N_NEG, 12)
    out = f.contains_many(neg)
    res["neg_keys"] = dict(n=N_NEG, stream="odd_keys(n, 12)", false_positives=int(out.sum()),
                           answers_sha256_first_2p20=sha(out[: 1 << 20].astype(np.uint8)))
    res["set_bits"] = int(f.storage.total_set_bits())
    log(f"cfg{cfgno}: words {res['words_sha256']} fp {res['neg_keys']['false_positives']}")
    with open(os.path.join(OUT, f"fullsize_cfg{cfgno}.json"), "w") as fh:
        json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main(int(sys.argv[1]))
