"""The command-line front end (reference cli.py:118-171,253-330): argument
handling, exit codes and TSV formatting on the CPU; build / query / fpr / hist
end to end on the GPU, checked against the oracle and against filter files
written by the reference itself (tests/golden/bwch)."""

import os
import subprocess
import sys

import numpy as np
import pytest

from oracle import oracle as orc
from paper_2501_18977_b200 import cli

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden", "bwch")


def run_cli(*args, stdin=None):
    return subprocess.run([sys.executable, "-m", "paper_2501_18977_b200", *map(str, args)],
                          cwd=ROOT, capture_output=True, input=stdin, timeout=300)


def expected_tsv(keys, answers) -> bytes:
    return "".join(f"{k}\t{int(a)}\n" for k, a in zip(np.asarray(keys).tolist(),
                                                      np.asarray(answers).tolist())).encode()


# -- CPU ---------------------------------------------------------------------------------

def test_format_answers_matches_python_formatting():
    rng = np.random.default_rng(3)
    keys = rng.integers(0, 2**64, size=5000, dtype=np.uint64)
    keys[:8] = [0, 1, 9, 10, 99, 100, 10**19, 2**64 - 1]
    keys[8:2000] = rng.integers(0, 10**6, size=1992)
    ans = rng.integers(0, 2, size=keys.size).astype(bool)
    assert cli.format_answers(keys, ans) == expected_tsv(keys, ans)
    assert cli.format_answers(np.zeros(0, np.uint64), np.zeros(0, bool)) == b""
    with pytest.raises(ValueError):
        cli.format_answers(keys, ans[:-1])


def test_format_answers_large_batches_in_threads():
    """Batches of 2^18 keys and more are formatted by several threads (a
    length pass fixes every thread's output offset): every digit count, the
    powers of ten and their neighbours included, lands where the serial
    formatter puts it."""
    rng = np.random.default_rng(8)
    n = (1 << 19) + 77
    keys = rng.integers(0, 2**64, n, dtype=np.uint64)
    keys[: n // 2] >>= rng.integers(0, 64, n // 2).astype(np.uint64)
    edge = [0, 1, 9, 2**64 - 1] + [10**k for k in range(20)] + [10**k - 1 for k in range(1, 20)]
    keys[rng.choice(n, len(edge), replace=False)] = np.array(edge, dtype=np.uint64)
    ans = rng.integers(0, 2, n).astype(bool)
    assert cli.format_answers(keys, ans) == expected_tsv(keys, ans)


def test_usage_errors_exit_1():
    assert cli.main([]) == cli.EXIT_USAGE
    assert cli.main(["build", "--kind", "blowchoc"]) == cli.EXIT_USAGE
    assert cli.main(["build", "--kind", "nope", "--k", "3", "--keys", "x", "--out", "y"]) == 1
    # cost options on a non-blowchoc filter (cli.py:97-98)
    assert cli.main(["build", "--kind", "blocked", "--k", "4", "--n", "10", "--cost", "exp",
                     "--keys", "-", "--out", "/dev/null"]) == cli.EXIT_USAGE


def test_missing_and_corrupt_files(tmp_path):
    assert cli.main(["hist", "--filter", str(tmp_path / "absent.bwch")]) == cli.EXIT_IO
    bad = tmp_path / "bad.bwch"
    bad.write_bytes(b"NOTAFILTER" + bytes(200))
    assert cli.main(["hist", "--filter", str(bad)]) == cli.EXIT_CORRUPT
    good = open(os.path.join(GOLD, "blowchoc_mix.bwch"), "rb").read()
    trunc = tmp_path / "trunc.bwch"
    trunc.write_bytes(good[:-8])
    assert cli.main(["query", "--filter", str(trunc), "--keys", "-"]) == cli.EXIT_CORRUPT


def test_module_entry_point_usage():
    r = run_cli("--help")
    assert r.returncode == 0 and b"build" in r.stdout and b"query" in r.stdout
    assert run_cli("frobnicate").returncode == cli.EXIT_USAGE


# -- GPU ---------------------------------------------------------------------------------

def oracle_of(path):
    """Oracle filter with the geometry, hashes and words of a BWCH file."""
    from paper_2501_18977_b200.io import HEADER, _check_header

    raw = open(path, "rb").read()
    kind, k, c, strategy, cost, block_bits, nb, shards, seed, inserted = \
        _check_header(HEADER.unpack(raw[:HEADER.size]))
    code = {"exp": 0, "mix": 1, "la": 2}[cost.kind] if cost else 0
    o = orc.OracleFilter(kind=kind, k=k, choices=c, strategy=strategy, block_bits=block_bits,
                         num_blocks=nb, shards=shards, seed=seed, cost_code=code,
                         cost_param=cost.param if cost else orc.GOLDEN_BETA)
    o.words[:] = np.frombuffer(raw[HEADER.size:], dtype="<u8")
    return o, inserted


@pytest.mark.gpu
@pytest.mark.parametrize("name,n", [("blowchoc_mix", 300), ("standard", 200),
                                    ("distinct", 250)])
def test_query_reference_written_filters(name, n, tmp_path):
    """Query files the reference wrote (keys even_keys(n, 8), make_golden.py):
    the per-key TSV equals the oracle's answers on the file's own words."""
    path = os.path.join(GOLD, name + ".bwch")
    o, _ = oracle_of(path)
    probes = np.concatenate([orc.even_keys(n, 8), orc.odd_keys(3000, 9)])
    keyfile = tmp_path / "probes.txt"
    keyfile.write_text("\n".join(str(x) for x in probes.tolist()) + "\n")
    r = run_cli("query", "--filter", path, "--keys", keyfile, "--format", "text")
    assert r.returncode == 0, r.stderr.decode()
    want = o.contains_many(probes)
    assert want[:n].all()
    assert r.stdout == expected_tsv(probes, want)


@pytest.mark.gpu
@pytest.mark.parametrize("kind,c,threads", [("blowchoc", 2, 0), ("blowchoc", 3, 4),
                                            ("blocked", 1, 2), ("standard", 0, 0)])
def test_build_query_hist_fpr_end_to_end(kind, c, threads, tmp_path):
    """build -> file words equal the oracle's (ordered inserts, shards from
    --threads); query, hist and fpr agree with the oracle on them."""
    n, k = 20000, 9
    keys = orc.even_keys(n, 21)
    kf = tmp_path / "keys.u64"
    keys.astype("<u8").tofile(kf)
    out = tmp_path / "f.bwch"
    args = ["build", "--kind", kind, "--k", k, "--n", n, "--threads", threads, "--seed", 17,
            "--keys", kf, "--out", out]
    if kind == "blowchoc":
        args += ["--choices", c]
    r = run_cli(*args)
    assert r.returncode == 0, r.stderr.decode()
    head, row = r.stderr.decode().strip().splitlines()[-2:]
    assert head.split("\t")[0] == "keys_inserted" and row.split("\t")[0] == str(n)

    shards = 1 if kind == "standard" else max(1, threads)
    ref = orc.make_filter(kind, k=k, choices=c or None, n_capacity=n, seed=17, shards=shards)
    ref.insert_many(keys)
    o, inserted = oracle_of(out)
    assert inserted == n
    np.testing.assert_array_equal(o.words, ref.words)

    probes = np.concatenate([keys[::7], orc.odd_keys(50000, 22)])
    pf = tmp_path / "probes.u64"
    probes.astype("<u8").tofile(pf)
    r = run_cli("query", "--filter", out, "--keys", pf)
    assert r.returncode == 0, r.stderr.decode()
    assert r.stdout == expected_tsv(probes, ref.contains_many(probes))

    neg = orc.odd_keys(100000, 23)
    nf = tmp_path / "neg.u64"
    neg.astype("<u8").tofile(nf)
    r = run_cli("fpr", "--filter", out, "--keys", nf)
    assert r.returncode == 0, r.stderr.decode()
    header, vals = r.stdout.decode().strip().splitlines()
    row = dict(zip(header.split("\t"), vals.split("\t")))
    assert int(row["N"]) == neg.size
    assert int(row["W"]) == int(ref.contains_many(neg).sum())

    r = run_cli("hist", "--filter", out)  # standard: block-aligned windows
    assert r.returncode == 0, r.stderr.decode()
    lines = r.stdout.decode().strip().splitlines()
    counts = np.array([int(x.split("\t")[1]) for x in lines[1:]])
    np.testing.assert_array_equal(counts, ref.block_histogram())

    # fpr from generated negatives (the device odd-key stream): the count
    # equals the oracle's on the same numpy stream
    import paper_2501_18977_b200 as bb
    r = run_cli("fpr", "--filter", out, "--negatives", 300000, "--neg-seed", 77)
    assert r.returncode == 0, r.stderr.decode()
    header, vals = r.stdout.decode().strip().splitlines()
    row = dict(zip(header.split("\t"), vals.split("\t")))
    neg = np.concatenate([bb.odd_keys(min(bb.DEFAULT_CHUNK, 300000 - a),
                                      bb.derive_seed(77, i))
                          for i, a in enumerate(range(0, 300000, bb.DEFAULT_CHUNK))])
    assert int(row["N"]) == 300000
    assert int(row["W"]) == int(ref.contains_many(neg).sum())


@pytest.mark.gpu
@pytest.mark.parametrize("canonical", [True, False])
def test_fasta_build_fused_equals_record_stream(canonical, tmp_path):
    """build --format fasta runs the fused q-gram insert over batches of whole
    records; the words equal the oracle's insert of each record's q-grams in
    record order (c = 2, ordered), and query prints every window's key."""
    rng = np.random.default_rng(5)
    recs = []
    for i in range(7):
        seq = bytearray(rng.choice(np.frombuffer(b"ACGTacgt", np.uint8),
                                    size=int(rng.integers(5, 4000))).tobytes())
        for p in rng.integers(0, len(seq), size=3):
            seq[p] = ord("N")
        recs.append(bytes(seq))
    fa = tmp_path / "r.fa"
    fa.write_bytes(b"".join(b">r%d\n" % i + r[:60] + b"\n" + r[60:] + b"\n"
                            for i, r in enumerate(recs)))
    q, k = 21, 8
    keys = np.concatenate([orc.encode_qgrams(r, q, canonical) for r in recs])
    out = tmp_path / "f.bwch"
    args = ["build", "--kind", "blowchoc", "--k", k, "--choices", 2, "--n", keys.size,
            "--seed", 3, "--keys", fa, "--format", "fasta", "--q", q, "--out", out]
    if not canonical:
        args.append("--no-canonical")
    r = run_cli(*args)
    assert r.returncode == 0, r.stderr.decode()
    ref = orc.make_filter("blowchoc", k=k, choices=2, n_capacity=keys.size, seed=3)
    ref.insert_many(keys)
    o, inserted = oracle_of(out)
    assert inserted == keys.size
    np.testing.assert_array_equal(o.words, ref.words)
    qargs = ["query", "--filter", out, "--keys", fa, "--format", "fasta", "--q", q]
    if not canonical:
        qargs.append("--no-canonical")
    r = run_cli(*qargs)
    assert r.returncode == 0, r.stderr.decode()
    assert r.stdout == expected_tsv(keys, np.ones(keys.size, dtype=bool))
