"""BWCH v1 filter files and key streams (reference io.py; test_io.py:38-151).

CPU tests read and re-write files produced by the reference itself
(tests/golden/bwch, made by tests/golden/make_golden.py) and pin the byte
layout; the GPU test round-trips a GPU-built filter."""

import hashlib
import json
import os

import numpy as np
import pytest

import paper_2501_18977_b200 as bb
from paper_2501_18977_b200.io import (FilterFormatError, KeyFormatError, read_filter,
                                      read_keys, write_filter)

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "bwch")


def index():
    with open(os.path.join(GOLD, "index.json")) as fh:
        return json.load(fh)


@pytest.mark.parametrize("name", ["blocked_pinned", "blowchoc_mix", "standard", "distinct"])
def test_reference_files_roundtrip_bytes(name, tmp_path, monkeypatch):
    """Read a reference-written file and write it back: identical bytes."""
    import torch

    monkeypatch.setattr(torch.cuda, "is_available", lambda: False)  # host path
    src = os.path.join(GOLD, name + ".bwch")
    f = read_filter(src)
    dst = tmp_path / "out.bwch"
    write_filter(f, dst)
    raw = dst.read_bytes()
    assert hashlib.sha256(raw).hexdigest() == index()[name]["sha256"]
    assert raw == open(src, "rb").read()


def test_file_layout_is_pinned(tmp_path):
    filt = bb.Filter.from_config(bb.FilterConfig(kind="blocked", k=4, size_bits=2 * 512,
                                                 seed=0x1234))
    filt.storage.set_bits(0, {0, 1})
    filt.storage.set_bits(1, {64})
    p = tmp_path / "f"
    write_filter(filt, p)
    raw = p.read_bytes()
    assert len(raw) == 64 + 2 * 64
    assert raw[:4] == b"BWCH"
    assert raw[4:8] == (1).to_bytes(4, "little")
    assert raw[8] == 1
    assert raw[9:11] == (4).to_bytes(2, "little")
    assert raw[24:32] == (512).to_bytes(8, "little")
    assert raw[48:56] == (0x1234).to_bytes(8, "little")
    assert raw[64:72] == (0b11).to_bytes(8, "little")
    assert raw[128 + 8:128 + 16] == (1).to_bytes(8, "little")
    assert raw == open(os.path.join(GOLD, "blocked_pinned.bwch"), "rb").read()


def _mutated(tmp_path, offset, value, name="blocked_pinned"):
    raw = bytearray(open(os.path.join(GOLD, name + ".bwch"), "rb").read())
    raw[offset] = value
    p = tmp_path / "bad"
    p.write_bytes(bytes(raw))
    return p


def test_rejects_corrupt_headers(tmp_path):
    with pytest.raises(FilterFormatError, match="magic"):
        read_filter(_mutated(tmp_path, 0, ord("X")))
    with pytest.raises(FilterFormatError, match="version"):
        read_filter(_mutated(tmp_path, 4, 99))
    with pytest.raises(FilterFormatError, match="shard"):
        read_filter(_mutated(tmp_path, 40, 2, "standard"))
    with pytest.raises(FilterFormatError, match="choices"):
        read_filter(_mutated(tmp_path, 11, 0, "blowchoc_mix"))
    with pytest.raises(FilterFormatError, match="enum"):
        read_filter(_mutated(tmp_path, 8, 7))
    p = tmp_path / "short"
    p.write_bytes(b"BWCH" + b"\x00" * 10)
    with pytest.raises(FilterFormatError, match="header"):
        read_filter(p)


def test_rejects_truncated_or_extended_payload(tmp_path, monkeypatch):
    import torch

    monkeypatch.setattr(torch.cuda, "is_available", lambda: False)
    raw = open(os.path.join(GOLD, "blowchoc_mix.bwch"), "rb").read()
    p = tmp_path / "f"
    p.write_bytes(raw[:-8])
    with pytest.raises(FilterFormatError):
        read_filter(p)
    p.write_bytes(raw + b"\x00")
    with pytest.raises(FilterFormatError):
        read_filter(p)


def test_toy_width_does_not_serialize():
    f = bb.Filter.from_config(bb.FilterConfig(kind="blowchoc", k=2, size_bits=64, block_bits=16))
    with pytest.raises(ValueError):
        write_filter(f, "/dev/null")


def test_u64le_and_text_streams(tmp_path):
    keys = bb.even_keys(3000, 5)
    p = tmp_path / "k.u64"
    keys.astype("<u8").tofile(p)
    got = np.concatenate(list(read_keys(str(p), "u64le", chunk_size=1000)))
    np.testing.assert_array_equal(got, keys)
    p.write_bytes(keys.astype("<u8").tobytes() + b"\x01\x02")
    with pytest.raises(KeyFormatError, match="truncated"):
        list(read_keys(str(p), "u64le"))
    t = tmp_path / "k.txt"
    t.write_text("\n".join(str(int(v)) for v in keys[:50]) + "\n\n")
    np.testing.assert_array_equal(np.concatenate(list(read_keys(str(t), "text"))), keys[:50])
    t.write_text("12\nabc\n")
    with pytest.raises(KeyFormatError, match="line 2"):
        list(read_keys(str(t), "text"))
    t.write_text(str(2**64) + "\n")
    with pytest.raises(KeyFormatError, match="range"):
        list(read_keys(str(t), "text"))
    with pytest.raises(KeyFormatError):
        list(read_keys(str(t), "nope"))
    with pytest.raises(KeyFormatError, match="q-gram"):
        list(read_keys(str(t), "fasta"))


def test_fasta_batches_keep_records_whole_and_in_order(tmp_path):
    from paper_2501_18977_b200.io import fasta_batches, fasta_records

    recs = [b"ACGT" * 5, b"GGCA", b"", b"T" * 30, b"acgtN" * 3]
    fa = tmp_path / "r.fa"
    fa.write_bytes(b"".join(b">h%d desc\n" % i + r[:7] + b"\n" + r[7:] + b"\n"
                            for i, r in enumerate(recs)))
    with open(fa, "rb") as fh:
        kept = list(fasta_records(fh))
    assert kept == [r for r in recs if r]
    for size in (1, 25, 10**6):
        batches = list(fasta_batches(str(fa), batch_bytes=size))
        # joined with a non-ACGT separator: same windows as the records
        assert b"\n".join(batches) == bb.join_records(kept)
        assert all(b.count(b">") == 0 for b in batches)
    assert len(list(fasta_batches(str(fa), batch_bytes=1))) == len(kept)
    bad = tmp_path / "bad.fa"
    bad.write_bytes(b"ACGT\n>h\nACGT\n")
    with pytest.raises(KeyFormatError):
        list(fasta_batches(str(bad)))


def test_native_fasta_join_equals_the_line_loop(tmp_path):
    """bc_fasta_join (fasta_batches) against the reference's line loop
    (fasta_records, io.py:226-242) on ragged inputs: CRLF, blank and
    whitespace-only lines, indented lines, empty records, '>' inside a
    sequence line, no newline at the end, a header as the last line; read in
    chunks of a few bytes, so lines and records straddle every boundary."""
    import io as pyio

    from paper_2501_18977_b200.io import _fasta_joined, fasta_records

    rng = np.random.default_rng(11)
    pieces = [b">h\n", b">h desc > more\r\n", b"  >indented header\n", b"\n", b"  \t \r\n",
              b"ACGT\n", b"acgtnN\r\n", b"  GGA  \n", b"AC>GT\n", b"T" * 300 + b"\n",
              b"\x0b\x0cCA\x0c\n", b"A C\tG\n"]
    for trial in range(60):
        body = b">first\n" + b"".join(pieces[i] for i in rng.integers(0, len(pieces), 40))
        tail = [b"", b"ACG", b">last", b"  "][trial % 4]
        data = body + tail
        want = list(fasta_records(pyio.BytesIO(data)))
        for read_bytes in (1, 7, 64, 1 << 20):
            got = []
            for buf, ends in _fasta_joined(pyio.BytesIO(data), read_bytes=read_bytes):
                a = 0
                for e in ends:
                    got.append(buf[a:int(e)].tobytes())
                    a = int(e) + 1
            assert got == want, (trial, read_bytes)
    # more records than the parser's first record table holds (it stops at the
    # line that needs a slot and is called again with a larger table)
    many = b"".join(b">r%d\nAC\nG%s\n" % (i, b"T" * (i % 5)) for i in range(7000)) + b">x\nA"
    want = list(fasta_records(pyio.BytesIO(many)))
    got = []
    for buf, ends in _fasta_joined(pyio.BytesIO(many)):
        a = 0
        for e in ends:
            got.append(buf[a:int(e)].tobytes())
            a = int(e) + 1
    assert got == want and len(got) == 7001
    from paper_2501_18977_b200.io import fasta_batches
    fa = tmp_path / "many.fa"
    fa.write_bytes(many)
    arr = list(fasta_batches(str(fa), batch_bytes=1000, as_array=True))
    assert b"\n".join(a.tobytes() for a in arr) == bb.join_records(want)
    # parsed ahead in a background thread: same batches; closing early stops it
    ahead = list(fasta_batches(str(fa), batch_bytes=1000, prefetch=3))
    assert ahead == [a.tobytes() for a in arr]
    g = fasta_batches(str(fa), batch_bytes=100, prefetch=2)
    next(g)
    g.close()
    import threading
    assert not [t for t in threading.enumerate() if t.name == "fasta-prefetch"]
    with pytest.raises(KeyFormatError, match="header"):
        list(_fasta_joined(pyio.BytesIO(b"\n  \nACGT\n>h\nAC\n")))
    assert list(_fasta_joined(pyio.BytesIO(b""))) == []
    assert list(_fasta_joined(pyio.BytesIO(b">only a header"))) == []


@pytest.mark.gpu
def test_gpu_filter_roundtrip_and_fasta(tmp_path):
    from oracle import oracle as orc

    cfg = bb.FilterConfig(kind="blowchoc", k=9, n_capacity=50_000, choices=3, seed=4, shards=2)
    f = bb.Filter.from_config(cfg)
    keys = bb.even_keys(50_000, 1)
    f.insert_many(keys)
    p = tmp_path / "g.bwch"
    write_filter(f, p)
    g = read_filter(p)
    np.testing.assert_array_equal(g.storage.words, f.storage.words)
    assert g.inserted == f.inserted and g.cost == f.cost
    probes = np.concatenate([keys[:1000], bb.odd_keys(20_000, 2)])
    np.testing.assert_array_equal(g.contains_many(probes), f.contains_many(probes))
    # the reference-written files load onto the device with identical lookups
    for name in ("blowchoc_mix", "distinct"):
        h = read_filter(os.path.join(GOLD, name + ".bwch"))
        pr = np.concatenate([bb.even_keys(index()[name]["n"], 8), bb.odd_keys(3000, 9)])
        o = orc.make_filter(h.kind, k=h.k, choices=h.choices, strategy=h.strategy,
                            block_bits=h.block_bits, shards=h.shards, seed=h.seed,
                            size_bits=h.num_blocks * h.block_bits,
                            cost_code=h.cost.code, cost_param=h.cost.param)
        o.words[:] = h.storage.words
        np.testing.assert_array_equal(h.contains_many(pr), o.contains_many(pr))
        assert h.contains_many(pr[: index()[name]["n"]]).all()
    fa = tmp_path / "x.fa"
    fa.write_bytes(b">r1\nACGTACGTAC\nGTTTACG\n>r2 desc\nNNACGTAAAC\n")
    chunks = list(read_keys(str(fa), "fasta", q=5))
    assert len(chunks) == 2
    np.testing.assert_array_equal(chunks[0], orc.encode_qgrams(b"ACGTACGTACGTTTACG", 5))
    np.testing.assert_array_equal(chunks[1], orc.encode_qgrams(b"NNACGTAAAC", 5))


@pytest.mark.gpu
def test_gpu_filter_files_in_many_slices(tmp_path, monkeypatch):
    """Device filters are written and read through two pinned slices, the
    copies overlapped with the file I/O: with slices of 777 words (several per
    file, a ragged last one) the file equals the one written from the host
    copy, reads give back the words, and a truncated file is still rejected."""
    from paper_2501_18977_b200 import io as bio

    cfg = bb.FilterConfig(kind="blowchoc", k=9, n_capacity=50_000, choices=2, seed=6)
    f = bb.Filter.from_config(cfg)
    f.insert_many(torch_keys := bb.even_keys(50_000, 3, device="cuda"))
    want_words = f.storage.d_words.cpu().numpy().copy()
    monkeypatch.setattr(bio, "_SLICE_WORDS", 777)
    p = tmp_path / "sliced.bwch"
    write_filter(f, p)                      # device words, pinned slices
    raw = p.read_bytes()
    assert raw[64:] == want_words.astype("<u8").tobytes()
    g = read_filter(p)
    np.testing.assert_array_equal(g.storage.d_words.cpu().numpy(), want_words)
    assert g.contains_many(torch_keys).all()
    (tmp_path / "cut.bwch").write_bytes(raw[:-5])
    with pytest.raises(FilterFormatError, match="expected"):
        read_filter(tmp_path / "cut.bwch")
    (tmp_path / "long.bwch").write_bytes(raw + b"x")
    with pytest.raises(FilterFormatError, match="more than"):
        read_filter(tmp_path / "long.bwch")


def _python_keys(text: bytes):
    """The reference's text rule (io.py:206-223) restated in Python."""
    keys = []
    for line in text.split(b"\n"):
        line = line.strip()
        if line:
            keys.append(int(line))
    return keys


@pytest.mark.parametrize("block", [7, 64, 1 << 24])
def test_native_text_parser_matches_python_int(tmp_path, monkeypatch, block):
    """bc_parse_keys_text accepts exactly what int() accepts (sign, leading
    zeros, single underscores, surrounding whitespace, CRLF, blank lines),
    across read-block boundaries and output chunks."""
    import paper_2501_18977_b200.io as bio

    monkeypatch.setattr(bio, "_TEXT_BLOCK", block)
    rng = np.random.default_rng(9)
    vals = rng.integers(0, 2**64, size=500, dtype=np.uint64).tolist()
    forms = []
    for i, v in enumerate(vals):
        s = str(v)
        kind = i % 7
        if kind == 1:
            s = "+" + s
        elif kind == 2:
            s = "000" + s
        elif kind == 3 and len(s) > 3:
            s = s[:2] + "_" + s[2:]
        elif kind == 4:
            s = " \t" + s + " \r"
        elif kind == 5:
            s = s + "\n"  # a blank line follows
        forms.append(s)
    forms += ["-0", "0", str(2**64 - 1), "1_0_0"]
    text = ("\n".join(forms)).encode()  # no trailing newline
    p = tmp_path / "k.txt"
    p.write_bytes(text)
    got = np.concatenate(list(read_keys(str(p), "text", chunk_size=37)))
    assert got.tolist() == _python_keys(text)


@pytest.mark.parametrize("threads", ["1", "5"])
def test_native_text_parser_large_blocks(tmp_path, threads):
    """Blocks of several MB are cut at line ends and parsed by several threads
    (BC_PARSE_THREADS, read at first use, hence the subprocess): the keys
    equal Python's int() of every non-blank line; output chunks smaller than a
    block and a rejected line far into the file behave as with one thread
    (the reference's line number and wording, io.py:206-223)."""
    import subprocess
    import sys

    script = r"""
import numpy as np, sys
from paper_2501_18977_b200.io import read_keys, KeyFormatError
rng = np.random.default_rng(3)
vals = rng.integers(0, 2**64, size=400_000, dtype=np.uint64).tolist()
forms = []
for i, v in enumerate(vals):
    s = str(v)
    k = i % 9
    if k == 1: s = "+" + s
    elif k == 2: s = "00" + s
    elif k == 3 and len(s) > 4: s = s[:3] + "_" + s[3:]
    elif k == 4: s = "  " + s + " \r"
    elif k == 5: s = s + "\n"
    elif k == 6: s = s + "\n \t"
    forms.append(s)
text = ("\n".join(forms)).encode()
path = sys.argv[1]
open(path, "wb").write(text)
want = [int(l) for l in text.split(b"\n") if l.strip()]
for chunk in (1 << 20, 70_001):
    got = np.concatenate(list(read_keys(path, "text", chunk_size=chunk)))
    assert got.tolist() == want, chunk
lines = text.split(b"\n")
bad_at = len(lines) - 1000
lines[bad_at] = b"12x4"
open(path, "wb").write(b"\n".join(lines))
try:
    list(read_keys(path, "text"))
    print("no error")
except KeyFormatError as e:
    print(str(e) == f"line {bad_at + 1}: not an integer: b'12x4'", len(text))
"""
    out = subprocess.run([sys.executable, "-c", script, str(tmp_path / "big.txt")],
                         env=dict(os.environ, BC_PARSE_THREADS=threads), capture_output=True,
                         text=True, cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert out.returncode == 0, out.stderr
    ok, size = out.stdout.split()
    assert ok == "True" and int(size) > 6_000_000


@pytest.mark.parametrize("bad,msg", [
    (b"1__0", "line 3: not an integer"), (b"_1", "line 3: not an integer"),
    (b"1_", "line 3: not an integer"), (b"0x10", "line 3: not an integer"),
    (b"1 2", "line 3: not an integer"), (b"-1", "line 3: key out of 64-bit range: -1"),
    (str(2**64).encode(), f"line 3: key out of 64-bit range: {2**64}"),
])
def test_native_text_parser_errors(tmp_path, bad, msg):
    p = tmp_path / "k.txt"
    p.write_bytes(b"5\n\n" + bad + b"\n7\n")
    with pytest.raises(KeyFormatError, match=msg.replace("+", r"\+")):
        list(read_keys(str(p), "text"))
