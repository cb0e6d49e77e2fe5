"""Measurement of the SURVEY §8(f) rows around the hot path (GPU box, 1 GPU).

One JSON line per row, each with a parity check on the same data and a CPU
restatement of the reference's own implementation timed beside it:

  hist     block_load_histogram (analysis.py:135-146: np.bitwise_count per
           word, per-block sums, bincount) -- GPU kernel vs numpy; roofline is
           the streaming read of the words against MEASURED_PEAKS hbm_gbs
  fpr      estimate_fpr with the reference's negative stream generated on the
           device (analysis.py:86-107) -- count-only lookups, keys/s
  bwch     write_filter / read_filter round trip (io.py:60-121), GB/s
  u64le    read_keys(fmt="u64le") (io.py:191-203), MB/s
  text     read_keys(fmt="text") (io.py:206-223: int() per line) -- native
           parser vs the reference's per-line int()
  fasta    FASTA records -> fused q-gram insert (io.py:226-267 + 126-177),
           bases/s
  tsv      CLI query output (cli.py:141-142 f-string per key) -- native
           bc_format_answers vs the f-string join
  standard the standard (flat) Bloom kind (_kernels.py:214-237) at config 2's
           size -- not a BASELINE config; k random bits per key anywhere in
           the array (parity: tests/test_gpu_parity.py golden 'standard')

usage: python tools/bench_next.py [--out profiles/r1/bench_next.jsonl]
The oracle is not used: the CPU restatements here are numpy / Python
one-liners of the reference code cited above.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        for k in ("hbm_gbs", "hbm_copy_gbs"):
            if k in d:
                return float(d[k]), "MEASURED_PEAKS.json " + k
    except (OSError, ValueError):
        pass
    return 7672.0, "B200_PROFILING.md fallback"


def cuda_ms(fn, reps=5):
    import torch

    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def wall(fn, reps=1):
    fn()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    return (time.perf_counter() - t) / reps


def ref_hist(words: np.ndarray, wpb: int) -> np.ndarray:
    per_block = np.bitwise_count(words).reshape(-1, wpb).sum(axis=1, dtype=np.int64)
    return np.bincount(per_block, minlength=wpb * 64 + 1)


def row_hist(bb, torch, out):
    peak, src = hbm_peak()
    for label, mib in (("96 MiB (cfg2)", 96), ("512 MiB (cfg3)", 512), ("8 GiB (cfg5)", 8192)):
        f = bb.Filter.from_config(
            bb.FilterConfig(kind="blowchoc", k=11, choices=2, size_bits=mib << 23, seed=1))
        d = f.storage.d_words
        g = torch.Generator(device=d.device).manual_seed(5)
        d.view(torch.int64).copy_(torch.randint(-2**63, 2**63 - 1, (d.numel(),), device=d.device,
                                                dtype=torch.int64, generator=g))
        # ~55% of bits set, like a filter at design load
        d.view(torch.int64).bitwise_and_(torch.randint(-2**63, 2**63 - 1, (d.numel(),),
                                                       device=d.device, dtype=torch.int64,
                                                       generator=g) | 0x0101010101010101)
        f.storage.device_modified()
        ms = cuda_ms(lambda: f.storage.histogram())
        got = f.storage.histogram()
        nbytes = d.numel() * 8
        # the kernel alone (bc_block_histogram into a resident counts buffer),
        # without the counts' zeroing, D2H copy and host sync of the API call
        import ctypes

        from paper_2501_18977_b200 import _native

        counts = torch.zeros(513, dtype=torch.int64, device=d.device)
        stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        kms = cuda_ms(lambda: _native.check(_native.lib().bc_block_histogram(
            ctypes.c_void_p(d.data_ptr()), f.storage.num_blocks, 512,
            ctypes.c_void_p(counts.data_ptr()), stream)), reps=20)
        line = {"row": "hist", "workload": label, "call_ms": round(ms, 4),
                "kernel_ms": round(kms, 4), "kernel_gbs": round(nbytes / kms / 1e6, 1),
                "peak_gbs": peak, "peak_source": src,
                "kernel_frac": round(nbytes / kms / 1e6 / peak, 4)}
        if mib <= 512:
            host = d.cpu().numpy().view(np.uint64)
            t = wall(lambda: ref_hist(host, 8))
            line["parity"] = "identical" if np.array_equal(ref_hist(host, 8), got) else "DIFF"
            line["cpu_numpy_s"] = round(t, 4)
            line["cpu_numpy_gbs"] = round(nbytes / t / 1e9, 2)
        out(line)
        del f, d


def row_fpr(bb, torch, out):
    n = 1 << 26
    f = bb.Filter.from_config(bb.FilterConfig(kind="blocked", k=12, choices=1,
                                              size_bits=12 * n, seed=1))
    f.insert_many(bb.even_keys(n, 11, device=f.device))
    nq = 1 << 28
    ms = cuda_ms(lambda: bb.estimate_fpr(f, n_queries=nq, seed=12), reps=2)
    est = bb.estimate_fpr(f, n_queries=nq, seed=12)
    out({"row": "fpr", "workload": "cfg2 filter, 2^28 device-generated negatives (count-only)",
         "gpu_ms": round(ms, 3), "mkeys_s": round(nq / ms / 1e3, 1), "fpr": est.fpr,
         "reference_fpr_cfg2": 6.14e-3})


def row_bwch(bb, torch, out, tmp):
    from paper_2501_18977_b200 import io as bio

    n = 1 << 26
    f = bb.Filter.from_config(bb.FilterConfig(kind="blocked", k=12, choices=1,
                                              size_bits=12 * n, seed=1))
    f.insert_many(bb.even_keys(n, 11, device=f.device))
    path = os.path.join(tmp, "f.bwch")
    tw = wall(lambda: bio.write_filter(f, path))
    tr = wall(lambda: bio.read_filter(path))
    g = bio.read_filter(path)
    same = torch.equal(g.storage.d_words, f.storage.d_words)
    nbytes = os.path.getsize(path)
    out({"row": "bwch", "workload": "cfg2 filter (96 MiB) to a local file and back",
         "bytes": nbytes, "write_gbs": round(nbytes / tw / 1e9, 2),
         "read_gbs": round(nbytes / tr / 1e9, 2), "parity": "identical" if same else "DIFF"})


def row_keys(bb, torch, out, tmp):
    from paper_2501_18977_b200 import io as bio

    keys = bb.even_keys(1 << 24, 11)
    p = os.path.join(tmp, "k.u64")
    keys.astype("<u8").tofile(p)
    got = []
    t = wall(lambda: got.__setitem__(slice(None), list(bio.read_keys(p, "u64le"))))
    ok = np.array_equal(np.concatenate(got), keys)
    out({"row": "u64le", "workload": "2^24 keys (128 MiB)", "mb_s": round(keys.nbytes / t / 1e6, 1),
         "parity": "identical" if ok else "DIFF"})

    p = os.path.join(tmp, "k.txt")
    with open(p, "w") as fh:
        fh.write("\n".join(str(int(k)) for k in keys[: 1 << 22]) + "\n")
    size = os.path.getsize(p)
    t = wall(lambda: got.__setitem__(slice(None), list(bio.read_keys(p, "text"))))
    ok = np.array_equal(np.concatenate(got), keys[: 1 << 22])
    # the reference parses line by line with int() (io.py:206-223); timed on a sample
    sample = open(p, "rb").read(1 << 24)
    sample = sample[: sample.rfind(b"\n") + 1]

    def ref():
        return np.array([int(line) for line in sample.splitlines()], dtype=np.uint64)

    tr = wall(ref)
    out({"row": "text", "workload": "2^22 decimal keys", "bytes": size,
         "mb_s": round(size / t / 1e6, 1), "cpu_reference_mb_s": round(len(sample) / tr / 1e6, 1),
         "parity": "identical" if ok else "DIFF"})


def row_fasta(bb, torch, out, tmp):
    rng = np.random.default_rng(3)
    p = os.path.join(tmp, "g.fa")
    nrec, rec_len = 64, 1 << 20
    with open(p, "wb") as fh:
        for r in range(nrec):
            seq = np.frombuffer(b"ACGT", dtype=np.uint8)[rng.integers(0, 4, rec_len)]
            fh.write(b">r%d\n" % r)
            for a in range(0, rec_len, 80):
                fh.write(seq[a:a + 80].tobytes() + b"\n")
    from paper_2501_18977_b200 import io as bio

    enc = bb.QGramEncoder(q=31, canonical=True)
    cfg = bb.FilterConfig(kind="blowchoc", k=14, choices=2, size_bits=14 * nrec * rec_len, seed=1)

    def run():  # as the CLI's build does: no host sync per batch
        f = bb.Filter.from_config(cfg, insert_mode="relaxed")
        total = f.insert_qgram_batches(enc, bio.fasta_batches(p, batch_bytes=1 << 24,
                                                              as_array=True))
        torch.cuda.synchronize()
        return total

    def parse_only():
        return sum(len(b) for b in bio.fasta_batches(p, batch_bytes=1 << 24, as_array=True))

    def parse_python():  # the reference's line loop (io.py:226-242)
        with open(p, "rb") as fh:
            return sum(len(r) for r in bio.fasta_records(fh))

    batches = list(bio.fasta_batches(p, batch_bytes=1 << 24, as_array=True))

    def insert_only():
        f = bb.Filter.from_config(cfg, insert_mode="relaxed")
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for batch in batches:
            f.insert_qgrams(enc, batch)
        torch.cuda.synchronize()
        return time.perf_counter() - t0

    t = wall(run)
    total = run()
    tp = wall(parse_only)
    tpy = wall(parse_python)
    insert_only()
    ti = min(insert_only() for _ in range(3))
    out({"row": "fasta", "workload": f"{nrec} records x {rec_len} bp -> fused canonical 31-mer insert",
         "bases_s": round(nrec * rec_len / t, 1), "kmers": total,
         "kmers_expected": nrec * (rec_len - 30),
         "parse_bases_s": round(nrec * rec_len / tp, 1),
         "cpu_reference_parse_bases_s": round(nrec * rec_len / tpy, 1),
         "insert_bases_s": round(nrec * rec_len / ti, 1),
         "file_bytes": os.path.getsize(p), "host_cores": os.cpu_count(),
         "parity": "identical" if total == nrec * (rec_len - 30) else "DIFF"})


def row_tsv(bb, torch, out):
    from paper_2501_18977_b200 import cli

    keys = bb.even_keys(1 << 23, 11)
    ans = (keys & np.uint64(1 << 20)).astype(bool).astype(np.uint8)
    t = wall(lambda: cli.format_answers(keys, ans))
    blob = cli.format_answers(keys, ans)
    m = 1 << 18

    def ref():
        return "".join(f"{k}\t{int(a)}\n" for k, a in zip(keys[:m].tolist(), ans[:m].tolist()))

    tr = wall(ref)
    ok = blob[: len(ref().encode())] == ref().encode()
    out({"row": "tsv", "workload": "2^23 (key, answer) lines", "mb_s": round(len(blob) / t / 1e6, 1),
         "cpu_reference_mb_s": round(len(ref()) / tr / 1e6, 1),
         "parity": "identical" if ok else "DIFF"})


def row_standard(bb, torch, out):
    n = 1 << 26
    f = bb.Filter.from_config(bb.FilterConfig(kind="standard", k=12, size_bits=12 * n, seed=1))
    keys = bb.even_keys(n, 11, device=f.device)
    q = torch.cat([keys[: n], bb.odd_keys(n, 12, device=f.device)])
    res = torch.empty(q.numel(), dtype=torch.uint8, device=f.device)

    def build():
        f.storage.d_words.zero_()
        f.insert_many(keys)

    ins = cuda_ms(build)
    look = cuda_ms(lambda: f.contains_many(q, out=res))
    fn = int((res[:n] == 0).sum().item())
    out({"row": "standard", "workload": "standard Bloom, k = 12, 12 b/key (96 MiB), 2^26 keys, "
         "2^27 lookups (50% positive)", "insert_mkeys_s": round(n / ins / 1e3, 1),
         "lookup_mkeys_s": round(2 * n / look / 1e3, 1), "false_negatives": fn,
         "fpr": float(res[n:].float().mean().item())})


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import torch

    import paper_2501_18977_b200 as bb

    lines = []

    def out(d):
        print(json.dumps(d), flush=True)
        lines.append(d)

    with tempfile.TemporaryDirectory() as tmp:
        row_hist(bb, torch, out)
        row_fpr(bb, torch, out)
        row_bwch(bb, torch, out, tmp)
        row_keys(bb, torch, out, tmp)
        row_fasta(bb, torch, out, tmp)
        row_tsv(bb, torch, out)
        row_standard(bb, torch, out)
    if args.out:
        with open(args.out, "w") as fh:
            fh.writelines(json.dumps(d) + "\n" for d in lines)


if __name__ == "__main__":
    main()
