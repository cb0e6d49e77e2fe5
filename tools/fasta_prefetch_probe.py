import os, sys, time, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_2501_18977_b200 as bb
from paper_2501_18977_b200 import io as bio
rng = np.random.default_rng(3)
p = "/tmp/g.fa"; nrec, rec_len = 64, 1 << 20
with open(p, "wb") as fh:
    for r in range(nrec):
        seq = np.frombuffer(b"ACGT", dtype=np.uint8)[rng.integers(0, 4, rec_len)]
        fh.write(b">r%d\n" % r)
        for a in range(0, rec_len, 80): fh.write(seq[a:a + 80].tobytes() + b"\n")
enc = bb.QGramEncoder(q=31, canonical=True)
cfg = bb.FilterConfig(kind="blowchoc", k=14, choices=2, size_bits=14 * nrec * rec_len, seed=1)
def run(pf, bbytes):
    f = bb.Filter.from_config(cfg, insert_mode="relaxed")
    tot = 0
    for batch in bio.fasta_batches(p, batch_bytes=bbytes, as_array=True, prefetch=pf):
        tot += f.insert_qgrams(enc, batch)
    torch.cuda.synchronize()
    return tot
for bbytes in (1 << 24, 1 << 22):
  for pf in (0, 2, 0, 2, 4):
    run(pf, bbytes); t0 = time.perf_counter(); run(pf, bbytes); dt = time.perf_counter() - t0
    print("batch", bbytes, "prefetch", pf, round(nrec * rec_len / dt / 1e6, 1), "Mbp/s", flush=True)
