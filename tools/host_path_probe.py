import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time, numpy as np, torch, paper_2501_18977_b200 as bb
n = 1 << 26
f = bb.Filter.from_config(bb.FilterConfig(kind="blocked", k=12, size_bits=12 * n, seed=1))
keys = bb.even_keys(n, 11)
q = np.concatenate([keys, bb.odd_keys(n, 12)])
for rep in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    f.insert_many(keys)
    t1 = time.perf_counter()
    a = f.contains_many(q)
    t2 = time.perf_counter()
    print(f"pageable: insert {n/(t1-t)/1e6:.0f} Mkeys/s ({8*n/(t1-t)/1e9:.1f} GB/s), lookup {2*n/(t2-t1)/1e6:.0f} Mkeys/s, step {(n+2*n)/(t2-t)/1e6:.0f} Mkeys/s")
pk = torch.empty(n, dtype=torch.uint64, pin_memory=True).numpy(); pk[:] = keys
pq = torch.empty(2*n, dtype=torch.uint64, pin_memory=True).numpy(); pq[:] = q
po = torch.empty(2*n, dtype=torch.uint8, pin_memory=True).numpy()
for rep in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    f.insert_many(pk)
    t1 = time.perf_counter()
    f.contains_many(pq, out=po)
    t2 = time.perf_counter()
    print(f"pinned:   insert {n/(t1-t)/1e6:.0f} Mkeys/s, lookup {2*n/(t2-t1)/1e6:.0f} Mkeys/s, step {(n+2*n)/(t2-t)/1e6:.0f} Mkeys/s")
