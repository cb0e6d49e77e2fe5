"""Dependency depth of an exact-order (stream-order) build: the longest chain
of keys in which each key shares a candidate block with the previous one.
This is the critical path of the ticket dataflow (ordered_ticket.cu) and a
lower bound on the claim rounds of ordered512_kernel, whatever the window.
Block indices are drawn uniformly (the hash family makes them so).

    python tools/chain_depth.py M n c        (config 1: 32768 1048576 2 -> 274)
"""
import sys

import numpy as np


def depth(M: int, n: int, c: int, seed: int = 1) -> int:
    rng = np.random.default_rng(seed)
    bl = rng.integers(0, M, size=(n, c))
    last = np.zeros(M, dtype=np.int64)  # depth of the latest key on each block
    d = 0
    for row in bl:
        v = 1 + int(last[row].max())
        last[row] = v
        d = max(d, v)
    return d


if __name__ == "__main__":
    M, n, c = (int(a) for a in sys.argv[1:4])
    print(f"M={M} n={n} c={c}: chain depth {depth(M, n, c)}")
