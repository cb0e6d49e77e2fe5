"""Exact-order inserts in small batches into a large filter (cfg5 geometry):
median time per insert_many call by batch size.

    python tools/small_batch_probe.py
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_18977_b200 as bb  # noqa: E402


def main():
    f = bb.Filter.from_config(bb.FilterConfig(kind="blowchoc", k=11, choices=2,
                                              size_bits=2**36, seed=1))
    keys = bb.even_keys(1 << 24, 11, device="cuda")
    for lg in (10, 14, 16, 18, 20, 22):
        n = 1 << lg
        calls = min(64, keys.numel() // n)
        times = []
        for i in range(calls):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            f.insert_many(keys[i * n:(i + 1) * n])
            b.record()
            torch.cuda.synchronize()
            times.append(a.elapsed_time(b))
        us = sorted(times)[len(times) // 2] * 1e3
        print(json.dumps({"batch": n, "calls": calls, "us_per_call": round(us, 1),
                          "mkeys_s": round(n / us, 1)}), flush=True)


if __name__ == "__main__":
    main()
