"""One-GPU timing of the partitioned relaxed insert (bc_insert_peers) against
the plain relaxed insert on config 5: W replicas held on this GPU stand in for
the W ranks' replicas, every rank's launch issued in turn with its key slice
and its share of the M/2 keys in flight.  On one GPU every "remote" access is
local, so this measures the kernel's partition addressing and the in-flight
split, not NVLink.

    python tools/partition_probe.py [W ...]
"""
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_18977_b200 as bb  # noqa: E402
from paper_2501_18977_b200 import _native  # noqa: E402
from paper_2501_18977_b200.distributed import slice_bounds  # noqa: E402


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b))
    return sorted(out)[len(out) // 2]


def main():
    worlds = [int(a) for a in sys.argv[1:]] or [1, 2, 4, 8]
    cfg = bb.FilterConfig(kind="blowchoc", k=11, choices=2, size_bits=2**36, seed=1)
    n = int(1.2 * 2**32)
    keys = bb.even_keys(n, 11, device="cuda")
    f = bb.Filter.from_config(cfg, insert_mode="relaxed")

    def plain():
        f.storage.d_words.zero_()
        f.insert_many(keys)

    ms = timed(plain)
    print(json.dumps({"variant": "relaxed insert", "ms": round(ms, 2),
                      "mkeys_s": round(n / ms / 1e3, 1)}), flush=True)
    k64 = keys.view(torch.int64)
    stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    nw = f.storage.d_words.numel()
    for w in worlds:
        reps = [f.storage.d_words.view(torch.int64)] + [
            torch.zeros(nw, dtype=torch.int64, device="cuda") for _ in range(w - 1)]
        ptrs = (ctypes.c_uint64 * w)(*[r.data_ptr() for r in reps])
        share = max(256, (f.num_blocks // 2) // w)
        bounds = slice_bounds(n, w)

        def parted():
            for r in reps:
                r.zero_()
            for lo, hi in bounds:
                part = k64[lo:hi]
                _native.check(_native.lib().bc_insert_peers(
                    ctypes.c_void_p(f.handle), ptrs, w, ctypes.c_void_p(part.data_ptr()),
                    part.numel(), share, stream))

        ms = timed(parted)
        print(json.dumps({"variant": f"partitioned over {w} replicas on one GPU, ranks in turn",
                          "ms": round(ms, 2), "mkeys_s": round(n / ms / 1e3, 1)}), flush=True)
        del reps
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
