"""Time the exact-order (Filter default) insert of one BASELINE config on the
GPU and check its bits: cfg1 against the reference's golden digest, the
others against the fixture digests when given.

    python tools/ordered_probe.py [cfg ...]        (env knobs: BC_CLUSTER_*, BC_ORDERED_*)
"""
import hashlib
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_18977_b200 as bb  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))
CFGS = {
    1: (dict(kind="blowchoc", k=14, choices=2, size_bits=16 * 2**20, seed=1), 2**20,
        GOLD["cfg1"]["words_sha256"]),
    3: (dict(kind="blowchoc", k=16, choices=3, size_bits=16 * 2**28, seed=1), 2**28, None),
    5: (dict(kind="blowchoc", k=11, choices=2, size_bits=2**36, seed=1), int(1.2 * 2**32), None),
}


def spec(a: str):
    """A BASELINE config number, or bits:n:c:k for another geometry."""
    if ":" in a:
        bits, n, c, k = (int(v) for v in a.split(":"))
        return a, (dict(kind="blowchoc", k=k, choices=c, size_bits=bits, seed=1), n, None)
    return int(a), CFGS[int(a)]


def main():
    cfgs = [spec(a) for a in sys.argv[1:]] or [spec("1")]
    for c, (kw, n, want) in cfgs:
        if c == 3:
            want = json.load(open(os.path.join(ROOT, "tests/golden/fullsize_cfg3.json")))["words_sha256"]
        f = bb.Filter.from_config(bb.FilterConfig(**kw))
        keys = bb.even_keys(n, 11, device="cuda")
        reps = 10 if c == 1 else 3
        times = []
        for r in range(reps + 1):
            f.storage.d_words.zero_()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            f.insert_many(keys)
            b.record()
            torch.cuda.synchronize()
            if r:
                times.append(a.elapsed_time(b))
        h = hashlib.sha256()
        w = f.storage.d_words.view(torch.uint8)
        for i in range(0, w.numel(), 1 << 30):
            h.update(w[i:i + (1 << 30)].cpu().numpy().tobytes())
        ok = (h.hexdigest() == want) if want else None
        ms = sorted(times)[len(times) // 2]
        print(json.dumps({"config": c, "n": n, "ms_median": round(ms, 4),
                          "mkeys_s": round(n / ms / 1e3, 1), "bits_equal_reference": ok,
                          "env": {k: v for k, v in os.environ.items() if k.startswith("BC_")}}),
              flush=True)
        del f, keys
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
