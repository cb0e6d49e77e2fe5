"""cfg3 relaxed insert, one timed build (a target for tools/r2_ncu_app.sh)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_18977_b200 as bb  # noqa: E402
f = bb.Filter.from_config(bb.FilterConfig(kind="blowchoc", k=16, choices=3, size_bits=16 * 2**28, seed=1))
keys = bb.even_keys(2**28, 11, device="cuda")
for _ in range(2):
    f.storage.d_words.zero_()
    f.insert_many(keys, mode="relaxed")
torch.cuda.synchronize()
print("done")
