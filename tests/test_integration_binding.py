"""CPU checks of the reference-side binding (integration/blowchoc_gpu.py):
the descriptor it derives from the reference's own ``_kernel_args()`` /
``_cost_args()`` tuples is the one the package derives from the same
configuration, and its struct mirrors ``bc_filter_desc``.  No GPU calls."""

import ctypes
import os
import sys

import numpy as np
import pytest

from integration import blowchoc_gpu as bg
from paper_2501_18977_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


def test_desc_layout_matches_package():
    assert ctypes.sizeof(bg.Desc) == ctypes.sizeof(_native.BcFilterDesc)
    for (n1, t1), (n2, t2) in zip(bg.Desc._fields_, _native.BcFilterDesc._fields_):
        assert n1 == n2 and ctypes.sizeof(t1) == ctypes.sizeof(t2)
        assert getattr(bg.Desc, n1).offset == getattr(_native.BcFilterDesc, n2).offset


def ref_blowchoc():
    if not os.path.isdir(os.path.join(REF, "blowchoc")):
        pytest.skip("reference not installed in baseline/_ref")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import blowchoc

    return blowchoc


CASES = [
    dict(kind="standard", k=7, n_capacity=1000, seed=3),
    dict(kind="blocked", k=7, n_capacity=1000, choices=1, seed=5),
    dict(kind="blowchoc", k=9, n_capacity=5000, choices=3, shards=4, seed=7),
    dict(kind="blowchoc", k=2, n_capacity=400, choices=2, strategy="distinct",
         block_bits=16, seed=9),
    dict(kind="blowchoc", k=14, size_bits=2**20, choices=2, seed=11,
         cost=("mix", 0.75)),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c['kind']}-{c.get('choices')}")
def test_binding_desc_equals_package_desc(case, monkeypatch):
    ref = ref_blowchoc()
    import paper_2501_18977_b200 as bb

    def cfg(mod):
        kw = dict(case)
        if "cost" in kw:
            kind, param = kw["cost"]
            kw["cost"] = mod.CostModel(kind=kind, param=param, k=kw["k"])
        return mod.FilterConfig(**kw)

    rf = ref.Filter.from_config(cfg(ref))
    of = bb.Filter.from_config(cfg(bb))  # keeps the desc's bit arrays alive
    ours = of._kernel_args()
    seen = {}

    def capture(kind, k, c, strategy, block_bits, num_blocks, shards, shard_a, block_a,
                bit_a, bit_b, cost_code=0, cost_param=0.0):
        seen.update(kind=kind, k=k, c=c, strategy=strategy, num_blocks=num_blocks,
                    shards=shards, shard_a=shard_a, block_a=[int(a) for a in block_a],
                    bit_a=np.asarray(bit_a).tolist(), block_bits=block_bits,
                    cost=(cost_code, cost_param), bits_total=num_blocks * block_bits)
        return 0

    monkeypatch.setattr(bg, "_handle", capture)
    args = rf._kernel_args()
    if rf.kind == "standard":
        bg._flat_handle(args[0], args[1])
        assert seen["bits_total"] == ours.num_blocks * ours.block_bits
    else:
        bg._blocks_handle(args, rf._cost_args()[:2])
        assert seen["num_blocks"] == ours.num_blocks and seen["shards"] == ours.shards
        assert seen["block_bits"] == ours.block_bits and seen["shard_a"] == ours.shard_a
        assert seen["block_a"] == [ours.block_a[i] for i in range(ours.choices)]
        if ours.choices >= 2:
            assert seen["cost"] == (ours.cost_code, ours.cost_param)
    assert (seen["kind"], seen["k"], seen["c"], seen["strategy"]) == \
        (ours.kind, ours.k, ours.choices, ours.strategy)
    assert seen["bit_a"] == [ours.bit_a[i] for i in range(ours.k)]
