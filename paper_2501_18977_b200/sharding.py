"""Shard geometry and builds (reference sharding.py:1-136).

The reference splits the bit array into ``shards`` sub-arrays, routes every
key with the shard hash h0, and runs one writer thread per shard so each
shard sees its keys in stream order.  On a GPU the whole stream is inserted
by one launch sequence that already preserves every shard's stream order
(ordered mode) -- so ``build_sharded`` is bit-identical to
``build_sequential`` here too, with the dispatcher and FIFOs gone.  Across
GPUs, shards map to devices (``distributed.build_subfilters``).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Iterable

import numpy as np

from .filters import Filter, FilterConfig
from .hashing import HashSpec, eval_hash, eval_hash_many

BATCH_KEYS = 1024
QUEUE_CAPACITY = 1 << 16


@dataclass(frozen=True)
class ShardPlan:
    shards: int
    blocks_per_shard: int
    h0: HashSpec
    queue_capacity: int = QUEUE_CAPACITY

    @classmethod
    def for_filter(cls, filt: Filter) -> "ShardPlan":
        return cls(shards=filt.shards, blocks_per_shard=filt.blocks_per_shard,
                   h0=filt.shard_spec)

    def owner_range(self, rank: int, world: int) -> tuple:
        """Contiguous shard range [lo, hi) owned by ``rank`` of ``world``."""
        if self.shards % world != 0:
            raise ValueError(f"{self.shards} shards do not split over {world} devices")
        per = self.shards // world
        return rank * per, (rank + 1) * per


def route(plan: ShardPlan, x: int) -> int:
    return eval_hash(plan.h0, x)


def route_many(plan: ShardPlan, keys):
    """Shard per key, on the GPU."""
    return eval_hash_many(plan.h0, keys)


def _chunks(keys) -> Iterable:
    if hasattr(keys, "shape"):
        yield keys
        return
    yield from keys


def build_sequential(config: FilterConfig, keys, **kw) -> Filter:
    filt = Filter.from_config(config, **kw)
    for chunk in _chunks(keys):
        filt.insert_many(chunk)
    return filt


def build_sharded(config: FilterConfig, keys, *, parallel: bool | None = None,
                  reader_thread: bool = False, queue_capacity: int = QUEUE_CAPACITY,
                  **kw) -> Filter:
    """Same bits as ``build_sequential`` (sharding.py:1-9).  ``parallel``,
    ``reader_thread`` and ``queue_capacity`` are accepted for API
    compatibility; on the GPU every shard is written concurrently anyway."""
    del parallel, reader_thread, queue_capacity
    return build_sequential(config.validated(), keys, **kw)


def partition_by_shard(keys: np.ndarray, shard_of: np.ndarray, shards: int) -> list:
    """Stable per-shard split of a host key chunk (the dispatcher's
    partition, sharding.py:121-125): order within each shard is kept."""
    order = np.argsort(shard_of, kind="stable")
    bounds = np.searchsorted(shard_of[order], np.arange(shards + 1))
    return [keys[order[bounds[s]:bounds[s + 1]]] for s in range(shards)]
