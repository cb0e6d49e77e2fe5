"""Multi-GPU layer: one process per GPU, torch.distributed (NCCL) plumbing.

Two data-parallel patterns, both from the reference's own parallel design
(sharding.py:1-136, analysis.py:96-107):

* **Lookups shard by key over replicas.**  Every rank holds a full copy of
  the bit array (NCCL broadcast from the rank that built it); a key batch is
  split into contiguous per-rank slices, each rank answers its slice with
  the lookup kernel, and answers are all-gathered (or hit counts
  all-reduced).  The lookup itself has no communication, so it scales with
  the number of GPUs; the one-time broadcast is reported separately.

* **Order-free builds (one choice, standard) split the keys.**  Each rank
  ORs a contiguous slice of the stream into its replica, then the replicas
  are OR-all-reduced (``or_allreduce_words``); the result is the sequential
  bit array because OR commutes.

* **Multi-choice inserts go to hash-partitioned subfilters only where the
  reference's layout has them** (``shards = T > 1``).  Shard s owns words
  [s*wps, (s+1)*wps); rank r owns the contiguous shard range
  [r*T/W, (r+1)*T/W).  Keys are routed with the shard hash h0 on the
  device; each rank inserts, in stream order, the keys of its shards only
  (so ordered builds stay bit-identical to the reference's sequential
  build, sharding.py:1-9), then an all-gather of the W contiguous word
  ranges replicates the filter.  With T = 1 and c >= 2 rank 0 builds and
  broadcasts.

Every collective acts on the filter's word tensor; no collective runs inside
a lookup or insert kernel.  The functions only use the filter's public
interface (``route_many``, ``insert_many``, ``contains_many``,
``count_hits``, ``storage.d_words``), so the orchestration is tested on CPU
with gloo and the oracle standing in for the kernels.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np
import torch
import torch.distributed as dist


def _rank_world(group):
    return dist.get_rank(group), dist.get_world_size(group)


def _words_i64(filt) -> torch.Tensor:
    return filt.storage.d_words.view(torch.int64)


def slice_bounds(n: int, world: int) -> list:
    """Contiguous [lo, hi) per rank (np.array_split sizing, analysis.py:103)."""
    base, extra = divmod(n, world)
    bounds, lo = [], 0
    for r in range(world):
        hi = lo + base + (1 if r < extra else 0)
        bounds.append((lo, hi))
        lo = hi
    return bounds


def broadcast_filter(filt, src: int = 0, group=None) -> None:
    """Replicate the bit array (and the inserted-key count) from ``src``."""
    dist.broadcast(_words_i64(filt), src=src, group=group)
    meta = torch.tensor([filt.inserted], dtype=torch.int64,
                        device=filt.storage.d_words.device)
    dist.broadcast(meta, src=src, group=group)
    filt.inserted = int(meta.item())
    filt.storage.device_modified()


def _local_slice(keys, group):
    rank, world = _rank_world(group)
    lo, hi = slice_bounds(len(keys), world)[rank]
    return keys[lo:hi], lo, hi


def contains_many_sharded(filt, keys, group=None, gather: bool = True):
    """Key-sharded lookup on replicated filters.  ``keys`` is the full batch
    (identical on every rank); each rank answers its contiguous slice.
    Returns the full answer array on every rank (``gather``), else this
    rank's slice."""
    rank, world = _rank_world(group)
    part, lo, hi = _local_slice(keys, group)
    ans = filt.contains_many(part)
    if not gather or world == 1:
        return ans
    dev = filt.storage.d_words.device
    bounds = slice_bounds(len(keys), world)
    width = max(h - l for l, h in bounds)
    local = torch.zeros(width, dtype=torch.uint8, device=dev)
    a = torch.as_tensor(np.asarray(ans) if not isinstance(ans, torch.Tensor) else ans)
    local[: hi - lo] = a.to(device=dev, dtype=torch.uint8)
    outs = [torch.empty(width, dtype=torch.uint8, device=dev) for _ in range(world)]
    dist.all_gather(outs, local, group=group)
    full = torch.cat([o[: h - l] for o, (l, h) in zip(outs, bounds)]).bool()
    return full if isinstance(keys, torch.Tensor) and keys.is_cuda else full.cpu().numpy()


def count_hits_sharded(filt, keys, group=None) -> int:
    """Hits over the whole batch: per-rank count + all-reduce(sum)."""
    part, _, _ = _local_slice(keys, group)
    hits = torch.tensor([filt.count_hits(part)], dtype=torch.int64,
                        device=filt.storage.d_words.device)
    dist.all_reduce(hits, group=group)
    return int(hits.item())


def _as_numpy_u64(keys) -> np.ndarray:
    if isinstance(keys, torch.Tensor):
        return keys.detach().cpu().view(torch.uint64).numpy() if keys.dtype == torch.int64 \
            else keys.detach().cpu().numpy().astype(np.uint64)
    return np.ascontiguousarray(keys, dtype=np.uint64)


def owned_keys(filt, keys, rank: int, world: int):
    """The keys of ``keys`` whose shard rank ``rank`` owns, in stream order."""
    if filt.shards % world != 0:
        raise ValueError(f"{filt.shards} shards do not split over {world} ranks")
    per = filt.shards // world
    shard = filt.route_many(keys)
    if isinstance(shard, torch.Tensor):
        # torch has no compare / index kernels for uint64: work on int64 views
        shard = shard.view(torch.int64)  # shard ids < T, no sign issue
        sel = (shard >= rank * per) & (shard < (rank + 1) * per)
        k64 = keys.view(torch.int64) if keys.dtype == torch.uint64 else keys
        return k64[sel]
    shard = np.asarray(shard)
    sel = (shard >= rank * per) & (shard < (rank + 1) * per)
    return np.asarray(keys)[sel]


def gather_subfilters(filt, group=None) -> None:
    """All-gather the W contiguous shard ranges so every rank holds the
    whole bit array."""
    rank, world = _rank_world(group)
    words = _words_i64(filt)
    span = words.numel() // world
    mine = words[rank * span:(rank + 1) * span].clone()
    parts = [words[r * span:(r + 1) * span] for r in range(world)]
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(words, mine, group=group)
    else:
        outs = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(outs, mine, group=group)
        for p, o in zip(parts, outs):
            p.copy_(o)
    counts = torch.tensor([filt.inserted], dtype=torch.int64, device=words.device)
    dist.all_reduce(counts, group=group)
    filt.inserted = int(counts.item())
    filt.storage.device_modified()


# -- replica merge over peer memory ------------------------------------------------------

def _peer_mode() -> int:
    """BC_PEER_ALLREDUCE: 0 never, 1 always (any backend, e.g. gloo ranks
    sharing a GPU in tests), unset: NCCL groups whose GPUs reach each other."""
    v = os.environ.get("BC_PEER_ALLREDUCE")
    return -1 if v is None else int(v)


# (id(group), ptr, numel) -> PeerReplicas (successful mappings only).  An
# entry holds no reference to the replica tensor (an 8 GiB filter must not be
# kept alive by a cache); whether it may be reused is decided collectively
# and re-validated against the allocation's current IPC handle (see
# _peer_replicas).
_PEER_CACHE: dict = {}
_IPC_OPEN: dict = {}  # peer allocation handle -> [base address here, users]


class PeerReplicas:
    """The ranks' replicas of one word tensor, mapped into this process
    (CUDA IPC; lazy peer access over NVLink)."""

    def __init__(self, words: torch.Tensor, rank: int, ptrs: list, own: tuple, peers: list):
        self.world, self.rank, self.nwords = len(ptrs), rank, words.numel()
        self.ptrs = (ctypes.c_uint64 * len(ptrs))(*ptrs)
        self.own = own        # this rank's (handle, offset) when the mapping was made
        self.peers = peers    # imported handles (released in close())

    def or_allreduce(self, stream) -> None:
        from . import _native

        _native.check(_native.lib().bc_or_allreduce_peers(
            self.ptrs, self.world, self.rank, self.nwords, ctypes.c_void_p(stream)))

    def close(self) -> None:
        _release(self.peers)
        self.peers = []


def _export(words: torch.Tensor):
    """(IPC handle bytes, offset) of this rank's replica, or None."""
    from . import _native

    try:
        handle = (ctypes.c_ubyte * 64)()
        off = ctypes.c_uint64()
        _native.check(_native.lib().bc_ipc_export(ctypes.c_void_p(words.data_ptr()), handle,
                                                  ctypes.byref(off)))
        return bytes(handle), off.value
    except (RuntimeError, ValueError, MemoryError):
        return None


def _release(handles: list) -> None:
    """Drop one use of each imported peer allocation; unmap at zero."""
    from . import _native

    for h in handles:
        ent = _IPC_OPEN.get(h)
        if ent is None:
            continue
        ent[1] -= 1
        if ent[1] <= 0:
            del _IPC_OPEN[h]
            try:
                _native.check(_native.lib().bc_ipc_close(ctypes.c_void_p(ent[0]), 0))
            except (RuntimeError, ValueError):
                pass


def _import(infos: list, rank: int, words: torch.Tensor):
    """(this process's addresses of every rank's replica, imported handles),
    or None."""
    from . import _native

    ptrs, used = [], []
    try:
        for j, (h, o) in enumerate(infos):
            if j == rank:
                ptrs.append(words.data_ptr())
                continue
            if h not in _IPC_OPEN:
                base = ctypes.c_void_p()
                _native.check(_native.lib().bc_ipc_import(h, 0, ctypes.byref(base)))
                _IPC_OPEN[h] = [base.value, 0]
            _IPC_OPEN[h][1] += 1
            used.append(h)
            ptrs.append(_IPC_OPEN[h][0] + o)
    except (RuntimeError, ValueError, MemoryError):
        _release(used)
        return None
    return ptrs, used


def _peer_replicas(words: torch.Tensor, group):
    """PeerReplicas when every rank can map every other rank's replica, else
    None.  Every rank runs the same collectives in the same order whatever
    fails locally, and every decision is the AND over ranks: a cached mapping
    is reused only if, on every rank, it exists and this replica still lives
    in the allocation (IPC handle and offset) the mapping was made for --
    address reuse after a free, on some ranks only, therefore rebuilds the
    mapping on all of them instead of splitting the ranks between two code
    paths."""
    mode = _peer_mode()
    if mode == 0 or not words.is_cuda or not words.is_contiguous():
        return None
    if mode != 1 and dist.get_backend(group) != "nccl":
        return None
    rank, world = _rank_world(group)

    def agree(local):
        out = [None] * world
        dist.all_gather_object(out, local, group=group)
        return out

    key = (id(group), words.data_ptr(), words.numel())
    own = _export(words)
    cached = _PEER_CACHE.get(key)
    if all(agree(cached is not None and own is not None and cached.own == own)):
        return cached
    if cached is not None:
        cached.close()
        del _PEER_CACHE[key]
    dev = words.device.index
    devs = agree(dev)
    ok = own is not None and words.data_ptr() % 16 == 0 and world <= 16 and all(
        d == dev or torch.cuda.can_device_access_peer(dev, d) for d in devs)
    if not all(agree(bool(ok))):
        return None
    infos = agree(own)
    imp = _import(infos, rank, words)
    if not all(agree(imp is not None)):
        if imp is not None:
            _release(imp[1])
        return None
    reps = PeerReplicas(words, rank, imp[0], own, imp[1])
    _PEER_CACHE[key] = reps
    return reps


def _device_barrier(group, device) -> None:
    """Every rank's earlier work on its current stream is finished before
    anything after this runs on any rank: a one-element NCCL all-reduce on
    the stream, or (other backends) a host sync plus a barrier."""
    if dist.get_backend(group) == "nccl":
        dist.all_reduce(torch.zeros(1, device=device), group=group)
    else:
        torch.cuda.synchronize(device)
        dist.barrier(group=group)


def or_allreduce_peer_(words: torch.Tensor, reps: PeerReplicas, group=None) -> torch.Tensor:
    """OR all-reduce through peer memory: each rank's single kernel ORs its
    word range over all replicas and writes it back into all of them
    (bc_or_allreduce_peers), between two cross-rank barriers."""
    _device_barrier(group, words.device)
    reps.or_allreduce(torch.cuda.current_stream(words.device).cuda_stream)
    _device_barrier(group, words.device)
    return words


def or_allreduce_(words: torch.Tensor, group=None) -> torch.Tensor:
    """In-place bitwise-OR all-reduce of an int64 word tensor.

    GPUs that reach each other's memory (NVLink / NVSwitch) use one peer-memory
    kernel per rank (or_allreduce_peer_).  Otherwise, since NCCL has no OR
    reduction: an all-to-all of W equal word ranges (the reduce-scatter
    layout), an OR fold of the W pieces each rank received, and an all-gather
    of the folded ranges.  Every rank moves 2 (W-1)/W of the array either way,
    like a ring all-reduce.  Stream-ordered, no host synchronisation."""
    rank, world = _rank_world(group)
    if world == 1:
        return words
    reps = _peer_replicas(words, group)
    if reps is not None:
        return or_allreduce_peer_(words, reps, group)
    n = words.numel()
    span = -(-n // world)
    pad = span * world - n
    src = words if pad == 0 else torch.cat([words, words.new_zeros(pad)])
    recv = torch.empty_like(src)
    dist.all_to_all_single(recv, src, group=group)
    pieces = recv.view(world, span)  # piece j: rank j's words of range `rank`
    acc = pieces[0].clone()
    for j in range(1, world):
        acc.bitwise_or_(pieces[j])
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(src, acc, group=group)
    else:
        outs = [torch.empty_like(acc) for _ in range(world)]
        dist.all_gather(outs, acc, group=group)
        torch.cat(outs, out=src)
    if pad:
        words.copy_(src[:n])
    return words


def or_allreduce_words(filt, group=None) -> None:
    """OR all-reduce of the ranks' bit arrays (or_allreduce_) and the sum of
    their inserted-key counts."""
    words = _words_i64(filt)
    or_allreduce_(words, group=group)
    counts = torch.tensor([filt.inserted], dtype=torch.int64, device=words.device)
    dist.all_reduce(counts, group=group)
    filt.inserted = int(counts.item())
    filt.storage.device_modified()


def order_free(filt) -> bool:
    """Inserts commute (one choice, or the standard kind): the bit array is
    the OR of the keys' masks whatever the order (_kernels.py:142-147,221)."""
    return filt.kind in ("blocked", "standard")


def build_subfilters(filt, keys, group=None, mode: str | None = None):
    """Insert a key stream (identical on every rank) into ``filt``.

    ``shards > 1``: each rank inserts the keys of its shard range (device
    routing, no data exchange), then the ranges are all-gathered.
    ``shards == 1``, order-free kinds: each rank inserts a contiguous slice
    into its replica, then the replicas are OR-all-reduced.
    ``shards == 1``, c >= 2: rank 0 inserts everything, then broadcasts."""
    rank, world = _rank_world(group)
    if filt.shards == 1 and world > 1 and order_free(filt):
        part, _, _ = _local_slice(keys, group)
        before = filt.inserted
        filt.insert_many(part, mode=mode) if mode else filt.insert_many(part)
        filt.inserted -= before  # this rank's share; summed by the all-reduce
        or_allreduce_words(filt, group=group)
        filt.inserted += before
        return filt
    if filt.shards == 1 or world == 1:
        if rank == 0:
            filt.insert_many(keys, mode=mode) if mode else filt.insert_many(keys)
        if world > 1:
            broadcast_filter(filt, src=0, group=group)
        return filt
    mine = owned_keys(filt, keys, rank, world)
    before = filt.inserted
    filt.insert_many(mine, mode=mode) if mode else filt.insert_many(mine)
    filt.inserted = filt.inserted - before  # this rank's share; summed below
    gather_subfilters(filt, group=group)
    filt.inserted += before
    return filt


# -- partitioned multi-choice build over peer memory ----------------------------------

def partitionable(filt) -> bool:
    """Filters the partitioned relaxed build covers (bc_insert_peers): one
    shard, 2..4 choices, 512-bit blocks, random bit strategy."""
    return (filt.kind == "blowchoc" and 2 <= filt.choices <= 4 and filt.block_bits == 512
            and filt.strategy == "random" and filt.shards == 1)


def part_ranges(num_blocks: int, world: int) -> list:
    """Word ranges [lo, hi) of the ranks' partitions: rank r owns blocks
    [r*per, (r+1)*per), per = ceil(M / W) (the kernel's split)."""
    per = -(-num_blocks // world)
    return [(min(num_blocks, r * per) * 8, min(num_blocks, (r + 1) * per) * 8)
            for r in range(world)]


def peer_map(filt, group=None):
    """The ranks' replicas of ``filt`` mapped into this process (collective;
    None on every rank when any rank cannot map them)."""
    return _peer_replicas(_words_i64(filt), group)


def build_partitioned(filt, keys, group=None, reps=None) -> bool:
    """Relaxed multi-choice build spread over the GPUs, for T = 1 filters
    the reference builds on one writer (c >= 2).

    Every rank inserts its contiguous slice of the stream (``keys`` is the
    whole stream, identical on every rank) into ONE filter partitioned over
    the ranks' replicas: block b lives in the replica of rank b / per, and
    each key's candidate reads and its RED go there, over NVLink when remote
    (one ``bc_insert_peers`` kernel per rank, between two cross-rank
    barriers).  The ranks' keys in flight add up to M/2, the bound the relaxed
    tolerance is stated for, so the result is a relaxed build like the
    single-GPU one.  The owners' ranges are then broadcast so every rank
    holds the whole filter.  Replaces rank-0 build + broadcast, which leaves
    W - 1 GPUs idle during the build.

    Returns False, having done nothing, when the replicas cannot be mapped
    (the decision is collective), so the caller can fall back to
    ``build_subfilters``."""
    from . import _native

    rank, world = _rank_world(group)
    if not partitionable(filt):
        raise ValueError("partitioned builds need T = 1, 2..4 choices, 512-bit random blocks")
    words = _words_i64(filt)
    if reps is None:
        reps = peer_map(filt, group)
    if reps is None:
        return False
    dev = words.device
    part, lo, hi = _local_slice(keys, group)
    if not isinstance(part, torch.Tensor):
        part = torch.from_numpy(np.ascontiguousarray(part, dtype=np.uint64).view(np.int64))
    part = part.to(dev).contiguous()
    share = max(256, (filt.num_blocks // 2) // world)
    _device_barrier(group, dev)  # every replica holds the filter before any remote write
    stream = torch.cuda.current_stream(dev).cuda_stream
    _native.check(_native.lib().bc_insert_peers(
        ctypes.c_void_p(filt.handle), reps.ptrs, world, ctypes.c_void_p(part.data_ptr()),
        part.numel(), share, ctypes.c_void_p(stream)))
    _device_barrier(group, dev)  # every rank's inserts are in
    for r, (a, b) in enumerate(part_ranges(filt.num_blocks, world)):
        if b > a:
            dist.broadcast(words[a:b], src=r, group=group)
    filt.inserted += len(keys)
    filt.storage.device_modified()
    return True


def exchange_by_shard(filt, local_keys, group=None):
    """Route a rank-local slice of the stream to the shard owners
    (all-to-all).  Rank r is assumed to hold the r-th contiguous part of the
    stream; received pieces are concatenated in source-rank order, which
    keeps every shard's stream order."""
    rank, world = _rank_world(group)
    per = filt.shards // world
    keys = _as_numpy_u64(local_keys)
    shard = np.asarray(filt.route_many(keys))
    owner = shard // per
    order = np.argsort(owner, kind="stable")
    send = torch.from_numpy(keys[order].view(np.int64).copy())
    send_counts = np.bincount(owner, minlength=world).astype(np.int64)
    dev = filt.storage.d_words.device
    sc = torch.from_numpy(send_counts).to(dev)
    rc = torch.empty_like(sc)
    dist.all_to_all_single(rc, sc, group=group)
    recv_counts = rc.cpu().numpy()
    recv = torch.empty(int(recv_counts.sum()), dtype=torch.int64, device=dev)
    dist.all_to_all_single(recv, send.to(dev), output_split_sizes=recv_counts.tolist(),
                           input_split_sizes=send_counts.tolist(), group=group)
    return recv.view(torch.uint64) if dev.type == "cuda" else recv.numpy().view(np.uint64)
