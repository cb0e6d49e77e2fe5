"""Multi-process (gloo, world_size 2, CPU) tests of the multi-GPU orchestration
in paper_2501_18977_b200.distributed.  The per-rank kernels are replaced by
the CPU oracle through the same duck-typed filter interface, so what is
tested is the partitioning, routing and collectives."""

import os
import socket
from types import SimpleNamespace

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as orc


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def np_hash(a: int, b: int, keys: np.ndarray) -> np.ndarray:
    """hashing.py:90-100 restated in numpy (test-side)."""
    ax = np.uint64(a) * keys
    mode, s = orc.hash_branch(b)
    if mode == 1:
        return (ax >> np.uint64(s)) % np.uint64(b)
    if mode == 2:
        ax = ax ^ (ax >> np.uint64(s))
    return ax % np.uint64(b)


class OracleFilter:
    """The filter interface distributed.py relies on, backed by the oracle."""

    def __init__(self, **kw):
        self.o = orc.make_filter(**kw)
        self.kind = kw["kind"]
        self.shards = self.o.shards
        self.inserted = 0
        self.storage = SimpleNamespace(d_words=torch.from_numpy(self.o.words),
                                       device_modified=lambda: None)

    def route_many(self, keys):
        return np_hash(self.o.shard_a, self.shards, np.asarray(keys, dtype=np.uint64))

    def insert_many(self, keys, mode=None):
        keys = np.asarray(keys, dtype=np.uint64)
        self.o.insert_many(keys)
        self.inserted += keys.shape[0]

    def contains_many(self, keys):
        return self.o.contains_many(np.asarray(keys, dtype=np.uint64))

    def count_hits(self, keys):
        return int(self.contains_many(keys).sum())


CFG = dict(kind="blowchoc", k=7, choices=2, n_capacity=20_000, shards=4, seed=17)


def _worker(rank, world, port, case):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2501_18977_b200 import distributed as D

        keys = orc.even_keys(20_000, 5)
        ref = orc.make_filter(**CFG)
        ref.insert_many(keys)
        if case == "subfilters":
            f = OracleFilter(**CFG)
            D.build_subfilters(f, keys)
            assert np.array_equal(f.o.words, ref.words)
            assert f.inserted == keys.shape[0]
        elif case == "broadcast":
            cfg1 = dict(CFG, shards=1)
            ref1 = orc.make_filter(**cfg1)
            ref1.insert_many(keys)
            f = OracleFilter(**cfg1)
            D.build_subfilters(f, keys)
            assert np.array_equal(f.o.words, ref1.words)
        elif case == "lookups":
            f = OracleFilter(**CFG)
            if rank == 0:
                f.insert_many(keys)
            D.broadcast_filter(f, src=0)
            probes = np.concatenate([keys[:5000], orc.odd_keys(7001, 9)])
            full = D.contains_many_sharded(f, probes)
            assert np.array_equal(full, ref.contains_many(probes))
            assert D.count_hits_sharded(f, probes) == int(ref.contains_many(probes).sum())
        elif case == "exchange":
            f = OracleFilter(**CFG)
            lo, hi = D.slice_bounds(keys.shape[0], world)[rank]
            mine = D.exchange_by_shard(f, keys[lo:hi])
            per = f.shards // world
            assert np.all(np.asarray(f.route_many(mine)) // per == rank)
            f.insert_many(mine)
            f.inserted = int(np.asarray(mine).shape[0])
            D.gather_subfilters(f)
            assert np.array_equal(f.o.words, ref.words)
            assert f.inserted == keys.shape[0]
        elif case in ("or_blocked", "or_standard"):
            kind = case[3:]
            cfg = dict(kind=kind, k=9, n_capacity=30_001, seed=23,
                       **({"block_bits": 512} if kind == "blocked" else {}))
            ref2 = orc.make_filter(**cfg)
            ref2.insert_many(keys)
            f = OracleFilter(**cfg)
            D.build_subfilters(f, keys)
            assert np.array_equal(f.o.words, ref2.words)
            assert f.inserted == keys.shape[0]
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", ["subfilters", "broadcast", "lookups", "exchange",
                                  "or_blocked", "or_standard"])
def test_two_rank_gloo(case):
    mp.spawn(_worker, args=(2, free_port(), case), nprocs=2, join=True)


def test_three_rank_or_build_with_padding():
    """OR all-reduce when the word count does not split evenly over ranks."""
    mp.spawn(_worker, args=(3, free_port(), "or_blocked"), nprocs=3, join=True)


def test_slice_bounds_cover():
    from paper_2501_18977_b200.distributed import slice_bounds

    for n in (0, 1, 7, 100, 2**20 + 3):
        for w in (1, 2, 3, 8):
            b = slice_bounds(n, w)
            assert b[0][0] == 0 and b[-1][1] == n
            assert all(b[i][1] == b[i + 1][0] for i in range(w - 1))
            assert max(h - l for l, h in b) - min(h - l for l, h in b) <= 1


def _nccl_worker(rank, world, port):
    import torch

    import paper_2501_18977_b200 as bb
    from paper_2501_18977_b200 import distributed as D

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device("cuda", rank))
    try:
        cfg = bb.FilterConfig(kind="blowchoc", k=7, choices=2, n_capacity=20_000, shards=4,
                              seed=17)
        keys = bb.even_keys(20_000, 5)
        f = bb.Filter.from_config(cfg)
        mine = D.owned_keys(f, torch.from_numpy(keys).cuda(), rank, world)
        f.insert_many(mine)
        D.gather_subfilters(f)
        ref = orc.make_filter(**CFG)
        ref.insert_many(keys)
        assert np.array_equal(f.storage.words, ref.words)
        D.broadcast_filter(f, src=0)
        probes = np.concatenate([keys[:5000], orc.odd_keys(7001, 9)])
        assert np.array_equal(D.contains_many_sharded(f, probes), ref.contains_many(probes))
        assert D.count_hits_sharded(f, probes) == int(ref.contains_many(probes).sum())
        # order-free build from key slices + OR all-reduce
        g = bb.Filter.from_config(bb.FilterConfig(kind="blocked", k=9, n_capacity=30_001,
                                                  seed=23))
        D.build_subfilters(g, torch.from_numpy(keys).cuda())
        ref2 = orc.make_filter(kind="blocked", k=9, n_capacity=30_001, seed=23)
        ref2.insert_many(keys)
        assert np.array_equal(g.storage.words, ref2.words)
        assert g.inserted == keys.shape[0]
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_nccl_collectives_on_device():
    """The NCCL code paths (all_gather_into_tensor of subfilter ranges,
    broadcast, key-sharded lookups) on the GPUs present (world = #GPUs)."""
    import torch

    world = torch.cuda.device_count()
    if 4 % world:  # the test filter has 4 shards
        world = 1
    mp.spawn(_nccl_worker, args=(world, free_port()), nprocs=world, join=True)


@pytest.mark.gpu
@pytest.mark.parametrize("world,nwords", [(2, 1 << 16), (3, 1 << 16), (4, 12_345), (5, 999),
                                          (8, (1 << 20) + 7), (1, 33)])
def test_peer_or_kernel_emulated_ranks(world, nwords):
    """bc_or_allreduce_peers over W replicas held on one GPU (the ranks
    emulated in one process, each rank's call launched in turn): every
    replica ends up as the OR of all of them, odd tails included."""
    import ctypes

    import torch

    from paper_2501_18977_b200 import _native

    L = _native.lib()
    g = torch.Generator(device="cuda").manual_seed(world * 1000 + nwords)
    reps = [torch.randint(-2**63, 2**63 - 1, (nwords,), dtype=torch.int64, device="cuda",
                          generator=g) for _ in range(world)]
    want = reps[0].clone()
    for r in reps[1:]:
        want |= r
    ptrs = (ctypes.c_uint64 * world)(*[r.data_ptr() for r in reps])
    stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    for rank in range(world):
        _native.check(L.bc_or_allreduce_peers(ptrs, world, rank, nwords, stream))
    torch.cuda.synchronize()
    for r in reps:
        assert torch.equal(r, want)
    span = ctypes.c_uint64()
    _native.check(L.bc_peer_span(nwords, world, ctypes.byref(span)))
    assert span.value % 32 == 0 and span.value * world >= nwords
    with pytest.raises(ValueError):
        _native.check(L.bc_or_allreduce_peers(ptrs, world, world, nwords, stream))


def _peer_worker(rank, world, port):
    import torch

    import paper_2501_18977_b200 as bb
    from paper_2501_18977_b200 import distributed as D

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["BC_PEER_ALLREDUCE"] = "1"
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        for kind, k, n in (("blocked", 9, 30_001), ("standard", 5, 12_345)):
            cfg = bb.FilterConfig(kind=kind, k=k, n_capacity=n, seed=23)
            keys = bb.even_keys(n, 3)
            # an allocation ahead of the words, so they sit at an offset inside
            # the caching allocator's segment
            pad = torch.empty(1000 + 77 * rank, dtype=torch.uint8, device="cuda")
            f = bb.Filter.from_config(cfg)
            D.build_subfilters(f, torch.from_numpy(keys).cuda())
            assert D._peer_replicas(D._words_i64(f), None) is not None
            ref = orc.make_filter(kind=kind, k=k, n_capacity=n, seed=23)
            ref.insert_many(keys)
            assert np.array_equal(f.storage.words, ref.words)
            assert f.inserted == n
            # a second merge reuses the mappings and changes nothing
            D.or_allreduce_(D._words_i64(f))
            f.storage.device_modified()
            assert np.array_equal(f.storage.words, ref.words)
            del pad
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_peer_or_allreduce_two_processes_one_gpu():
    """The peer-memory merge end to end: two ranks (gloo barriers) sharing
    cuda:0 exchange CUDA IPC handles of their replicas, each runs its one
    merge kernel, and both hold the sequential build.  No kernel waits on the
    other rank (the barriers are on the host)."""
    mp.spawn(_peer_worker, args=(2, free_port()), nprocs=2, join=True)


# -- partitioned multi-choice build (bc_insert_peers) ------------------------------------

def test_part_ranges_cover():
    from paper_2501_18977_b200.distributed import part_ranges

    for M in (1, 7, 512, 32768, 1_572_864, 1_000_003):
        for w in (1, 2, 3, 8, 16):
            r = part_ranges(M, w)
            assert r[0][0] == 0 and r[-1][1] == 8 * M
            assert all(r[i][1] == r[i + 1][0] for i in range(w - 1))
            assert all(a % 8 == 0 and b % 8 == 0 for a, b in r)


def _relaxed_close_to_exact(bb, relaxed, exact, keys):
    """SURVEY §8(a) relaxed tolerances against the exact build (as in the GPU
    parity tests): no false negatives, FPR within 0.1 + 3 sigma in log2 over
    2^24 negatives, mean load within 1 bit, variance within 15% (+3 sigma of
    its estimate)."""
    import math

    assert relaxed.contains_many(keys).all(), "partitioned build: false negatives"
    neg = bb.odd_keys(1 << 24, 12, device="cuda")
    fp_e, fp_r = exact.count_hits(neg), relaxed.count_hits(neg)
    sigma = math.sqrt(1 / max(fp_e, 1) + 1 / max(fp_r, 1)) / math.log(2)
    assert abs(math.log2(max(fp_r, 1) / max(fp_e, 1))) <= 0.1 + 3 * sigma, (fp_e, fp_r)
    h_r, h_e = bb.block_load_histogram(relaxed), bb.block_load_histogram(exact)
    assert abs(h_r.mean_load - h_e.mean_load) <= 1.0
    tol = 0.15 + 3 * math.sqrt(2.0 / relaxed.num_blocks)
    assert abs(h_r.variance / h_e.variance - 1) <= tol, (h_r.variance, h_e.variance)


@pytest.mark.gpu
@pytest.mark.parametrize("world,cfgkw,n", [
    (1, dict(kind="blowchoc", k=14, choices=2, size_bits=16 * 2**20, seed=1), 2**20),
    (2, dict(kind="blowchoc", k=14, choices=2, size_bits=16 * 2**20, seed=1), 2**20),
    (3, dict(kind="blowchoc", k=14, choices=2, size_bits=16 * 2**20, seed=1), 2**20),
    (4, dict(kind="blowchoc", k=16, choices=3, size_bits=16 * 300_007, seed=5), 300_007),
    (8, dict(kind="blowchoc", k=11, choices=2, size_bits=2**26, seed=1), 5_000_000),
    (16, dict(kind="blowchoc", k=8, choices=4, n_capacity=400_000, seed=9), 400_000),
])
def test_partitioned_insert_emulated_ranks(world, cfgkw, n):
    """bc_insert_peers with W replicas held on one GPU (each rank's call
    launched in turn with its key slice and every replica's address): each
    block is written only in its owner's replica, and the owners' ranges put
    together are a relaxed build of the whole stream within the stated
    tolerance of the exact (reference-order) build."""
    import ctypes

    import paper_2501_18977_b200 as bb
    from paper_2501_18977_b200 import _native
    from paper_2501_18977_b200.distributed import part_ranges, slice_bounds

    cfg = bb.FilterConfig(**cfgkw)
    keys = bb.even_keys(n, 11, device="cuda")
    exact = bb.Filter.from_config(cfg)
    exact.insert_many(keys)
    f = bb.Filter.from_config(cfg, insert_mode="relaxed")
    nw = f.storage.d_words.numel()
    reps = [torch.zeros(nw, dtype=torch.int64, device="cuda") for _ in range(world)]
    ptrs = (ctypes.c_uint64 * world)(*[r.data_ptr() for r in reps])
    stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    k64 = keys.view(torch.int64)
    share = max(256, (f.num_blocks // 2) // world)
    for rank, (lo, hi) in enumerate(slice_bounds(n, world)):
        part = k64[lo:hi].contiguous()
        _native.check(_native.lib().bc_insert_peers(
            ctypes.c_void_p(f.handle), ptrs, world, ctypes.c_void_p(part.data_ptr()),
            part.numel(), share, stream))
    torch.cuda.synchronize()
    ranges = part_ranges(f.num_blocks, world)
    full = torch.zeros(nw, dtype=torch.int64, device="cuda")
    for r, (a, b) in enumerate(ranges):
        outside = torch.cat([reps[r][:a], reps[r][b:]])
        assert not bool(outside.any()), f"replica {r} written outside its partition"
        full[a:b] = reps[r][a:b]
    f.storage.d_words.view(torch.int64).copy_(full)
    f.storage.device_modified()
    _relaxed_close_to_exact(bb, f, exact, keys)
    with pytest.raises(RuntimeError):  # not a partitionable geometry (BC_EUNSUP)
        g = bb.Filter.from_config(bb.FilterConfig(kind="blocked", k=8, n_capacity=1000, seed=1))
        _native.check(_native.lib().bc_insert_peers(ctypes.c_void_p(g.handle), ptrs, world,
                                                    ctypes.c_void_p(0), 0, 0, stream))


def _partition_worker(rank, world, port):
    import hashlib

    import paper_2501_18977_b200 as bb
    from paper_2501_18977_b200 import distributed as D

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["BC_PEER_ALLREDUCE"] = "1"
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = bb.FilterConfig(kind="blowchoc", k=14, choices=2, size_bits=16 * 2**20, seed=1)
        keys = bb.even_keys(2**20, 11, device="cuda")
        pad = torch.empty(4096 + 192 * rank, dtype=torch.uint8, device="cuda")  # interior pointers
        f = bb.Filter.from_config(cfg, insert_mode="relaxed")
        assert D.build_partitioned(f, keys)
        assert f.inserted == keys.numel()
        digest = hashlib.sha256(f.storage.words.tobytes()).hexdigest()
        seen = [None] * world
        dist.all_gather_object(seen, digest)
        assert len(set(seen)) == 1, "replicas differ after the partitioned build"
        exact = bb.Filter.from_config(cfg)
        exact.insert_many(keys)
        _relaxed_close_to_exact(bb, f, exact, keys)
        del pad
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_partitioned_build_two_processes_one_gpu():
    """build_partitioned end to end: two ranks (gloo barriers) sharing cuda:0
    map each other's replicas over CUDA IPC, each inserts its half of the
    stream into the partitioned filter with one kernel, the owners' ranges
    are broadcast, and both ranks end with the same relaxed build within
    tolerance of the exact one."""
    mp.spawn(_partition_worker, args=(2, free_port()), nprocs=2, join=True)
