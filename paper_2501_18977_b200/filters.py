"""Filter model and the batched API -- the drop-in for the reference's
``blowchoc.filters`` (filters.py:1-402).

Construction, validation, sizing, hash derivation and the scalar helpers are
host code with the reference's exact semantics.  The batched operations
(``insert_many``, ``contains_many``, ``count_hits``, q-gram insert/lookup)
call the sm_100a kernels of ``libbbchoc.so`` through the C ABI -- the
reference's four ``_kernels.*`` call sites (filters.py:381-394) map onto
``bc_insert`` / ``bc_contains``.

Inputs may be numpy arrays (host; results come back as numpy) or CUDA
tensors (results stay on the device).  ``insert_mode``:

* ``"ordered"`` (default) -- multi-choice inserts reproduce the reference's
  stream order exactly (bit-identical bit arrays);
* ``"relaxed"`` -- atomic inserts with at most M/2 keys in flight; zero false
  negatives and FPR / load histogram within the tolerance of DESIGN.md §5.

Single-choice and standard inserts are order-free: both modes are
bit-identical to the reference.
"""

from __future__ import annotations

import ctypes
import math
import threading
from dataclasses import dataclass, replace

import numpy as np
import torch

from . import _native
from ._native import BC_INSERT_ORDERED, BC_INSERT_RELAXED, BcFilterDesc, check, lib
from .blockstore import BlockArray, valid_block_bits
from .hashing import BitSelector, HashSpec, SplitMix64, eval_hash, hash_branch, make_hash

KINDS = ("standard", "blocked", "blowchoc")
COST_KINDS = ("exp", "mix", "la")
MAX_CHOICES = 8
INSERT_MODES = {"ordered": BC_INSERT_ORDERED, "relaxed": BC_INSERT_RELAXED}

#: default base of the exponential cost (filters.py:33)
GOLDEN_BETA = (1 + math.sqrt(5)) / 2


class ConfigError(ValueError):
    """Invalid filter configuration."""


# -- cost models (filters.py:40-62; evaluated in float64 like the reference) ----------

def cost_exp(j: int, a: int, k: int, beta: float, block_bits: int = 512) -> float:
    return beta ** (j / (block_bits / 4)) + a / k


def cost_mix(j: int, a: int, k: int, sigma: float, block_bits: int = 512) -> float:
    return sigma * k * (j / (block_bits / 2)) ** float(k) + a


def cost_la(j: int, a: int, k: int, mu: float, block_bits: int = 512) -> float:
    return k * ((j + mu * k) / (block_bits / 2)) ** float(k) + a


@dataclass(frozen=True)
class CostModel:
    kind: str
    param: float
    k: int

    def __post_init__(self):
        if self.kind not in COST_KINDS:
            raise ConfigError(f"unknown cost kind {self.kind!r}")
        if self.kind == "exp" and not self.param > 0:
            raise ConfigError(f"exp cost needs a base > 0, got {self.param}")
        if self.kind in ("mix", "la") and self.param < 0:
            raise ConfigError(f"{self.kind} cost needs a parameter >= 0, got {self.param}")
        if self.k < 1:
            raise ConfigError(f"cost model needs k >= 1, got {self.k}")

    def evaluate(self, j: int, a: int, block_bits: int = 512) -> float:
        fn = {"exp": cost_exp, "mix": cost_mix, "la": cost_la}[self.kind]
        return fn(j, a, self.k, self.param, block_bits)

    @property
    def code(self) -> int:
        return COST_KINDS.index(self.kind)


def default_cost(k: int) -> CostModel:
    return CostModel(kind="exp", param=GOLDEN_BETA, k=k)


def cost_table(kind: str, param: float, k: int, block_bits: int) -> np.ndarray:
    """float64 costs of every (j, a), j in [0, B], a in [0, k], computed with
    the kernel formulas of the reference (_kernels.py:100-109)."""
    kf = float(k)
    quarter, half = block_bits / 4.0, block_bits / 2.0
    tab = np.empty((block_bits + 1, k + 1), dtype=np.float64)
    for j in range(block_bits + 1):
        jf = float(j)
        for a in range(k + 1):
            af = float(a)
            if kind == "exp":
                v = param ** (jf / quarter) + af / kf
            elif kind == "mix":
                v = param * kf * (jf / half) ** kf + af
            else:
                v = kf * ((jf + param * kf) / half) ** kf + af
            tab[j, a] = v
    return tab


# -- sizing -------------------------------------------------------------------------------

def size_for(n: int, k: int, relative_size: float = 1.0, block_bits: int = 512,
             shards: int = 1) -> tuple:
    """(m bits, M blocks) for n keys at k bits each, expected load 1/2 at
    relative_size 1, rounded to whole blocks and a shard multiple
    (filters.py:99-114)."""
    if n < 1:
        raise ConfigError(f"capacity must be >= 1, got {n}")
    if k < 1:
        raise ConfigError(f"k must be >= 1, got {k}")
    blocks = math.ceil(relative_size * n * k / math.log(2) / block_bits)
    blocks = -(-blocks // shards) * shards
    return blocks * block_bits, blocks


def overload_fpr(gamma: float, k: int) -> float:
    """(1 - 2^-gamma)^k (filters.py:117-122)."""
    if k < 1:
        raise ConfigError(f"k must be >= 1, got {k}")
    return (1.0 - 2.0 ** -gamma) ** k


@dataclass(frozen=True)
class FilterConfig:
    """Build parameters; ``validated()`` normalises them (filters.py:125-203)."""

    kind: str
    k: int
    n_capacity: int | None = None
    size_bits: int | None = None
    choices: int | None = None
    cost: CostModel | None = None
    strategy: str = "random"
    relative_size: float = 1.0
    shards: int = 1
    seed: int = 0
    block_bits: int = 512

    def _problems(self):
        """The configuration errors, in the order the reference checks them
        (filters.py:147-194): (condition, message) pairs, lazily."""
        bb = self.block_bits
        yield self.kind not in KINDS, lambda: f"unknown filter kind {self.kind!r}"
        yield not valid_block_bits(bb), lambda: f"invalid block_bits {bb}"
        yield not 1 <= self.k <= bb, \
            lambda: f"k must be in [1, {bb}] for {bb}-bit blocks, got {self.k}"
        yield self.strategy not in ("random", "distinct"), \
            lambda: f"unknown bit strategy {self.strategy!r}"
        yield (self.n_capacity is None) == (self.size_bits is None), \
            lambda: "give exactly one of n_capacity and size_bits"
        yield self.n_capacity is not None and self.n_capacity < 1, \
            lambda: f"capacity must be >= 1, got {self.n_capacity}"
        sized = self.size_bits is not None
        yield sized and self.size_bits < 1, lambda: f"size_bits must be >= 1, got {self.size_bits}"
        yield sized and self.relative_size != 1.0, \
            lambda: "relative_size only applies to capacity-based sizing"
        yield not self.relative_size > 0, \
            lambda: f"relative_size must be > 0, got {self.relative_size}"
        yield self.shards < 1, lambda: f"shard count must be >= 1, got {self.shards}"

    def _per_kind(self) -> tuple:
        """(choices, cost) normalised for the kind, or ConfigError."""
        c, cost = self.choices, self.cost
        if self.kind == "standard":
            checks = ((self.strategy != "random",
                       "the distinct strategy applies only to blocked filters"),
                      (self.shards != 1,
                       "standard filters do not shard (bits span the whole array)"),
                      (self.block_bits % 64 != 0,
                       "standard filters need word-multiple block_bits"))
            for bad, msg in checks:
                if bad:
                    raise ConfigError(msg)
            return 0, None
        if self.kind == "blocked":
            if c not in (None, 1):
                raise ConfigError(f"blocked filters have exactly one choice, got {c}")
            return 1, None
        c = 2 if c is None else c
        if not 2 <= c <= MAX_CHOICES:
            raise ConfigError(f"blowchoc needs between 2 and {MAX_CHOICES} choices, got {c}")
        cost = cost if cost is not None else default_cost(self.k)
        if cost.k != self.k:
            raise ConfigError(f"cost model k={cost.k} does not match filter k={self.k}")
        return c, cost

    def validated(self) -> "FilterConfig":
        """A normalised copy (choices and cost filled in per kind, 64-bit seed),
        or ConfigError with the reference's message."""
        for bad, message in self._problems():
            if bad:
                raise ConfigError(message())
        choices, cost = self._per_kind()
        return replace(self, choices=choices, cost=cost, seed=self.seed % (1 << 64))

    def sizing(self) -> tuple:
        """(m bits, M blocks): ``size_bits`` rounded up to whole blocks and a
        shard multiple, else ``size_for`` of the capacity."""
        if self.size_bits is None:
            return size_for(self.n_capacity, self.k, self.relative_size, self.block_bits,
                            self.shards)
        blocks = -(-self.size_bits // (self.block_bits * self.shards)) * self.shards
        return blocks * self.block_bits, blocks


_KIND_CODE = {"standard": 0, "blocked": 1, "blowchoc": 2}
_HANDLE_LOCK = threading.Lock()


class Filter:
    """A live filter: configuration, hash functions and the GPU bit store."""

    def __init__(self, *, kind: str, k: int, choices: int, strategy: str,
                 cost: CostModel | None, block_bits: int, num_blocks: int, shards: int,
                 seed: int, inserted: int = 0, words: np.ndarray | None = None,
                 device: torch.device | None = None, insert_mode: str = "ordered"):
        if insert_mode not in INSERT_MODES:
            raise ConfigError(f"unknown insert mode {insert_mode!r}")
        self.kind = kind
        self.k = k
        self.choices = choices
        self.strategy = strategy
        self.cost = cost
        self.shards = shards
        self.seed = seed
        self.inserted = inserted
        self.insert_mode = insert_mode
        if num_blocks % shards != 0:
            raise ConfigError(f"{num_blocks} blocks do not split into {shards} shards")
        self.storage = BlockArray(num_blocks, block_bits, device)
        if words is not None:
            if np.asarray(words).shape != (self.storage.num_words,):
                raise ConfigError("word array does not match the filter geometry")
            self.storage.load_words(words)
        self._derive_hashes()
        self._handle = None

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h:
            try:
                lib().bc_filter_destroy(h)
            except Exception:
                pass

    @classmethod
    def from_config(cls, config: FilterConfig, **kw) -> "Filter":
        cfg = config.validated()
        _, num_blocks = cfg.sizing()
        return cls(kind=cfg.kind, k=cfg.k, choices=cfg.choices, strategy=cfg.strategy,
                   cost=cfg.cost, block_bits=cfg.block_bits, num_blocks=num_blocks,
                   shards=cfg.shards, seed=cfg.seed, **kw)

    def _derive_hashes(self) -> None:
        # draw order: shard hash, block hashes, bit hashes (filters.py:252-263)
        rng = SplitMix64(self.seed)
        self.shard_spec: HashSpec = make_hash(rng, self.shards)
        if self.kind == "standard":
            self.block_specs: tuple = ()
            self.bit_selector = None
            self.bit_specs = tuple(make_hash(rng, self.m) for _ in range(self.k))
        else:
            per = self.num_blocks // self.shards
            self.block_specs = tuple(make_hash(rng, per) for _ in range(self.choices))
            self.bit_selector = BitSelector.draw(rng, self.strategy, self.k, self.block_bits)
            self.bit_specs = self.bit_selector.specs

    # -- geometry ---------------------------------------------------------------------
    @property
    def num_blocks(self) -> int:
        return self.storage.num_blocks

    @property
    def block_bits(self) -> int:
        return self.storage.block_bits

    @property
    def m(self) -> int:
        return self.storage.total_bits

    @property
    def blocks_per_shard(self) -> int:
        return self.num_blocks // self.shards

    @property
    def device(self) -> torch.device:
        return self.storage.device

    # -- scalar API (host semantics of filters.py:285-343) -----------------------------
    def shard_of(self, x: int) -> int:
        return eval_hash(self.shard_spec, x)

    def candidate_blocks(self, x: int) -> list:
        base = self.shard_of(x) * self.blocks_per_shard
        return [base + eval_hash(h, x) for h in self.block_specs]

    def choose_block(self, blocks, addrs) -> tuple:
        """(choice index, no-op) for inserting ``addrs`` among ``blocks``."""
        sims = []
        for i, b in enumerate(blocks):
            j, a = self.storage.simulate_insertion(b, addrs)
            if a == 0:
                return i, True
            sims.append((j, a))
        if len(blocks) == 1:
            return 0, False
        costs = [self.cost.evaluate(j, a, self.block_bits) for j, a in sims]
        return min(range(len(costs)), key=costs.__getitem__), False

    def insert(self, x: int) -> None:
        """Insert one key (a batch of one through the GPU path)."""
        self.insert_many(np.array([x], dtype=np.uint64))

    def lookup(self, x: int) -> bool:
        return bool(self.contains_many(np.array([x], dtype=np.uint64))[0])

    def __contains__(self, x: int) -> bool:
        return self.lookup(x)

    def load(self) -> float:
        return self.storage.total_set_bits() / self.m

    # -- native handle --------------------------------------------------------------------
    def _kernel_args(self) -> BcFilterDesc:
        """The C-ABI mirror of the reference's _kernel_args()/_cost_args()."""
        d = BcFilterDesc()
        d.kind = _KIND_CODE[self.kind]
        d.k = self.k
        d.choices = self.choices
        d.strategy = 0 if self.strategy == "random" else 1
        d.block_bits = self.block_bits
        d.num_blocks = self.num_blocks
        d.shards = self.shards
        d.shard_a = self.shard_spec.a
        for i, h in enumerate(self.block_specs):
            d.block_a[i] = h.a
        self._bit_a = np.array([s.a for s in self.bit_specs], dtype=np.uint64)
        self._bit_b = np.array([s.b for s in self.bit_specs], dtype=np.uint64)
        d.bit_a = self._bit_a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))
        d.bit_b = self._bit_b.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))
        if self.cost is not None:
            d.cost_code = self.cost.code
            d.cost_param = float(self.cost.param)
            self._cost_tab = np.ascontiguousarray(
                cost_table(self.cost.kind, float(self.cost.param), self.k, self.block_bits))
            d.cost_table = self._cost_tab.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        return d

    @property
    def handle(self):
        """The C-ABI handle, created once (thread-safe: lookups may run from
        several threads, as in the reference's query pool)."""
        if self._handle is None:
            with _HANDLE_LOCK:
                if self._handle is None:
                    dev = self.device
                    with torch.cuda.device(dev):
                        h = ctypes.c_void_p()
                        check(lib().bc_filter_create(ctypes.byref(self._kernel_args()),
                                                     ctypes.byref(h)))
                    self._handle = h.value
        return self._handle

    # -- batched operations (the hot path) --------------------------------------------------
    def _mode(self, mode) -> int:
        mode = self.insert_mode if mode is None else mode
        if mode not in INSERT_MODES:
            raise ConfigError(f"unknown insert mode {mode!r}")
        return INSERT_MODES[mode]

    def insert_many(self, keys, mode: str | None = None) -> None:
        """Insert a key array in stream order (one writer per shard)."""
        from ._device import as_device_u64, host_u64, is_device_tensor, ptr, stream_ptr

        m = self._mode(mode)
        dev = self.device
        with torch.cuda.device(dev):
            words = self.storage.d_words
            if is_device_tensor(keys):
                d_keys = as_device_u64(keys, dev)
                n = d_keys.numel()
                check(lib().bc_insert(self.handle, ptr(words), ptr(d_keys), n, m,
                                      stream_ptr(dev)))
            else:
                h = host_u64(keys)
                n = h.shape[0]
                check(lib().bc_insert_host(self.handle, ptr(words), h.ctypes.data, n, m,
                                           stream_ptr(dev)))
        self.storage.device_modified()
        self.inserted += n

    def contains_many(self, keys, out=None):
        """Membership per key: numpy bool for host keys, CUDA bool tensor for
        device keys.  ``out`` (optional) receives the answers: a uint8/bool
        numpy array (pinned memory is written directly by the copy engine) or
        a CUDA tensor for device keys."""
        from ._device import as_device_u64, host_u64, is_device_tensor, ptr, stream_ptr

        dev = self.device
        with torch.cuda.device(dev):
            words = self.storage.d_words
            if is_device_tensor(keys):
                d_keys = as_device_u64(keys, dev)
                n = d_keys.numel()
                if out is None:
                    out = torch.empty(n, dtype=torch.uint8, device=dev)
                elif not (is_device_tensor(out) and out.numel() == n and out.is_contiguous()
                          and out.element_size() == 1):
                    raise ValueError("out must be a contiguous 1-byte CUDA tensor of n elements")
                check(lib().bc_contains(self.handle, ptr(words), ptr(d_keys), n,
                                        ptr(out), None, stream_ptr(dev)))
                return out.view(torch.bool)
            h = host_u64(keys)
            if out is None:
                out = np.empty(h.shape[0], dtype=np.uint8)
            elif not (isinstance(out, np.ndarray) and out.shape == (h.shape[0],)
                      and out.dtype.itemsize == 1 and out.flags.c_contiguous):
                raise ValueError("out must be a contiguous 1-byte numpy array of n elements")
            check(lib().bc_contains_host(self.handle, ptr(words), h.ctypes.data, h.shape[0],
                                         out.ctypes.data, None, stream_ptr(dev)))
            return out.view(np.bool_)

    def count_hits(self, keys) -> int:
        from ._device import as_device_u64, host_u64, is_device_tensor, ptr, stream_ptr

        dev = self.device
        with torch.cuda.device(dev):
            words = self.storage.d_words
            if is_device_tensor(keys):
                d_keys = as_device_u64(keys, dev)
                hits = torch.zeros(1, dtype=torch.int64, device=dev)
                check(lib().bc_contains(self.handle, ptr(words), ptr(d_keys), d_keys.numel(),
                                        None, ptr(hits), stream_ptr(dev)))
                return int(hits.item())
            h = host_u64(keys)
            hits = ctypes.c_ulonglong(0)
            check(lib().bc_contains_host(self.handle, ptr(words), h.ctypes.data, h.shape[0],
                                         None, ctypes.byref(hits), stream_ptr(dev)))
            return int(hits.value)

    # -- fused DNA q-gram path ------------------------------------------------------------------
    def insert_qgrams(self, enc, sequence, mode: str | None = None,
                      record_len: int | None = None) -> int:
        """== insert_many(encode_qgrams(enc, sequence)); returns the number of
        keys inserted.  The key array is never materialised.  A 2-D byte array
        (reads x length), or ``record_len``, marks fixed-length records that
        no window may cross."""
        from ._device import as_device_bytes, ptr, sequence_records, stream_ptr

        m = self._mode(mode)
        dev = self.device
        with torch.cuda.device(dev):
            flat, rec = sequence_records(sequence, record_len)
            seq = as_device_bytes(flat, dev)
            n = seq.numel()
            d_cnt = torch.zeros(1, dtype=torch.int64, device=dev)
            check(lib().bc_insert_qgrams(self.handle, ptr(self.storage.d_words),
                                         ptr(seq) if n else None, n, enc.q,
                                         int(enc.canonical), rec, m, ptr(d_cnt),
                                         stream_ptr(dev)))
            cnt = int(d_cnt.item())
        self.storage.device_modified()
        self.inserted += cnt
        return cnt

    def insert_qgram_batches(self, enc, batches, mode: str | None = None) -> int:
        """insert_qgrams over an iterable of sequences (e.g. io.fasta_batches)
        without a host sync per batch: every batch's count stays on the device
        and all are read once at the end, so the host prepares (reads, parses)
        the next batch while the GPU inserts this one.  Returns the total."""
        from ._device import as_device_bytes, ptr, sequence_records, stream_ptr

        m = self._mode(mode)
        dev = self.device
        slots: list = []  # device count arrays, 1024 batches each
        used = 0
        with torch.cuda.device(dev):
            for sequence in batches:
                flat, rec = sequence_records(sequence, None)
                seq = as_device_bytes(flat, dev)
                n = seq.numel()
                if used % 1024 == 0:
                    slots.append(torch.zeros(1024, dtype=torch.int64, device=dev))
                check(lib().bc_insert_qgrams(self.handle, ptr(self.storage.d_words),
                                             ptr(seq) if n else None, n, enc.q,
                                             int(enc.canonical), rec, m,
                                             ptr(slots[-1]) + 8 * (used % 1024),
                                             stream_ptr(dev)))
                used += 1
            cnt = sum(int(t.sum().item()) for t in slots)
        self.storage.device_modified()
        self.inserted += cnt
        return cnt

    def _qgram_lookup(self, enc, sequence, record_len, want_answers: bool):
        from ._device import as_device_bytes, ptr, sequence_records, stream_ptr

        dev = self.device
        with torch.cuda.device(dev):
            flat, rec = sequence_records(sequence, record_len)
            seq = as_device_bytes(flat, dev)
            n = seq.numel()
            out = cnt = hits = None
            if want_answers:
                out = torch.empty(max(n - enc.q + 1, 1), dtype=torch.uint8, device=dev)
                cnt = torch.zeros(1, dtype=torch.int64, device=dev)
            else:
                hits = torch.zeros(1, dtype=torch.int64, device=dev)
            check(lib().bc_contains_qgrams(self.handle, ptr(self.storage.d_words),
                                           ptr(seq) if n else None, n, enc.q,
                                           int(enc.canonical), rec, ptr(out), ptr(cnt),
                                           ptr(hits), stream_ptr(dev)))
            if want_answers:
                return out[:int(cnt.item())].view(torch.bool)
            return int(hits.item())

    def contains_qgrams(self, enc, sequence, record_len: int | None = None):
        """== contains_many(encode_qgrams(enc, sequence)); records as in
        ``insert_qgrams``."""
        from ._device import is_device_tensor

        res = self._qgram_lookup(enc, sequence, record_len, True)
        return res if is_device_tensor(sequence) else res.cpu().numpy()

    def count_qgram_hits(self, enc, sequence, record_len: int | None = None) -> int:
        return self._qgram_lookup(enc, sequence, record_len, False)

    def route_many(self, keys):
        """Shard index per key (GPU)."""
        from ._device import eval_hash

        return eval_hash(self.shard_spec.a, self.shard_spec.b, keys)


__all__ = ["KINDS", "COST_KINDS", "MAX_CHOICES", "GOLDEN_BETA", "ConfigError", "cost_exp",
           "cost_mix", "cost_la", "CostModel", "default_cost", "cost_table", "size_for",
           "overload_fpr", "FilterConfig", "Filter", "hash_branch", "_native"]
