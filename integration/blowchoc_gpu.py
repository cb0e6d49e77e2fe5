"""Drop-in replacement for the reference's compiled layer, ``blowchoc._kernels``.

This is the binding a maintainer of the reference adds: a
ctypes module over ``libbbchoc.so`` exposing the four numba kernels the
reference calls from ``Filter.insert_many`` / ``contains_many``
(``pkg/src/blowchoc/filters.py:377-395``) with their exact signatures:

    insert_blocks(words, keys, *_kernel_args(), *_cost_args())   # _kernels.py:112-174
    contains_blocks(words, keys, *_kernel_args(), out)           # _kernels.py:177-211
    insert_flat(words, keys, *_kernel_args())                    # _kernels.py:214-222
    contains_flat(words, keys, *_kernel_args(), out)             # _kernels.py:225-237

Switching the reference over is one line in filters.py,
``from . import _kernels`` -> ``import blowchoc_gpu as _kernels`` (or, as the
GPU integration test does, ``blowchoc.filters._kernels = blowchoc_gpu``).
Nothing else in the reference changes: it keeps owning ``storage.words`` as a
host numpy array, which its own tests and scalar helpers read and write
directly (``test_acceptance.py:204``, ``storage.set_bits``).

Coherence: every call mirrors the host words into a device copy
(``_DeviceWords``), runs the kernel, and (inserts) copies the words back,
under one lock per host array -- so the reference's sharded builder, whose
worker threads insert into one filter concurrently (``sharding.py:68-133``),
stays correct.  The copies make this binding PCIe-bound; it is the
correctness-first drop-in.  ``paper_2501_18977_b200`` is the resident
version (words stay in HBM, the host mirror is synced lazily).

No CPU fallback: without ``libbbchoc.so`` or a CUDA device every call raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get(
    "BBCHOC_LIB", os.path.join(_HERE, "..", "paper_2501_18977_b200", "libbbchoc.so"))

P, u64, ci = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int
BC_INSERT_ORDERED = 0  # the reference's stream order, bit for bit
MAX_CHOICES = 8


class Desc(ctypes.Structure):
    """``bc_filter_desc`` (include/bbchoc.h)."""

    _fields_ = [("kind", ctypes.c_int32), ("k", ctypes.c_int32), ("choices", ctypes.c_int32),
                ("strategy", ctypes.c_int32), ("block_bits", ctypes.c_int32),
                ("reserved0", ctypes.c_int32), ("num_blocks", u64), ("shards", u64),
                ("shard_a", u64), ("block_a", u64 * MAX_CHOICES),
                ("bit_a", ctypes.POINTER(u64)), ("bit_b", ctypes.POINTER(u64)),
                ("cost_code", ctypes.c_int32), ("reserved1", ctypes.c_int32),
                ("cost_param", ctypes.c_double), ("cost_table", ctypes.POINTER(ctypes.c_double))]


_L = None
_lib_lock = threading.Lock()
calls = {"insert_blocks": 0, "contains_blocks": 0, "insert_flat": 0, "contains_flat": 0}


def lib() -> ctypes.CDLL:
    global _L
    with _lib_lock:
        if _L is None:
            L = ctypes.CDLL(LIB_PATH)
            L.bc_filter_create.argtypes = [ctypes.POINTER(Desc), ctypes.POINTER(P)]
            L.bc_filter_create.restype = ci
            L.bc_filter_destroy.argtypes = [P]
            L.bc_filter_destroy.restype = None
            L.bc_insert.argtypes = [P, P, P, u64, ci, P]
            L.bc_insert.restype = ci
            L.bc_contains.argtypes = [P, P, P, u64, P, P, P]
            L.bc_contains.restype = ci
            L.bc_insert_host.argtypes = [P, P, P, u64, ci, P]
            L.bc_insert_host.restype = ci
            L.bc_contains_host.argtypes = [P, P, P, u64, P, P, P]
            L.bc_contains_host.restype = ci
            L.bc_last_error.restype = ctypes.c_char_p
            _L = L
        return _L


def _check(rc: int) -> None:
    if rc:
        msg = lib().bc_last_error().decode(errors="replace")
        raise (ValueError if rc == -1 else RuntimeError)(msg)


# -- handles: one per distinct _kernel_args() tuple ---------------------------------------

_handles: dict = {}
_handles_lock = threading.Lock()


def _handle(kind: int, k: int, c: int, strategy: int, block_bits: int, num_blocks: int,
            shards: int, shard_a: int, block_a, bit_a: np.ndarray, bit_b: np.ndarray,
            cost_code: int = 0, cost_param: float = 0.0):
    key = (kind, k, c, strategy, block_bits, num_blocks, shards, shard_a, tuple(block_a),
           bit_a.tobytes(), bit_b.tobytes(), cost_code, float(cost_param))
    with _handles_lock:
        h = _handles.get(key)
        if h is None:
            d = Desc()
            d.kind, d.k, d.choices, d.strategy = kind, k, c, strategy
            d.block_bits, d.num_blocks, d.shards, d.shard_a = block_bits, num_blocks, shards, shard_a
            for i, a in enumerate(block_a):
                d.block_a[i] = int(a)
            a_arr = np.ascontiguousarray(bit_a, dtype=np.uint64)
            b_arr = np.ascontiguousarray(bit_b, dtype=np.uint64)
            d.bit_a = a_arr.ctypes.data_as(ctypes.POINTER(u64))
            d.bit_b = b_arr.ctypes.data_as(ctypes.POINTER(u64))
            d.cost_code, d.cost_param = int(cost_code), float(cost_param)
            hp = P()
            _check(lib().bc_filter_create(ctypes.byref(d), ctypes.byref(hp)))
            h = _handles[key] = hp.value
        return h


def _blocks_handle(keys_args, cost=(0, 0.0)):
    (shard_a, shard_b, _smode, _sshift, _wps, block_a, block_b, _bmode, _bshift,
     bit_a, bit_b, _bitmode, _bitshift, strategy, _wpb) = keys_args
    c = int(block_a.shape[0])
    # bit ranges are B for "random" and B - i for "distinct" (hashing.py:153-160),
    # so the block width is the first range either way
    block_bits = int(bit_b[0])
    return _handle(1 if c == 1 else 2, int(bit_a.shape[0]), c, int(strategy), block_bits,
                   int(shard_b) * int(block_b), int(shard_b), int(shard_a), block_a,
                   bit_a, bit_b, *cost)


def _flat_handle(bit_a, flat_b):
    m = int(flat_b)
    k = int(bit_a.shape[0])
    # any (B, M) with M * B = m addresses the same flat array; B must cover k
    block_bits = next(b for b in (512, 256, 128, 64) if m % b == 0 and (b >= k or b == 64))
    if k > block_bits:
        block_bits = m
    bit_b = np.full(k, m, dtype=np.uint64)
    return _handle(0, k, 0, 0, block_bits, m // block_bits, 1, 0, (), bit_a, bit_b)


# -- the device mirror of storage.words ---------------------------------------------------

class _DeviceWords:
    """Device copy of one host ``storage.words`` array (torch for the
    allocation; any cudaMalloc'd buffer would do).  ``push`` uploads the
    host words, ``pull`` writes the device words back into the host array.
    One mirror per live host array; it is dropped with the array."""

    _registry: dict = {}
    _registry_lock = threading.Lock()

    def __init__(self, nwords: int):
        import torch

        self.dev = torch.empty(nwords, dtype=torch.int64, device="cuda")
        self.lock = threading.Lock()

    @classmethod
    def of(cls, words: np.ndarray) -> "_DeviceWords":
        import weakref

        key = id(words)
        with cls._registry_lock:
            dw = cls._registry.get(key)
            if dw is None or dw.dev.numel() != words.shape[0]:
                dw = cls._registry[key] = cls(words.shape[0])
                weakref.finalize(words, cls._registry.pop, key, None)
            return dw

    @property
    def ptr(self) -> int:
        return self.dev.data_ptr()

    def push(self, words: np.ndarray) -> None:
        import torch

        self.dev.copy_(torch.from_numpy(words.view(np.int64)))

    def pull(self, words: np.ndarray) -> None:
        import torch

        torch.cuda.current_stream().synchronize()
        words.view(np.int64)[:] = self.dev.cpu().numpy()


def _stream() -> int:
    import torch

    return torch.cuda.current_stream().cuda_stream


def _insert(h, words, keys) -> None:
    keys = np.ascontiguousarray(keys, dtype=np.uint64)
    dw = _DeviceWords.of(words)
    with dw.lock:
        dw.push(words)
        _check(lib().bc_insert_host(h, dw.ptr, keys.ctypes.data, keys.shape[0],
                                    BC_INSERT_ORDERED, _stream()))
        dw.pull(words)


def _contains(h, words, keys, out) -> None:
    keys = np.ascontiguousarray(keys, dtype=np.uint64)
    if out.dtype != np.uint8 or not out.flags.c_contiguous:
        raise ValueError("out must be a contiguous uint8 array")
    dw = _DeviceWords.of(words)
    with dw.lock:
        dw.push(words)
        _check(lib().bc_contains_host(h, dw.ptr, keys.ctypes.data, keys.shape[0],
                                      out.ctypes.data, None, _stream()))


# -- the four entry points, reference signatures -------------------------------------------

def insert_blocks(words, keys, shard_a, shard_b, shard_mode, shard_shift, wps,
                  block_a, block_b, block_mode, block_shift,
                  bit_a, bit_b, bit_mode, bit_shift, strategy, wpb,
                  cost_code, cost_param, quarter, half):
    """``_kernels.insert_blocks`` (stream order, bit-exact) on the GPU."""
    calls["insert_blocks"] += 1
    args = (shard_a, shard_b, shard_mode, shard_shift, wps, block_a, block_b, block_mode,
            block_shift, bit_a, bit_b, bit_mode, bit_shift, strategy, wpb)
    h = _blocks_handle(args, (int(cost_code), float(cost_param)))
    _insert(h, words, keys)


def contains_blocks(words, keys, shard_a, shard_b, shard_mode, shard_shift, wps,
                    block_a, block_b, block_mode, block_shift,
                    bit_a, bit_b, bit_mode, bit_shift, strategy, wpb, out):
    """``_kernels.contains_blocks`` on the GPU; answers written into ``out``."""
    calls["contains_blocks"] += 1
    args = (shard_a, shard_b, shard_mode, shard_shift, wps, block_a, block_b, block_mode,
            block_shift, bit_a, bit_b, bit_mode, bit_shift, strategy, wpb)
    _contains(_blocks_handle(args), words, keys, out)


def insert_flat(words, keys, bit_a, flat_b, flat_mode, flat_shift):
    """``_kernels.insert_flat`` (standard Bloom) on the GPU."""
    calls["insert_flat"] += 1
    _insert(_flat_handle(bit_a, flat_b), words, keys)


def contains_flat(words, keys, bit_a, flat_b, flat_mode, flat_shift, out):
    """``_kernels.contains_flat`` on the GPU."""
    calls["contains_flat"] += 1
    _contains(_flat_handle(bit_a, flat_b), words, keys, out)


def install(blowchoc_filters_module) -> None:
    """Swap the reference's compiled layer for this one
    (== editing ``from . import _kernels`` in filters.py)."""
    import sys

    blowchoc_filters_module._kernels = sys.modules[__name__]
