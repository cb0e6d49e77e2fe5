"""ctypes binding of ``libbbchoc.so`` (the C ABI declared in include/bbchoc.h).

The library is built in-tree by ``python -m paper_2501_18977_b200.build``
(``__graft_entry__.build()`` does it).  There is no fallback: if the library
or a CUDA device is missing, every batched operation raises.
"""

from __future__ import annotations

import atexit
import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
# BC_LIBRARY: load another build of the same ABI (A/B measurements)
LIB_PATH = os.environ.get("BC_LIBRARY") or os.path.join(HERE, "libbbchoc.so")

BC_OK, BC_EINVAL, BC_ECUDA, BC_ENOMEM, BC_EUNSUP = 0, -1, -2, -3, -4
BC_INSERT_ORDERED, BC_INSERT_RELAXED = 0, 1
MAX_CHOICES = 8

#: every symbol include/bbchoc.h declares (checked by the CPU test-suite)
EXPORTS = (
    "bc_filter_create", "bc_filter_destroy", "bc_insert", "bc_contains",
    "bc_insert_host", "bc_contains_host", "bc_encode_qgrams", "bc_insert_qgrams",
    "bc_contains_qgrams", "bc_block_histogram", "bc_route", "bc_eval_hash",
    "bc_last_error", "bc_launch_count", "bc_version", "bc_pcg64_fill", "bc_l2_release",
    "bc_format_answers", "bc_parse_keys_text", "bc_fasta_join", "bc_ipc_export", "bc_ipc_import",
    "bc_ipc_close", "bc_peer_span", "bc_or_allreduce_peers", "bc_insert_peers",
)


class BcFilterDesc(ctypes.Structure):
    """Mirror of ``bc_filter_desc``."""

    _fields_ = [
        ("kind", ctypes.c_int32),
        ("k", ctypes.c_int32),
        ("choices", ctypes.c_int32),
        ("strategy", ctypes.c_int32),
        ("block_bits", ctypes.c_int32),
        ("reserved0", ctypes.c_int32),
        ("num_blocks", ctypes.c_uint64),
        ("shards", ctypes.c_uint64),
        ("shard_a", ctypes.c_uint64),
        ("block_a", ctypes.c_uint64 * MAX_CHOICES),
        ("bit_a", ctypes.POINTER(ctypes.c_uint64)),
        ("bit_b", ctypes.POINTER(ctypes.c_uint64)),
        ("cost_code", ctypes.c_int32),
        ("reserved1", ctypes.c_int32),
        ("cost_param", ctypes.c_double),
        ("cost_table", ctypes.POINTER(ctypes.c_double)),
    ]


_lib = None
_lock = threading.Lock()


class NativeError(RuntimeError):
    """A CUDA-side failure reported by libbbchoc."""


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing; build it with `python -m paper_2501_18977_b200.build`"
            )
        L = ctypes.CDLL(LIB_PATH)
        P, u64, ci = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int
        L.bc_filter_create.argtypes = [ctypes.POINTER(BcFilterDesc), ctypes.POINTER(P)]
        L.bc_filter_destroy.argtypes = [P]
        L.bc_filter_destroy.restype = None
        L.bc_insert.argtypes = [P, P, P, u64, ci, P]
        L.bc_contains.argtypes = [P, P, P, u64, P, P, P]
        L.bc_insert_host.argtypes = [P, P, P, u64, ci, P]
        L.bc_contains_host.argtypes = [P, P, P, u64, P, P, P]
        L.bc_encode_qgrams.argtypes = [P, u64, ci, ci, u64, P, P, P]
        L.bc_insert_qgrams.argtypes = [P, P, P, u64, ci, ci, u64, ci, P, P]
        L.bc_contains_qgrams.argtypes = [P, P, P, u64, ci, ci, u64, P, P, P, P]
        L.bc_block_histogram.argtypes = [P, u64, ci, P, P]
        L.bc_route.argtypes = [P, P, u64, P, P]
        L.bc_eval_hash.argtypes = [u64, u64, P, u64, P, P]
        L.bc_pcg64_fill.argtypes = [u64, u64, u64, u64, u64, u64, u64, u64, P, P]
        L.bc_last_error.restype = ctypes.c_char_p
        L.bc_launch_count.restype = ctypes.c_ulonglong
        L.bc_version.restype = ctypes.c_char_p
        L.bc_l2_release.restype = None
        L.bc_format_answers.argtypes = [P, P, u64, P, u64, P]
        L.bc_parse_keys_text.argtypes = [P, u64, P, u64, P, P, P]
        L.bc_fasta_join.argtypes = [P, u64, ci, ctypes.c_uint8, P, P, u64, P, P, u64, P, P]
        L.bc_ipc_export.argtypes = [P, P, P]
        L.bc_ipc_import.argtypes = [P, u64, P]
        L.bc_ipc_close.argtypes = [P, u64]
        L.bc_peer_span.argtypes = [u64, ci, P]
        L.bc_or_allreduce_peers.argtypes = [P, ci, ci, u64, P]
        L.bc_insert_peers.argtypes = [P, P, ci, P, u64, u64, P]
        for name in EXPORTS:
            fn = getattr(L, name)
            if fn.restype is ctypes.c_int or name in (
                    "bc_filter_create", "bc_insert", "bc_contains", "bc_insert_host",
                    "bc_contains_host", "bc_encode_qgrams", "bc_insert_qgrams",
                    "bc_contains_qgrams", "bc_block_histogram", "bc_route", "bc_eval_hash",
                    "bc_pcg64_fill", "bc_format_answers", "bc_parse_keys_text", "bc_fasta_join",
                    "bc_ipc_export", "bc_ipc_import", "bc_ipc_close", "bc_peer_span",
                    "bc_or_allreduce_peers", "bc_insert_peers"):
                fn.restype = ctypes.c_int
        _lib = L
        atexit.register(L.bc_l2_release)
        return L


def check(rc: int) -> None:
    if rc == BC_OK:
        return
    msg = lib().bc_last_error().decode(errors="replace")
    if rc == BC_EINVAL:
        raise ValueError(msg)
    if rc == BC_ENOMEM:
        raise MemoryError(msg)
    raise NativeError(f"libbbchoc error {rc}: {msg}")


def launch_count() -> int:
    return int(lib().bc_launch_count())
