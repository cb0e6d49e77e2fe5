"""Device plumbing: CUDA tensors (via torch) handed to the C ABI as raw
pointers, the caller's current stream, and host<->device conversions.

torch is used only as the device allocator / stream provider; every kernel
is ours (libbbchoc.so).
"""

from __future__ import annotations

import ctypes

import warnings

import numpy as np
import torch

from . import _native
from ._native import check, lib


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2501_18977_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr(device: torch.device | None = None) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _foreign_cuda(x):
    """Zero-copy torch view of a non-torch CUDA array (__cuda_array_interface__
    or DLPack on a CUDA device, e.g. CuPy / Numba / JAX arrays), else None."""
    if isinstance(x, (torch.Tensor, np.ndarray)):
        return None
    if hasattr(x, "__cuda_array_interface__"):
        return torch.as_tensor(x, device="cuda")
    if hasattr(x, "__dlpack__") and hasattr(x, "__dlpack_device__"):
        dev_type, _ = x.__dlpack_device__()
        if int(dev_type) in (2, 13):  # kDLCUDA, kDLCUDAManaged
            return torch.from_dlpack(x)
    return None


def is_device_tensor(x) -> bool:
    """CUDA input: a CUDA torch tensor or any array exposing CUDA memory."""
    if isinstance(x, torch.Tensor):
        return x.is_cuda
    return _foreign_cuda(x) is not None


def as_device_u64(x, device: torch.device) -> torch.Tensor:
    """A contiguous uint64 CUDA tensor holding the keys of ``x``."""
    foreign = _foreign_cuda(x)
    if foreign is not None:
        x = foreign
    if isinstance(x, torch.Tensor):
        if x.dtype == torch.int64:
            x = x.view(torch.uint64)
        elif x.dtype != torch.uint64:
            x = x.to(torch.int64).view(torch.uint64)
        return x.to(device).contiguous()
    arr = np.ascontiguousarray(x, dtype=np.uint64)
    return torch.from_numpy(arr).to(device)


def host_u64(x) -> np.ndarray:
    return np.ascontiguousarray(x, dtype=np.uint64)


def sequence_records(seq, record_len=None) -> tuple:
    """(sequence, record length): a 2-D byte array (reads x length) is a
    matrix of fixed-length records -- flattened, with record_len its row
    length; anything else is one sequence (record_len as given, 0 = none)."""
    foreign = _foreign_cuda(seq)
    if foreign is not None:
        seq = foreign
    if isinstance(seq, (torch.Tensor, np.ndarray)) and seq.ndim == 2:
        rows, cols = seq.shape
        if record_len not in (None, cols):
            raise ValueError(f"record_len {record_len} does not match the row length {cols}")
        return seq.reshape(rows * cols), int(cols)
    return seq, int(record_len or 0)


def as_device_bytes(seq, device: torch.device) -> torch.Tensor:
    foreign = _foreign_cuda(seq)
    if foreign is not None:
        seq = foreign
    if isinstance(seq, torch.Tensor):
        return seq.to(device=device, dtype=torch.uint8).contiguous()
    if isinstance(seq, np.ndarray):
        raw = np.ascontiguousarray(seq, dtype=np.uint8).reshape(-1)
        if not raw.size:
            return torch.empty(0, dtype=torch.uint8, device=device)
        if raw.flags.writeable:
            return torch.from_numpy(raw).to(device)
        # a read-only array (np.frombuffer over bytes) is only copied from, so
        # torch's warning about non-writable tensors does not apply
        with warnings.catch_warnings():
            warnings.simplefilter("ignore", UserWarning)
            return torch.from_numpy(raw).to(device)
    if isinstance(seq, str):
        seq = seq.encode("ascii", errors="replace")
    raw = np.frombuffer(bytes(seq), dtype=np.uint8)
    if raw.shape[0] == 0:
        return torch.empty(0, dtype=torch.uint8, device=device)
    return torch.from_numpy(raw.copy()).to(device)


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def eval_hash(a: int, b: int, keys):
    dev = require_cuda()
    on_device = is_device_tensor(keys)
    d_keys = as_device_u64(keys, dev)
    out = torch.empty_like(d_keys)
    check(lib().bc_eval_hash(a, b, ptr(d_keys), d_keys.numel(), ptr(out), stream_ptr(dev)))
    return out if on_device else out.cpu().numpy()


def histogram(d_words: torch.Tensor, num_blocks: int, block_bits: int) -> np.ndarray:
    dev = d_words.device
    counts = torch.zeros(block_bits + 1, dtype=torch.int64, device=dev)
    check(lib().bc_block_histogram(ptr(d_words), num_blocks, block_bits, ptr(counts),
                                   stream_ptr(dev)))
    return counts.cpu().numpy()


def encode_qgrams(seq, q: int, canonical: bool, record_len=None):
    """Device q-gram encoder; returns numpy (or a CUDA tensor for device input).
    A 2-D input is a matrix of fixed-length records (no window crosses rows)."""
    dev = require_cuda()
    on_device = is_device_tensor(seq)
    seq, rec = sequence_records(seq, record_len)
    d_seq = as_device_bytes(seq, dev)
    n = d_seq.numel()
    nwin = n - q + 1 if n >= q else 0
    keys = torch.empty(max(nwin, 1), dtype=torch.uint64, device=dev)
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    check(lib().bc_encode_qgrams(ptr(d_seq) if n else None, n, q, int(bool(canonical)), rec,
                                 ptr(keys), ptr(cnt), stream_ptr(dev)))
    m = int(cnt.item())
    out = keys[:m]
    return out if on_device else out.cpu().numpy()


def launch_count() -> int:
    return _native.launch_count()


__all__ = ["require_cuda", "stream_ptr", "as_device_u64", "as_device_bytes", "ptr",
           "eval_hash", "histogram", "encode_qgrams", "launch_count", "ctypes"]
