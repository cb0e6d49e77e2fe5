"""Device-resident bit store with the reference's word layout.

Layout contract (blockstore.py:1-7, 52, 72-75 of the reference): block ``b``
is words ``[b*wpb, (b+1)*wpb)`` with ``wpb = max(1, B/64)``; bit ``i`` of a
block is bit ``i % 64`` of word ``i // 64`` (LSB first).  Toy widths 8/16/32
use the low B bits of one word per block.

The words live in HBM (``d_words``, a uint64 CUDA tensor allocated through
torch; cudaMalloc alignment is 256 B, so no 64-byte block straddles a
line).  ``words`` is a host mirror for code that reads or edits the array
directly (tests, serialization, the scalar helpers): reading it copies the
device array down when the device copy is newer; the next batched operation
uploads it again in case the caller wrote into it.
"""

from __future__ import annotations

import numpy as np
import torch

DEFAULT_BLOCK_BITS = 512
CACHE_LINE_BYTES = 64
_TOY_BLOCK_BITS = (8, 16, 32)


def valid_block_bits(block_bits: int) -> bool:
    return (block_bits > 0 and block_bits % 64 == 0) or block_bits in _TOY_BLOCK_BITS


def popcount_words(words: np.ndarray) -> np.ndarray:
    return np.bitwise_count(words)


class BlockArray:
    """``num_blocks`` zeroed blocks of ``block_bits`` bits, resident on a GPU."""

    def __init__(self, num_blocks: int, block_bits: int = DEFAULT_BLOCK_BITS,
                 device: torch.device | None = None):
        if num_blocks < 1:
            raise ValueError(f"need at least one block, got {num_blocks}")
        if not valid_block_bits(block_bits):
            raise ValueError(f"block_bits must be a positive multiple of 64 (or one of "
                             f"{_TOY_BLOCK_BITS} for testing), got {block_bits}")
        self.num_blocks = num_blocks
        self.block_bits = block_bits
        self.words_per_block = max(1, block_bits // 64)
        self.num_words = num_blocks * self.words_per_block
        self._device = device
        self._d_words: torch.Tensor | None = None
        self._host: np.ndarray | None = None
        self._host_valid = False   # host mirror equals the device array
        self._host_lent = False    # caller holds a writable host view

    # -- device side -------------------------------------------------------------
    @property
    def device(self) -> torch.device:
        if self._device is None:
            from ._device import require_cuda

            self._device = require_cuda()
        return self._device

    @property
    def d_words(self) -> torch.Tensor:
        """The device words, current (uploads host edits first)."""
        if self._d_words is None:
            self._d_words = torch.zeros(self.num_words, dtype=torch.uint64, device=self.device)
        if self._host_lent:
            self._d_words.copy_(torch.from_numpy(self._host))
            self._host_lent = False
        return self._d_words

    def device_modified(self) -> None:
        """Called after a kernel wrote ``d_words``."""
        self._host_valid = False

    # -- host mirror ---------------------------------------------------------------
    def _synced_host(self) -> np.ndarray:
        """The host mirror, current; lending is the caller's business."""
        if self._host is None:
            self._host = np.zeros(self.num_words, dtype=np.uint64)
            self._host_valid = self._d_words is None
        if not self._host_valid:
            self._host[:] = self._d_words.cpu().numpy()
            self._host_valid = True
        return self._host

    @property
    def words(self) -> np.ndarray:
        """The host mirror, writable like the reference's numpy attribute
        (its tests write through it, test_filters.py:103): it is lent out, and
        the next device operation uploads it."""
        host = self._synced_host()
        self._host_lent = True
        return host

    def words_readonly(self) -> np.ndarray:
        """A read-only view of the current host mirror; reading does not
        force the next device operation to re-upload the filter."""
        v = self._synced_host().view()
        v.flags.writeable = False
        return v

    def load_words(self, words: np.ndarray) -> None:
        words = np.asarray(words, dtype=np.uint64)
        if words.shape != (self.num_words,):
            raise ValueError("word array does not match the filter geometry")
        self.words[:] = words

    @property
    def total_bits(self) -> int:
        return self.num_blocks * self.block_bits

    # -- scalar primitives on the host mirror (the reference's per-key API) ---------
    def _addresses(self, block: int, addrs) -> np.ndarray:
        """Validated bit addresses as an int64 array (IndexError like the
        reference for a bad block or address)."""
        if not 0 <= block < self.num_blocks:
            raise IndexError(f"block {block} out of range [0, {self.num_blocks})")
        vals = [int(v) for v in addrs]
        first_bad = next((v for v in vals if not 0 <= v < self.block_bits), None)
        if first_bad is not None:
            raise IndexError(f"bit address {first_bad} out of range [0, {self.block_bits})")
        return np.array(vals, dtype=np.int64)

    def _mask_of(self, a: np.ndarray) -> np.ndarray:
        m = np.zeros(self.words_per_block, dtype=np.uint64)
        np.bitwise_or.at(m, a >> 6, np.left_shift(np.uint64(1), (a & 63).astype(np.uint64)))
        return m

    def block_words(self, block: int) -> np.ndarray:
        """Writable view of one block's words on the host mirror."""
        lo = block * self.words_per_block
        return self.words[lo:lo + self.words_per_block]

    def _block_readonly(self, block: int) -> np.ndarray:
        lo = block * self.words_per_block
        return self.words_readonly()[lo:lo + self.words_per_block]

    def set_bits(self, block: int, addrs) -> None:
        m = self._mask_of(self._addresses(block, addrs))
        np.bitwise_or(self.block_words(block), m, out=self.block_words(block))

    def test_all(self, block: int, addrs) -> bool:
        m = self._mask_of(self._addresses(block, addrs))
        return not np.any(m & ~self._block_readonly(block))

    def popcount_block(self, block: int) -> int:
        self._addresses(block, ())
        return int(np.bitwise_count(self._block_readonly(block)).sum())

    def simulate_insertion(self, block: int, addrs) -> tuple:
        """(j, a): set bits after inserting ``addrs`` and how many of them are
        new; the block is left untouched (a == 0: all already set)."""
        m = self._mask_of(self._addresses(block, addrs))
        view = self._block_readonly(block)
        new = int(np.bitwise_count(m & ~view).sum())
        return int(np.bitwise_count(view).sum()) + new, new

    def histogram(self) -> np.ndarray:
        """counts[j] = blocks with j set bits, on the GPU."""
        from ._device import histogram

        return histogram(self.d_words, self.num_blocks, self.block_bits)

    def total_set_bits(self) -> int:
        if self._host_valid or self._d_words is None:
            return int(popcount_words(self.words_readonly()).sum())
        counts = self.histogram()
        return int((np.arange(counts.shape[0], dtype=np.int64) * counts).sum())
