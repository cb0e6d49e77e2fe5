"""DNA q-gram keys (reference io.py:126-177).

``encode_qgrams`` runs on the GPU (``bc_encode_qgrams``).  The filter's
``insert_qgrams`` / ``contains_qgrams`` fuse encoding with hashing and probing
so the key array is never materialised.  Several records can be encoded in
one call by joining them with a separator byte (``join_records``): a window
that touches a non-ACGT byte is skipped, so no window spans two records --
exactly the per-record behaviour of the reference's FASTA reader
(io.py:226-241).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class QGramEncoder:
    """2-bit packing of DNA q-grams: A=0 C=1 G=2 T=3, first base most
    significant; ``canonical`` keeps min(code, reverse complement)."""

    q: int
    canonical: bool = True

    def __post_init__(self):
        if not 1 <= self.q <= 32:
            raise ValueError(f"q must be in [1, 32], got {self.q}")


def encode_qgrams(enc: QGramEncoder, sequence, record_len: int | None = None):
    """All valid q-gram keys of a sequence, in sequence order (GPU).  A 2-D
    byte array (reads x length), or ``record_len``, marks fixed-length records
    that no window may cross."""
    from ._device import encode_qgrams as _enc

    return _enc(sequence, enc.q, enc.canonical, record_len)


def join_records(records, sep: bytes = b"\n") -> bytes:
    """Concatenate records so that no q-gram window spans two of them."""
    if len(sep) != 1 or sep.upper() in b"ACGT":
        raise ValueError("separator must be one non-ACGT byte")
    return sep.join(r.encode("ascii") if isinstance(r, str) else bytes(r) for r in records)


def record_slices(records, q: int) -> np.ndarray:
    """Per-record [start, end) offsets into the concatenated answer array of
    ``contains_qgrams(enc, join_records(records))`` (host arithmetic on the
    record lengths; assumes records are pure ACGT)."""
    n = np.array([max(0, len(r) - q + 1) for r in records], dtype=np.int64)
    ends = np.cumsum(n)
    return np.stack([ends - n, ends], axis=1)
