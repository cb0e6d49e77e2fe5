"""Filter files (BWCH v1) and key input streams (reference io.py:1-121, 182-267).

The file format is the reference's, byte for byte (pinned by the reference's
test_io.py:70-86 and by tests/test_io_format.py here):

    0  4s  magic "BWCH"          24 Q  block width in bits
    4  I   version (1)           32 Q  number of blocks
    8  B   kind 0/1/2            40 Q  shard count
    9  H   k                     48 Q  seed
    11 B   choices               56 Q  keys inserted
    12 B   strategy 0/1          64 ... bit array: blocks in order, 64-bit
    13 B   cost kind 0/1/2               little-endian words, LSB first
    14 2x  reserved
    16 d   cost parameter

Filters live in HBM; ``write_filter`` streams the device words to the file in
slices and ``read_filter`` streams them back, so multi-GiB filters never need
a second full host copy.  Hash functions are re-derived from the stored seed.
"""

from __future__ import annotations

import ctypes
import struct
import sys
from typing import BinaryIO, Iterator

import numpy as np

from . import _native
from .filters import CostModel, Filter
from .qgrams import QGramEncoder, encode_qgrams, join_records

MAGIC = b"BWCH"
FORMAT_VERSION = 1
HEADER = struct.Struct("<4sIBHBBB2xdQQQQQ")
assert HEADER.size == 64

KIND_CODES = {"standard": 0, "blocked": 1, "blowchoc": 2}
STRATEGY_CODES = {"random": 0, "distinct": 1}
COST_CODES = {"exp": 0, "mix": 1, "la": 2}
KEY_FORMATS = ("u64le", "text", "fasta")

_SLICE_WORDS = 1 << 24  # 128 MiB per device<->file transfer


class FilterFormatError(Exception):
    """The file is not a valid filter of a supported version."""


class KeyFormatError(Exception):
    """A key input stream could not be decoded."""


def _inverse(d: dict) -> dict:
    return {v: k for k, v in d.items()}


def write_filter(filt: Filter, path) -> None:
    if filt.block_bits % 64 != 0:
        raise ValueError("only word-multiple block widths serialize")
    code, param = (COST_CODES[filt.cost.kind], float(filt.cost.param)) if filt.cost else (0, 0.0)
    header = HEADER.pack(MAGIC, FORMAT_VERSION, KIND_CODES[filt.kind], filt.k, filt.choices,
                         STRATEGY_CODES[filt.strategy], code, param, filt.block_bits,
                         filt.num_blocks, filt.shards, filt.seed, filt.inserted)
    st = filt.storage
    with open(path, "wb") as fh:
        fh.write(header)
        if st._d_words is None or st._host_valid:
            fh.write(np.ascontiguousarray(st.words_readonly(), dtype="<u8").tobytes())
            return
        d = st.d_words
        if sys.byteorder != "little":
            for a in range(0, st.num_words, _SLICE_WORDS):
                b = min(st.num_words, a + _SLICE_WORDS)
                fh.write(d[a:b].cpu().numpy().astype("<u8", copy=False).tobytes())
            return
        # two pinned slices: the device->host copy of slice i runs under the
        # file write of slice i - 1, and the file is written from the pinned
        # buffer itself (no bytes copies)
        import torch

        pins, evs = _pinned_slices(min(st.num_words, _SLICE_WORDS))
        prev = None  # (buffer index, words)
        for i, a in enumerate(range(0, st.num_words, _SLICE_WORDS)):
            b = min(st.num_words, a + _SLICE_WORDS)
            pins[i % 2][:b - a].copy_(d[a:b].view(torch.int64), non_blocking=True)
            evs[i % 2].record()
            if prev is not None:
                evs[prev[0]].synchronize()
                fh.write(memoryview(pins[prev[0]].numpy())[:prev[1]])
            prev = (i % 2, b - a)
        if prev is not None:
            evs[prev[0]].synchronize()
            fh.write(memoryview(pins[prev[0]].numpy())[:prev[1]])


def _pinned_slices(nwords: int):
    """Two page-locked int64 buffers of nwords and an event for each."""
    import torch

    pins = [torch.empty(nwords, dtype=torch.int64, pin_memory=True) for _ in range(2)]
    evs = [torch.cuda.Event() for _ in range(2)]
    return pins, evs


def _check_header(fields) -> tuple:
    (magic, version, kind_code, k, choices, strategy_code, cost_code, cost_param,
     block_bits, num_blocks, shards, seed, inserted) = fields
    if magic != MAGIC:
        raise FilterFormatError(f"bad magic {magic!r}")
    if version != FORMAT_VERSION:
        raise FilterFormatError(f"unsupported format version {version}")
    kinds, strategies, costs = _inverse(KIND_CODES), _inverse(STRATEGY_CODES), _inverse(COST_CODES)
    if kind_code not in kinds or strategy_code not in strategies or cost_code not in costs:
        raise FilterFormatError("unknown enum value in header")
    if (block_bits == 0 or block_bits % 64 or num_blocks == 0 or shards == 0
            or num_blocks % shards or not 1 <= k <= block_bits):
        raise FilterFormatError("inconsistent filter geometry")
    kind = kinds[kind_code]
    ok = {"standard": choices == 0, "blocked": choices == 1,
          "blowchoc": 2 <= choices <= 8}[kind]
    if not ok:
        raise FilterFormatError(f"{kind} filter with {choices} choices")
    if kind == "standard" and shards != 1:
        raise FilterFormatError("standard filters do not shard")
    cost = CostModel(costs[cost_code], cost_param, k) if kind == "blowchoc" else None
    return (kind, k, choices, strategies[strategy_code], cost, block_bits, num_blocks, shards,
            seed, inserted)


def read_filter(path, **kw) -> Filter:
    with open(path, "rb") as fh:
        raw = fh.read(HEADER.size)
        if len(raw) < HEADER.size:
            raise FilterFormatError("truncated header")
        (kind, k, choices, strategy, cost, block_bits, num_blocks, shards, seed,
         inserted) = _check_header(HEADER.unpack(raw))
        nbytes = num_blocks * block_bits // 8
        try:
            filt = Filter(kind=kind, k=k, choices=choices, strategy=strategy, cost=cost,
                          block_bits=block_bits, num_blocks=num_blocks, shards=shards,
                          seed=seed, inserted=inserted, **kw)
        except ValueError as exc:
            raise FilterFormatError(str(exc)) from exc
        st = filt.storage
        import torch

        on_device = torch.cuda.is_available()
        host = None if on_device else np.empty(st.num_words, dtype=np.uint64)
        got = 0
        if on_device and sys.byteorder == "little":
            # the file is read straight into two pinned slices; the host->device
            # copy of slice i runs under the read of slice i + 1
            pins, evs = _pinned_slices(min(st.num_words, _SLICE_WORDS))
            dw = st.d_words.view(torch.int64)
            for i, a in enumerate(range(0, st.num_words, _SLICE_WORDS)):
                b = min(st.num_words, a + _SLICE_WORDS)
                evs[i % 2].synchronize()  # its last copy out of this buffer is done
                view = memoryview(pins[i % 2].numpy()).cast("B")[:(b - a) * 8]
                n = 0
                while n < len(view):  # short reads (pipes) are topped up
                    r = fh.readinto(view[n:])
                    if not r:
                        break
                    n += r
                got += n
                if n != (b - a) * 8:
                    raise FilterFormatError(f"bit array has {got} bytes, expected {nbytes}")
                dw[a:b].copy_(pins[i % 2][:b - a], non_blocking=True)
                evs[i % 2].record()
            torch.cuda.current_stream().synchronize()
        else:
            for a in range(0, st.num_words, _SLICE_WORDS):
                b = min(st.num_words, a + _SLICE_WORDS)
                chunk = fh.read((b - a) * 8)
                got += len(chunk)
                if len(chunk) != (b - a) * 8:
                    raise FilterFormatError(f"bit array has {got} bytes, expected {nbytes}")
                words = np.frombuffer(chunk, dtype="<u8").astype(np.uint64)
                if on_device:
                    st.d_words[a:b].copy_(torch.from_numpy(words))
                else:
                    host[a:b] = words
        if fh.read(1):
            raise FilterFormatError(f"bit array has more than {nbytes} bytes, expected {nbytes}")
    if on_device:
        st.device_modified()
    else:
        st.load_words(host)
    return filt


# -- key streams -----------------------------------------------------------------------

def _open_binary(path) -> BinaryIO:
    return sys.stdin.buffer if path == "-" else open(path, "rb")


def _read_u64le(fh: BinaryIO, chunk: int) -> Iterator[np.ndarray]:
    """Raw little-endian records; short reads (pipes) are topped up, and a
    stream whose length is not a multiple of 8 is an error (io.py:191-203)."""
    if sys.byteorder != "little" or not hasattr(fh, "readinto"):
        buf = bytearray()
        want = chunk * 8
        while True:
            got = fh.read(want - len(buf))
            if got:
                buf += got
            if len(buf) >= want or (not got and len(buf) >= 8):
                whole = len(buf) - len(buf) % 8
                yield np.frombuffer(bytes(buf[:whole]), dtype="<u8").astype(np.uint64)
                del buf[:whole]
            if not got:
                break
        if buf:
            raise KeyFormatError(f"u64le stream truncated ({len(buf)} stray bytes)")
        return
    # read straight into each chunk's array (no bytes objects in between)
    stray = b""
    while True:
        arr = np.empty(chunk, dtype=np.uint64)
        view = memoryview(arr).cast("B")
        view[:len(stray)] = stray
        n = len(stray)
        eof = False
        while n < len(view):
            r = fh.readinto(view[n:])
            if not r:
                eof = True
                break
            n += r
        whole = n - n % 8
        stray = bytes(view[whole:n])
        if whole:
            yield arr[:whole // 8]
        if eof:
            break
    if stray:
        raise KeyFormatError(f"u64le stream truncated ({len(stray)} stray bytes)")


_TEXT_BLOCK = 1 << 24  # bytes per native parse call


def _text_error(line: bytes, lineno: int) -> KeyFormatError:
    """The reference's wording for a rejected line (io.py:206-223)."""
    line = line.strip()
    try:
        value = int(line)
    except ValueError:
        return KeyFormatError(f"line {lineno}: not an integer: {line!r}")
    return KeyFormatError(f"line {lineno}: key out of 64-bit range: {value}")


def _read_text(fh: BinaryIO, chunk: int) -> Iterator[np.ndarray]:
    """One decimal key per line, parsed natively (bc_parse_keys_text) in
    blocks of whole lines; keys are yielded in batches of up to ``chunk``."""
    lib = _native.lib()
    out = np.empty(chunk, dtype=np.uint64)
    used = ctypes.c_uint64()
    nlines = ctypes.c_uint64()
    nkeys = ctypes.c_uint64()
    fill = 0
    lineno = 1  # number of the first line still to parse
    # one reusable block: the unparsed tail of the last read moves to its front
    # and the file is read in behind it (no bytes objects, no concatenation)
    buf = bytearray(_TEXT_BLOCK + 4096)
    ntail = 0
    eof = False
    while not eof:
        if ntail + _TEXT_BLOCK + 1 > len(buf):  # a line longer than the slack
            buf.extend(bytes(ntail + _TEXT_BLOCK + 1 - len(buf)))
        mv = memoryview(buf)
        got = _readinto(fh, mv[ntail:ntail + _TEXT_BLOCK])
        mv.release()
        eof = got == 0
        n = ntail + got
        if eof:
            if not n:
                break
            buf[n:n + 1] = b"\n"  # the last line needs no newline
            n += 1
        view = np.frombuffer(buf, dtype=np.uint8)
        off = 0
        while off < n:
            rc = lib.bc_parse_keys_text(view.ctypes.data + off, n - off,
                                        out.ctypes.data + 8 * fill, chunk - fill,
                                        ctypes.byref(used), ctypes.byref(nlines),
                                        ctypes.byref(nkeys))
            fill += nkeys.value
            if rc != _native.BC_OK:
                start = off + used.value
                stop = buf.find(b"\n", start, n)
                raise _text_error(bytes(buf[start:stop]), lineno + nlines.value)
            off += used.value
            lineno += nlines.value
            if fill < chunk:
                break  # every whole line is parsed; a partial one may remain
            yield out.copy()
            fill = 0
        del view
        ntail = n - off
        buf[:ntail] = buf[off:n]
    if fill:
        yield out[:fill].copy()


def _readinto(fh: BinaryIO, view) -> int:
    """Fill view from fh (short reads of pipes topped up); bytes read."""
    n = 0
    while n < len(view):
        r = fh.readinto(view[n:])
        if not r:
            break
        n += r
    return n


def fasta_records(fh: BinaryIO) -> Iterator[bytes]:
    """Sequence of each FASTA record (lines joined, header dropped)."""
    parts: list = []
    seen = False
    for line in fh:
        line = line.strip()
        if line.startswith(b">"):
            if parts:
                yield b"".join(parts)
                parts = []
            seen = True
        elif line:
            if not seen:
                raise KeyFormatError("FASTA input does not start with a header line")
            parts.append(line)
    if parts:
        yield b"".join(parts)


def _fasta_joined(fh: BinaryIO, read_bytes: int = 1 << 24):
    """Records of a FASTA stream joined natively (bc_fasta_join: one memchr +
    memcpy per line instead of a Python loop over lines).  Yields (buf, ends):
    the records closed by one read, joined with b"\\n" in the uint8 array buf,
    ends[i] = end offset of record i.  A record still open at the end of a read
    is carried into the next one, so records are never split."""
    lib = _native.lib()
    state = ctypes.c_uint32(0)
    counters = (ctypes.c_uint64 * 3)()  # out_len, n_recs, consumed
    carry_text = b""
    carry_rec = np.empty(0, dtype=np.uint8)

    def join(buf, off, eof, out, out_len, ends, n_ends):
        """Parse buf[off:] (bytes); returns (out_len, ends, n_ends, bytes used)."""
        view = np.frombuffer(buf, dtype=np.uint8)
        used = 0
        while True:
            rc = lib.bc_fasta_join(view.ctypes.data + off + used, len(buf) - off - used,
                                   int(eof), 0x0A, ctypes.byref(state), out.ctypes.data,
                                   out_len, ctypes.byref(counters, 0),
                                   ends.ctypes.data + 8 * n_ends, ends.size - n_ends,
                                   ctypes.byref(counters, 8), ctypes.byref(counters, 16))
            if rc != _native.BC_OK:
                raise KeyFormatError(lib.bc_last_error().decode(errors="replace"))
            out_len = int(counters[0])
            n_ends += int(counters[1])
            used += int(counters[2])
            if n_ends < ends.size:
                return out_len, ends, n_ends, used
            # record table full: more space, and on from the line it stopped at
            ends = np.concatenate([ends, np.empty(max(1024, ends.size), dtype=np.uint64)])

    while True:
        data = fh.read(read_bytes)
        eof = not data
        ends = np.empty(1024 + len(data) // 4096, dtype=np.uint64)
        out = np.empty(carry_rec.size + len(carry_text) + len(data) + 2, dtype=np.uint8)
        out[:carry_rec.size] = carry_rec
        out_len, n = carry_rec.size, 0
        # the line the last read cut in two, completed with the head of this one
        # (only that line is copied; the rest of the read is parsed in place)
        nl = data.find(b"\n")
        if eof or nl < 0:
            head, off = carry_text + data, len(data)
        else:
            head, off = carry_text + data[:nl + 1], nl + 1
        out_len, ends, n, used = join(head, 0, eof, out, out_len, ends, n)
        carry_text = head[used:]
        if off < len(data):
            out_len, ends, n, used = join(data, off, False, out, out_len, ends, n)
            carry_text = data[off + used:]
        closed = int(ends[n - 1]) if n else 0
        if state.value & 2:  # the last record goes on in the next read
            start = closed + 1 if n else 0
            carry_rec = out[start:out_len].copy()
        else:
            carry_rec = np.empty(0, dtype=np.uint8)
        if n:
            yield out[:closed], ends[:n]
        if eof:
            return


def _prefetched(gen, depth: int):
    """Run a generator in a background thread, `depth` items ahead of the
    consumer (file reads and bc_fasta_join release the GIL, so parsing the
    next batch overlaps the consumer's copy and insert of this one).  Returns
    (iterator, stop): stop() ends the thread before the caller closes what
    the generator reads from."""
    import queue
    import threading

    q: queue.Queue = queue.Queue(maxsize=depth)
    halt = threading.Event()
    end = object()

    def put(item) -> bool:
        while not halt.is_set():
            try:
                q.put(item, timeout=0.05)
                return True
            except queue.Full:
                continue
        return False

    def work():
        try:
            for item in gen:
                if not put(item):
                    return
            put(end)
        except BaseException as exc:  # handed to the consumer
            put(exc)

    thread = threading.Thread(target=work, name="fasta-prefetch", daemon=True)
    thread.start()

    def items():
        while True:
            item = q.get()
            if item is end:
                return
            if isinstance(item, BaseException):
                raise item
            yield item

    def stop():
        halt.set()
        thread.join()

    return items(), stop


def fasta_batches(path, batch_bytes: int = 1 << 28, as_array: bool = False,
                  prefetch: int = 0) -> Iterator[bytes]:
    """FASTA records joined (join_records) into batches of about batch_bytes,
    for the fused q-gram kernels: the windows of a batch are those of its
    records, in order, and none spans two records.  as_array: yield uint8
    views of the parser's buffer instead of bytes copies.  prefetch: batches
    parsed ahead in a background thread (0, the default: parse in the caller's
    thread).  Measured on the B200 box with the fused insert as consumer
    (tools/fasta_prefetch_probe.py): 2 000 Mbp/s against 1 170-1 350 serial in
    one process, but 1 969 / 709 / 582 over three runs of tools/bench_next.py
    (bimodal, presumably where the parser thread's buffers land relative to
    the GPU's host bridge), so it stays opt-in."""
    fh = _open_binary(path)

    def batches():
        for buf, ends in _fasta_joined(fh):
            a = 0  # offset of the batch's first record
            i = 0
            while i < ends.size:
                # first record whose end brings the batch to batch_bytes
                # (each record counts its length plus one, as join_records would)
                j = int(np.searchsorted(ends, a + batch_bytes - 1, side="left"))
                j = min(max(j, i), ends.size - 1)
                e = int(ends[j])
                yield buf[a:e] if as_array else buf[a:e].tobytes()
                a, i = e + 1, j + 1

    stop = None
    try:
        if prefetch > 0:
            it, stop = _prefetched(batches(), prefetch)
            yield from it
        else:
            yield from batches()
    finally:
        if stop is not None:
            stop()
        if fh is not sys.stdin.buffer:
            fh.close()


def read_keys(path, fmt: str, *, q: int | None = None, canonical: bool = True,
              chunk_size: int = 1 << 20) -> Iterator[np.ndarray]:
    """Key chunks from a file ('-' = stdin): raw u64le, decimal text, or the
    q-grams of each FASTA record (encoded on the GPU)."""
    if fmt not in KEY_FORMATS:
        raise KeyFormatError(f"unknown key format {fmt!r}")
    if fmt == "fasta":
        if q is None:
            raise KeyFormatError("FASTA input needs a q-gram length")
        enc = QGramEncoder(q=q, canonical=canonical)
    fh = _open_binary(path)
    try:
        if fmt == "u64le":
            yield from _read_u64le(fh, chunk_size)
        elif fmt == "text":
            yield from _read_text(fh, chunk_size)
        else:
            for rec in fasta_records(fh):
                yield encode_qgrams(enc, rec)
    finally:
        if fh is not sys.stdin.buffer:
            fh.close()
