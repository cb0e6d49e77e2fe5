"""Command-line front end on the GPU API: ``build``, ``query``, ``fpr`` and
``hist`` with the reference's arguments, TSV output and exit codes
(reference ``blowchoc/cli.py:118-171,253-330``).

    python -m paper_2501_18977_b200 build --kind blowchoc --k 14 --choices 2 \
        --n 1000000 --keys keys.u64 --out f.bwch
    python -m paper_2501_18977_b200 query --filter f.bwch --keys probes.txt --format text

Exit codes: 0 ok, 1 usage error, 2 input/output error, 3 corrupt filter file.
Per-key query output (``key<TAB>0|1``) is formatted by native code
(bc_format_answers) instead of one Python string per key: at GPU lookup
rates the reference's per-key formatting would be the whole cost.
"""

from __future__ import annotations

import argparse
import ctypes
import math
import sys
import time

import numpy as np

from ._native import check, lib
from .analysis import block_load_histogram, estimate_fpr
from .filters import GOLDEN_BETA, ConfigError, CostModel, Filter, FilterConfig
from .io import (FilterFormatError, KeyFormatError, fasta_batches, read_filter, read_keys,
                 write_filter)
from .qgrams import QGramEncoder
from .sharding import build_sharded

EXIT_OK = 0
EXIT_USAGE = 1
EXIT_IO = 2
EXIT_CORRUPT = 3

_DEFAULT_COST_PARAM = {"exp": GOLDEN_BETA, "mix": 1.0, "la": 3.5}


class UsageError(Exception):
    pass


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # exit 1, not argparse's 2 (cli.py:56-58)
        raise UsageError(message)


def _fmt(x) -> str:
    if x is None:
        return "nan"
    if isinstance(x, float):
        return f"{x:.6g}"
    return str(x)


def _tsv(*fields) -> str:
    return "\t".join(_fmt(f) for f in fields)


_FPR_HEADER = _tsv("kind", "k", "c", "strategy", "rel_size", "N", "W", "fpr", "log2_fpr",
                   "stderr")


def format_answers(keys, answers) -> bytes:
    """``"".join(f"{key}\\t{int(ans)}\\n")`` over a key chunk (cli.py:141-142),
    formatted by the native library (bc_format_answers)."""
    keys = np.ascontiguousarray(keys, dtype=np.uint64)
    answers = np.ascontiguousarray(answers, dtype=np.uint8)
    n = keys.shape[0]
    if answers.shape != (n,):
        raise ValueError("one answer per key expected")
    if n == 0:
        return b""
    out = np.empty(23 * n, dtype=np.uint8)
    written = ctypes.c_uint64(0)
    check(lib().bc_format_answers(keys.ctypes.data, answers.ctypes.data, n, out.ctypes.data,
                                  out.nbytes, ctypes.byref(written)))
    return out[:written.value].tobytes()


def _effective_rel_size(filt: Filter) -> float:
    if filt.inserted == 0:
        return float("nan")
    return filt.m * math.log(2) / (filt.inserted * filt.k)


def _make_cost(args, k: int) -> CostModel | None:
    if args.cost is None and args.cost_param is None:
        return None
    kind = args.cost or "exp"
    param = args.cost_param if args.cost_param is not None else _DEFAULT_COST_PARAM[kind]
    return CostModel(kind=kind, param=param, k=k)


def _make_config(args) -> FilterConfig:
    cost = _make_cost(args, args.k)
    if cost is not None and args.kind != "blowchoc":
        raise UsageError("--cost/--cost-param apply to blowchoc filters only")
    # standard filters are never sharded; --threads T gives T shards otherwise
    shards = 1 if args.kind == "standard" else max(1, args.threads)
    return FilterConfig(kind=args.kind, k=args.k, n_capacity=args.n, size_bits=args.size_bits,
                        choices=args.choices, cost=cost, strategy=args.strategy,
                        relative_size=args.relative_size, shards=shards, seed=args.seed)


def _key_stream(args):
    return read_keys(args.keys, args.format, q=args.q, canonical=not args.no_canonical)


def cmd_build(args) -> int:
    config = _make_config(args)
    t0 = time.perf_counter()
    if args.format == "fasta":
        # FASTA: batches of whole records straight into the fused q-gram
        # insert (== inserting encode_qgrams of each record in order)
        if args.q is None:
            raise KeyFormatError("FASTA input needs a q-gram length")
        enc = QGramEncoder(q=args.q, canonical=not args.no_canonical)
        filt = Filter.from_config(config.validated())
        filt.insert_qgram_batches(enc, fasta_batches(args.keys, batch_bytes=1 << 24,
                                                     as_array=True))
    else:
        filt = build_sharded(config, _key_stream(args))
    wall = time.perf_counter() - t0
    write_filter(filt, args.out)
    print(_tsv("keys_inserted", "load", "wall_s", "m_bits", "blocks", "shards"),
          file=sys.stderr)
    print(_tsv(filt.inserted, filt.load(), round(wall, 3), filt.m, filt.num_blocks,
               filt.shards), file=sys.stderr)
    return EXIT_OK


def cmd_query(args) -> int:
    filt = read_filter(args.filter)
    out = sys.stdout
    out.flush()
    for chunk in _key_stream(args):
        answers = filt.contains_many(chunk)
        out.buffer.write(format_answers(chunk, answers))
    out.buffer.flush()
    return EXIT_OK


def cmd_fpr(args) -> int:
    filt = read_filter(args.filter)
    if args.keys is not None:
        est = estimate_fpr(filt, negatives=list(_key_stream(args)))
    else:
        est = estimate_fpr(filt, n_queries=args.negatives, seed=args.neg_seed)
    print(_FPR_HEADER)
    print(_tsv(filt.kind, filt.k, filt.choices, filt.strategy,
               round(_effective_rel_size(filt), 6), est.n_queries, est.false_positives,
               est.fpr, est.log2_fpr, est.stderr))
    return EXIT_OK


def cmd_hist(args) -> int:
    filt = read_filter(args.filter)
    hist = block_load_histogram(filt)
    lines = [_tsv("j", "count")] + [_tsv(j, c) for j, c in enumerate(hist.counts.tolist())]
    print("\n".join(lines))
    print(_tsv("# mean_load", hist.mean_load), file=sys.stderr)
    return EXIT_OK


# Command table: the reference's flags (cli.py:253-330) for the filter
# commands, as (flags, argparse keywords).  "@keys" / "@keys?" expand to the
# key-stream options (required / optional).
_KEY_INPUT = [
    ("--keys", dict(help="key file, '-' for stdin")),
    ("--format", dict(default="u64le", choices=["u64le", "text", "fasta"])),
    ("--q", dict(type=int, default=None, help="q-gram length for fasta")),
    ("--no-canonical", dict(action="store_true", help="keep q-grams strand-specific")),
]
_GPU_THREADS = ("--threads", dict(type=int, default=1, help="accepted; lookups run on the GPU"))
_COMMANDS = {
    "build": ("build a filter from a key stream", [
        ("--kind", dict(required=True, choices=["standard", "blocked", "blowchoc"])),
        ("--k", dict(type=int, required=True, help="bit address functions per key")),
        ("--choices", dict(type=int, default=None)),
        ("--n", dict(type=int, default=None, help="planned key count")),
        ("--size-bits", dict(type=int, default=None, help="filter size in bits instead of --n")),
        ("--relative-size", dict(type=float, default=1.0)),
        ("--cost", dict(choices=["exp", "mix", "la"], default=None)),
        ("--cost-param", dict(type=float, default=None)),
        ("--strategy", dict(choices=["random", "distinct"], default="random")),
        ("--threads", dict(type=int, default=0,
                           help="shards (the reference's worker threads); 0 = unsharded")),
        ("--seed", dict(type=int, default=0)),
        "@keys",
        ("--out", dict(required=True)),
    ], {}),
    "query": ("query keys against a stored filter",
              [("--filter", dict(required=True)), "@keys", _GPU_THREADS], {}),
    "fpr": ("estimate the empirical FPR of a filter", [
        ("--filter", dict(required=True)),
        ("--negatives", dict(type=int, default=10**6,
                             help="generated negative queries (odd keys)")),
        ("--neg-seed", dict(type=int, default=0xFEEDBEEF)),
        _GPU_THREADS,
        "@keys?",
    ], {"keys": None}),
    "hist": ("per-block load histogram of a filter", [("--filter", dict(required=True))], {}),
}
_HANDLERS = {"build": lambda a: cmd_build(a), "query": lambda a: cmd_query(a),
             "fpr": lambda a: cmd_fpr(a), "hist": lambda a: cmd_hist(a)}


def build_parser() -> argparse.ArgumentParser:
    parser = _Parser(prog="paper_2501_18977_b200", description=__doc__,
                     formatter_class=argparse.RawDescriptionHelpFormatter)
    sub = parser.add_subparsers(dest="command", required=True)
    for name, (help_text, options, defaults) in _COMMANDS.items():
        p = sub.add_parser(name, help=help_text)
        for opt in options:
            if isinstance(opt, str):  # the key-stream group
                for flag, kw in _KEY_INPUT:
                    kw = dict(kw, required=True) if flag == "--keys" and opt == "@keys" else kw
                    p.add_argument(flag, **kw)
            else:
                p.add_argument(opt[0], **opt[1])
        p.set_defaults(func=_HANDLERS[name], **defaults)
    return parser


def main(argv=None) -> int:
    parser = build_parser()
    try:
        args = parser.parse_args(argv)
        return args.func(args)
    except (UsageError, ConfigError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_USAGE
    except FilterFormatError as exc:
        print(f"error: corrupt filter file: {exc}", file=sys.stderr)
        return EXIT_CORRUPT
    except KeyFormatError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_IO
    except OSError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_IO


def entry() -> None:
    sys.exit(main(sys.argv[1:]))


if __name__ == "__main__":
    entry()
