"""Throughput of the insert / lookup hot path on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

A step is one pass of the hot path over one batch of synthetic input: build
the filter from zero (insert the config's n keys) and answer the config's
lookup batch.  The default workload is BASELINE.json configs[4] (config 5),
the largest single-GPU configuration and the one the metric's 1/2/4/8-GPU
clause is quoted on: a 2-choice 8 GiB filter (k = 11), 1.2 x 2^32 keys
inserted, 2^34 lookups (50% positive) sharded across the GPUs.  Keys are the
reference's own streams (even_keys(n, 11) / odd_keys(., 12), analysis.py:34-43)
generated on the device bit-identically to numpy.

``value``: keys (inserted + looked up) per second over the timed steps,
inputs resident in HBM.  ``e2e``: the same step through the public API
(Filter.insert_many / contains_many) from page-locked host buffers, every
key crossing the host link inside the timed region.  ``--impl reference``
times the reference itself -- the numba ``blowchoc`` package installed in
baseline/_ref -- on the box's host cores, each step a bounded sample of the
workload with the same insert : lookup mix.

Multi-GPU (torchrun, one rank per GPU, NCCL; strong scaling): the 2^34
lookups are split across the ranks, each answering its share on a replica of
the filter; the build is done on rank 0 and NCCL-broadcast (c >= 2 with
T = 1: the reference layout has no subfilters), or, for
order-free kinds (c = 1, standard), from per-rank key slices followed by an
OR all-reduce of the replicas.  value = all keys / max-over-ranks step time;
the lookup-only rate and the broadcast time are reported beside it.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# cfg5 holds ~130 GB of inputs in a few large tensors: avoid caching-allocator
# fragmentation between them
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")

METRIC = "insert & lookup Mkeys/s (1/2/4/8 B200); FPR; % of random-sector HBM roofline"

# BASELINE.json configs; lookup bytes/unit from SURVEY §8(d).  ``slice``: keys
# per lookup launch; ``distinct``: resident query slices per rank (cfg5's
# 2^34 lookups do not fit HBM next to its 41 GB of insert keys, so the step's
# four 2^32-key slices alternate between two resident query sets; each is
# 34 GB, far above L2).
CONFIGS = {
    1: dict(workload="cfg1: blowchoc c=2 k=14 16 b/key, 2^20 keys, 2^21 lookups (50% pos)",
            kind="blowchoc", c=2, k=14, n=2**20, bpk=16, nq=2**21, ref_keys=True,
            lookup_bytes=120.6),
    2: dict(workload="cfg2: blocked c=1 k=12 12 b/key (96 MiB), 2^26 keys, 2^27 lookups "
                     "(50% pos, shuffled)",
            kind="blocked", c=1, k=12, n=2**26, bpk=12, nq=2**27, ref_keys=True,
            lookup_bytes=73.0),
    3: dict(workload="cfg3: blowchoc c=3 k=16 16 b/key (512 MiB), 2^28 keys, 2^30 lookups "
                     "(50% pos, shuffled)",
            kind="blowchoc", c=3, k=16, n=2**28, bpk=16, nq=2**30, ref_keys=False,
            lookup_bytes=168.3),
    4: dict(workload="cfg4: DNA, seeded i.i.d. 1.2e9-bp genome, canonical 31-mers into "
                     "blowchoc c=2 k=14 at 14 b/key; lookups of 1e8 150-bp reads with 1% "
                     "substitutions + 1e8 reads of an independent genome (count-only)",
            kind="blowchoc", c=2, k=14, dna=True, genome=1_200_000_000, reads=10**8,
            read_len=150, sub=0.01, q=31, ref_keys=False, lookup_bytes=117.0),
    5: dict(workload="cfg5: blowchoc c=2 k=11 8 GiB, 1.2*2^32 keys inserted, 2^34 lookups "
                     "(50% pos) sharded across the GPUs",
            kind="blowchoc", c=2, k=11, n=int(1.2 * 2**32), size_bits=2**36, nq=2**34,
            slice=2**32, distinct=2, ref_keys=False, lookup_bytes=119.6),
}
DEFAULT_CONFIG = 5


def insert_bytes(c: int) -> float:
    return 8 + 64 * c + 64  # key + c candidate reads + one block write-back


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--insert-mode", default=None, choices=["ordered", "relaxed"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the untimed extras (exact-order insert rate, FPR curve)")
    ap.add_argument("--reads", type=int, default=None, help="config 4: reads per set")
    return ap.parse_args()


# -- distributed plumbing ---------------------------------------------------------------

# launched by torchrun (even with one rank): use torch.distributed / NCCL
DIST = "RANK" in os.environ and "LOCAL_RANK" in os.environ


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def host_mem_available() -> int:
    try:
        with open("/proc/meminfo") as fh:
            for line in fh:
                if line.startswith("MemAvailable:"):
                    return int(line.split()[1]) * 1024
    except OSError:
        pass
    return 0


def lookup_plan(cfg: dict, world: int) -> dict:
    """Per-rank lookup share of the step (strong scaling: the config's lookup
    batch is split across the ranks) and how it is laid out in launches."""
    per_rank = cfg["nq"] // world
    sl = min(cfg.get("slice", per_rank), per_rank)
    nslices = per_rank // sl
    distinct = min(cfg.get("distinct", 1), nslices)
    return dict(per_rank=per_rank, slice=sl, nslices=nslices, distinct=distinct)


# -- synthetic inputs ---------------------------------------------------------------------

def make_keys(cfg: dict, device):
    """The config's insert keys on the device: even_keys(n, 11)."""
    import torch

    from paper_2501_18977_b200 import even_keys

    if cfg["ref_keys"]:
        return torch.from_numpy(even_keys(cfg["n"], 11)).to(device)
    return even_keys(cfg["n"], 11, device=device)


def make_queries(cfg: dict, keys, plan: dict, rank: int, device):
    """``distinct`` query slices of this rank: 50% uniform samples of the
    inserted keys, 50% fresh odd keys (odd_keys(., 12 + rank) at disjoint
    stream offsets), mixed by a seeded coin; returns (slices, positive masks)."""
    import torch

    from paper_2501_18977_b200 import odd_keys

    n = keys.numel()
    sl = plan["slice"]
    g = torch.Generator(device=device).manual_seed(1234 + rank)
    span = 1 << 28
    kv = keys.view(torch.int64)
    qs, pos = [], []
    for d in range(plan["distinct"]):
        q = torch.empty(sl, dtype=torch.int64, device=device)
        sel = torch.empty(sl, dtype=torch.bool, device=device)
        for a in range(0, sl, span):
            b = min(sl, a + span)
            s = torch.randint(0, 2, (b - a,), device=device, dtype=torch.int64,
                              generator=g).bool()
            idx = torch.randint(0, n, (b - a,), device=device, dtype=torch.int64, generator=g)
            neg = odd_keys(b - a, 12 + rank, device=device, offset=d * sl + a).view(torch.int64)
            q[a:b] = torch.where(s, kv[idx], neg)
            sel[a:b] = s
            del s, idx, neg
        qs.append(q.view(torch.uint64))
        pos.append(sel)
    return qs, pos


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled while the timed region runs."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.12)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
            out, _ = self.proc.communicate()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        loaded = [v for v in sm if smax and v > 0.5 * smax] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": smax, "samples": len(sm), "reasons": sorted(reasons)}


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured copy, burst)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


def random_ceiling(filter_bytes: int):
    """Measured random 64-byte-gather ceiling (tools/gather_probe.cu, ld.global.cg,
    profiles/r1/gather_probe_*.txt) for the nearest filter size, in algorithmic
    GB/s of the lookup pattern (64 B block + 8 B key + 1 B answer)."""
    table = [(96 << 20, 7011.0), (512 << 20, 3145.0), (2 << 30, 2551.0), (8 << 30, 2415.0)]
    best = min(table, key=lambda t: abs(np.log2(t[0]) - np.log2(max(filter_bytes, 1))))
    return best[1], f"tools/gather_probe.cu at {best[0] >> 20} MiB (profiles/r1)"


def profiled_traffic(config: int, kernel: str):
    """DRAM bytes per launch of ``kernel`` from the committed ncu summary."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return d.get(f"cfg{config}", {}).get(kernel)
    except (OSError, ValueError):
        return None


# -- CPU side: the reference itself (baseline/_ref), and the oracle port ---------------

REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def import_reference():
    """The unmodified reference package (numba), installed in baseline/_ref."""
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_bench")
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import blowchoc

    if not os.path.abspath(blowchoc.__file__).startswith(REF_DIR):
        raise ImportError(f"blowchoc resolved outside baseline/_ref: {blowchoc.__file__}")
    return blowchoc


# fill density of the built filter (reference-measured, SURVEY §8(d) / BASELINE §2)
# and the AND/OR recipe of uniform random words that stands in for it
PREFILL = {2: (0.628, "a|b&c", 0.625), 3: (0.577, "a|b&c", 0.625),
           4: (0.60, "a|b&c", 0.625), 5: (0.56, "a|b&c&d", 0.5625)}


def prefill_words(words: np.ndarray, cfgno: int, seed: int = 99) -> str:
    """Random bits at the built filter's load, in place (bounded CPU samples
    cannot build a multi-GiB filter first)."""
    target, recipe, dens = PREFILL[cfgno]
    rng = np.random.default_rng(seed)
    tile = min(words.shape[0], 1 << 24)
    r = [rng.integers(0, 2**64, size=tile, dtype=np.uint64) for _ in range(recipe.count("&") + 2)]
    acc = r[1]
    for x in r[2:]:
        acc &= x
    pattern = r[0] | acc
    for a in range(0, words.shape[0], tile):
        m = min(tile, words.shape[0] - a)
        words[a:a + m] = pattern[:m]
    return (f"prefilled with random bits at density {dens} ({recipe} of uniform words, a "
            f"{tile}-word tile repeated) for the built filter's load {target}")


def ref_sample(cfgno: int, cfg: dict, bc, f, step_seed: int, threads: int) -> dict:
    """One bounded step of the reference path: Filter.insert_many of n_s fresh
    keys (one writer, stream order: filters.py:213-216) then contains_many of
    the step's lookup share in the same insert:lookup ratio, 50% positive,
    split over ``threads`` with np.array_split + a thread pool (the
    reference's query parallelism, cli.py:133-140 / analysis.py:96-107)."""
    from concurrent.futures import ThreadPoolExecutor

    n_s = min(cfg["n"], 1 << 21)
    nq_s = int(round(n_s * cfg["nq"] / cfg["n"]))
    keys = bc.even_keys(n_s, 1000 + step_seed)
    rng = np.random.default_rng(step_seed)
    q = np.concatenate([keys[rng.integers(0, n_s, nq_s // 2)],
                        bc.odd_keys(nq_s - nq_s // 2, 2000 + step_seed)])
    rng.shuffle(q)
    parts = np.array_split(q, threads)
    t0 = time.perf_counter()
    f.insert_many(keys)
    t1 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=threads) as pool:
        outs = list(pool.map(f.contains_many, parts))
    t2 = time.perf_counter()
    found = np.concatenate(outs)
    return dict(n_ins=n_s, n_look=nq_s, t_ins=t1 - t0, t_look=t2 - t1, hits=int(found.sum()))


def ref_dna_sample(cfg: dict, bc, f, step_seed: int, threads: int) -> dict:
    """One bounded config-4 step of the reference path: encode_qgrams +
    insert_many of a genome slice, encode_qgrams + contains_many of reads
    (threads over read blocks), k-mer counts in the workload's ratio."""
    from concurrent.futures import ThreadPoolExecutor

    q, RL = cfg["q"], cfg["read_len"]
    enc = bc.QGramEncoder(q, True)
    Lp = 1 << 20
    win = RL - q + 1
    kmers_look = int(round((Lp - q + 1) * 2 * cfg["reads"] * win / (cfg["genome"] - q + 1)))
    R = max(threads, kmers_look // win)
    rng = np.random.default_rng(step_seed)
    alphabet = np.frombuffer(b"ACGT", dtype=np.uint8)
    codes = rng.integers(0, 4, Lp)
    genome = alphabet[codes].tobytes()
    starts = rng.integers(0, Lp - RL, R // 2)
    reads = codes[starts[:, None] + np.arange(RL)]
    sub = rng.random(reads.shape) < cfg["sub"]
    reads = np.where(sub, (reads + rng.integers(1, 4, reads.shape)) % 4, reads)
    rand = rng.integers(0, 4, (R - R // 2, RL))
    blobs = [alphabet[r].tobytes() for r in np.concatenate([reads, rand])]
    # reads joined with '\n' separators: encode_qgrams skips every window
    # touching a non-ACGT byte, so no window spans two reads (io.py:158-177)
    chunks = [b"\n".join(blobs[i::threads]) for i in range(threads)]

    def look(chunk_reads: bytes) -> int:
        return int(f.contains_many(bc.encode_qgrams(enc, chunk_reads)).sum())

    t0 = time.perf_counter()
    keys = bc.encode_qgrams(enc, genome)
    f.insert_many(keys)
    t1 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=threads) as pool:
        hits = sum(pool.map(look, chunks))
    t2 = time.perf_counter()
    return dict(n_ins=int(keys.shape[0]), n_look=R * win, t_ins=t1 - t0, t_look=t2 - t1,
                hits=hits)


def reference_filter(cfgno: int, cfg: dict, bc):
    """The reference's filter at the workload's full geometry; multi-GiB
    filters are prefilled to the built filter's load (see prefill_words)."""
    if cfg.get("dna"):
        kw = dict(kind="blowchoc", k=cfg["k"], choices=cfg["c"],
                  size_bits=cfg["k"] * (cfg["genome"] - cfg["q"] + 1), seed=1)
    else:
        kw = dict(kind=cfg["kind"], k=cfg["k"], choices=cfg["c"], seed=1,
                  size_bits=cfg.get("size_bits", cfg.get("bpk", 0) * cfg["n"]))
    f = bc.Filter.from_config(bc.FilterConfig(**kw))
    state = "built from zero every step (the whole workload)"
    if cfgno in PREFILL:
        state = prefill_words(f.storage.words, cfgno)
    return f, kw, state


def reference_rate(cfgno: int, cfg: dict, steps: int, warmup: int) -> dict:
    """Time the reference (numba, baseline/_ref) on bounded sample steps."""
    bc = import_reference()
    threads = host_cores()
    t_setup = time.perf_counter()
    f, kw, state = reference_filter(cfgno, cfg, bc)
    # JIT compile + touch before timing (the reference's own bench.py:50)
    tiny = bc.Filter.from_config(bc.FilterConfig(**{**kw, "size_bits": 512 * 64}))
    tiny.insert_many(bc.even_keys(16, 1))
    tiny.contains_many(bc.odd_keys(16, 1))
    if cfg.get("dna"):
        bc.encode_qgrams(bc.QGramEncoder(cfg["q"], True), b"ACGT" * 16)
    setup_s = time.perf_counter() - t_setup
    full = cfgno == 1  # cfg1's whole step fits the CPU: rebuild from zero each step
    runs = []
    for i in range(warmup + steps):
        if full:
            f.storage.words[:] = 0
        r = (ref_dna_sample(cfg, bc, f, i, threads) if cfg.get("dna")
             else ref_sample(cfgno, cfg, bc, f, i, threads))
        if i >= warmup:
            runs.append(r)
    n_ins = sum(r["n_ins"] for r in runs)
    n_look = sum(r["n_look"] for r in runs)
    t_ins = sum(r["t_ins"] for r in runs)
    t_look = sum(r["t_look"] for r in runs)
    ms = (t_ins + t_look) / len(runs) * 1e3
    unit = "Mk-mers/s" if cfg.get("dna") else "Mkeys/s"
    return dict(
        value=round((n_ins + n_look) / (t_ins + t_look) / 1e6, 3), unit=unit, cores=threads,
        kind="reference", ms_per_step=round(ms, 2), setup_s=round(setup_s, 1),
        insert_rate=round(n_ins / t_ins / 1e6, 3), lookup_rate=round(n_look / t_look / 1e6, 3),
        sample=(f"reference blowchoc (numba, baseline/_ref) Filter.insert_many of "
                f"{runs[0]['n_ins']} keys (1 writer) + contains_many of {runs[0]['n_look']} "
                f"keys over {threads} threads per step, the workload's insert:lookup ratio; "
                f"full-geometry filter, {state}; value = measured keys / measured seconds"
                f" over {len(runs)} steps (no projection)"),
        cpu=cpu_model())


def port_rate(cfg: dict) -> dict | None:
    """Secondary row: the C restatement (oracle/, test infrastructure) on the
    same kind of bounded sample, all host threads for lookups."""
    if cfg.get("dna"):
        return None
    from oracle import oracle as orc

    threads = host_cores()
    f = orc.make_filter(cfg["kind"], k=cfg["k"], choices=cfg["c"], seed=1,
                        size_bits=cfg.get("size_bits", cfg.get("bpk", 0) * cfg["n"]))
    n_s = min(cfg["n"], 1 << 21)
    nq_s = int(round(n_s * cfg["nq"] / cfg["n"]))
    keys = orc.even_keys(n_s, 13)
    t0 = time.perf_counter()
    f.insert_many(keys)
    t1 = time.perf_counter()
    rng = np.random.default_rng(99)
    q = np.concatenate([keys[rng.integers(0, n_s, nq_s // 2)], orc.odd_keys(nq_s - nq_s // 2, 12)])
    t2 = time.perf_counter()
    f.contains_many(q, threads=threads)
    t3 = time.perf_counter()
    return dict(value=round((n_s + nq_s) / ((t1 - t0) + (t3 - t2)) / 1e6, 3), unit="Mkeys/s",
                cores=threads, kind="port",
                sample=f"oracle/ C port: {n_s} inserts (1 writer) + {nq_s} lookups "
                       f"({threads} threads) into an empty full-geometry filter")


def run_reference(args, cfg):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    t0 = time.perf_counter()
    try:
        r = reference_rate(args.config, cfg, args.steps, args.warmup)
    except ImportError as e:
        # baseline/_ref is missing (tools/install_reference.sh, or build()):
        # the oracle's C port stands in, and the line says so
        r = port_rate(cfg)
        if r is None:
            print(json.dumps({"impl": "reference",
                              "unavailable": f"reference not importable ({e}); no C port "
                                             f"for the DNA workload"}), flush=True)
            return
        r.update(ms_per_step=None, cpu=cpu_model(), insert_rate=None, lookup_rate=None,
                 setup_s=None, sample=r["sample"] + f" -- reference not importable ({e})")
    line = {
        "impl": "reference", "metric": METRIC, "value": r["value"], "unit": r["unit"],
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": r["ms_per_step"], "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u64",
        "data": "synthetic (reference key streams even_keys/odd_keys; seeded sample steps)",
        "config": {"workload": cfg["workload"], "sample_of_workload": args.config != 1},
        "cpu_baseline": {k: r[k] for k in ("value", "unit", "cores", "kind", "sample", "cpu",
                                           "insert_rate", "lookup_rate", "setup_s")},
        "e2e": {"value": r["value"], "unit": r["unit"], "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    try:
        line["port"] = port_rate(cfg)
    except Exception as e:  # the secondary row must not cost the primary one
        line["port"] = {"error": str(e)[:200]}
    line["wall_s"] = round(time.perf_counter() - t0, 1)
    print(json.dumps(line), flush=True)


# -- GPU arm -----------------------------------------------------------------------------

def timed_steps(step, nsteps, warmup, stream, world, dev):
    """W untimed steps, then K timed ones between barrier + synchronize; returns
    (max-over-ranks elapsed ms, per-step event lists, launches, clocks)."""
    import torch
    import torch.distributed as dist

    from paper_2501_18977_b200 import _native

    events = [[torch.cuda.Event(enable_timing=True) for _ in range(4)]
              for _ in range(warmup + nsteps)]
    sampler = ClockSampler(torch.cuda.current_device())
    for i in range(warmup):
        step(events[i])
    torch.cuda.synchronize()
    if DIST:
        dist.barrier()
    torch.cuda.synchronize()
    sampler.start()
    l0 = _native.launch_count()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for i in range(warmup, warmup + nsteps):
        step(events[i])
    t1.record(stream)
    torch.cuda.synchronize()
    launches = _native.launch_count() - l0
    if DIST:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = sampler.stop()
    elapsed = t0.elapsed_time(t1)
    if DIST:
        t = torch.tensor([elapsed], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed = float(t.item())
    return elapsed, events[warmup:], launches, clocks


def phase_ms(timed, a, b, dev):
    """Mean ms between events a and b over the timed steps, max over ranks."""
    import torch
    import torch.distributed as dist

    v = sum(e[a].elapsed_time(e[b]) for e in timed) / len(timed)
    if DIST:
        t = torch.tensor([v], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        v = float(t.item())
    return v


def run_ours(args, cfg):
    import torch
    import torch.distributed as dist

    import paper_2501_18977_b200 as bb
    from paper_2501_18977_b200 import _native
    from paper_2501_18977_b200 import distributed as D

    world, rank, local = dist_env()
    if DIST:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    mode = args.insert_mode or ("relaxed" if cfg["c"] >= 2 else "ordered")
    fkw = dict(kind=cfg["kind"], k=cfg["k"], choices=cfg["c"], seed=1)
    fkw["size_bits"] = cfg["size_bits"] if "size_bits" in cfg else cfg["bpk"] * cfg["n"]
    filt = bb.Filter.from_config(bb.FilterConfig(**fkw), insert_mode=mode)
    plan = lookup_plan(cfg, world)
    keys = make_keys(cfg, dev)
    queries, is_pos = make_queries(cfg, keys, plan, rank, dev)
    outs = [torch.empty(plan["slice"], dtype=torch.uint8, device=dev)
            for _ in range(plan["distinct"])]
    words = filt.storage.d_words
    stream = torch.cuda.current_stream()
    # N > 1: order-free kinds (c = 1, standard) build from per-rank key slices
    # and OR-all-reduce the replicas; relaxed c >= 2 builds are partitioned
    # over the ranks' replicas through peer memory (one kernel per rank,
    # distributed.build_partitioned) when the GPUs reach each other, else
    # rank 0 builds and broadcasts
    split = DIST and world > 1 and D.order_free(filt)
    reps = None
    if DIST and world > 1 and not split and mode == "relaxed" and D.partitionable(filt):
        reps = D.peer_map(filt)  # collective; None on every rank if any cannot map
    parted = reps is not None
    builder = split or parted or rank == 0
    lo, hi = D.slice_bounds(cfg["n"], world)[rank] if (split or parted) else (0, cfg["n"])
    my_keys = keys[lo:hi]

    def lookups():
        for j in range(plan["nslices"]):
            d = j % plan["distinct"]
            filt.contains_many(queries[d], out=outs[d])

    def step(ev):
        ev[0].record(stream)
        if parted:
            words.zero_()
            D.build_partitioned(filt, keys, reps=reps)  # inserts, then the owners' broadcasts
        elif builder:
            words.zero_()
            filt.insert_many(my_keys)
        ev[1].record(stream)
        if split:
            D.or_allreduce_(words.view(torch.int64))
        elif DIST and not parted:
            dist.broadcast(words.view(torch.int64), src=0)
        ev[2].record(stream)
        lookups()
        ev[3].record(stream)

    elapsed_ms, timed, launches, clocks = timed_steps(step, args.steps, args.warmup, stream,
                                                      world, dev)
    ins_ms = phase_ms(timed, 0, 1, dev)
    bc_ms = phase_ms(timed, 1, 2, dev)
    look_ms = phase_ms(timed, 2, 3, dev)
    ms_per_step = elapsed_ms / args.steps
    keys_per_step = cfg["n"] + world * plan["per_rank"]
    value = keys_per_step / (ms_per_step / 1e3) / 1e6

    # correctness of the measured run (outside the timed region)
    fn = fp = n_neg = 0
    span = 1 << 28  # bounded temporaries: a 2^32-key slice's int64 sums would be 32 GB
    for o, s in zip(outs, is_pos):
        for a in range(0, o.numel(), span):
            found, sp = o[a:a + span].bool(), s[a:a + span]
            fn += int(torch.count_nonzero(sp & ~found).item())
            n_neg += int(torch.count_nonzero(~sp).item())
            fp += int(torch.count_nonzero(~sp & found).item())
    if DIST:
        t = torch.tensor([fn, fp, n_neg], device=dev, dtype=torch.int64)
        dist.all_reduce(t)
        fn, fp, n_neg = (int(v) for v in t.tolist())

    # roofline of the dominant kernel
    peak, peak_src = measured_peak()
    l0 = _native.launch_count()
    if builder:
        words.zero_()
        filt.insert_many(my_keys)
    torch.cuda.synchronize()
    launches_ins = max(1, _native.launch_count() - l0)
    l0 = _native.launch_count()
    lookups()
    torch.cuda.synchronize()
    launches_look = max(1, _native.launch_count() - l0)
    ins_bytes = insert_bytes(cfg["c"]) * (hi - lo)
    look_bytes = cfg["lookup_bytes"] * plan["per_rank"]
    if look_ms >= ins_ms or not builder:
        kname, kms, kbytes, klaunch = "contains", look_ms, look_bytes, launches_look
    else:
        kname, kms, kbytes, klaunch = "insert", ins_ms, ins_bytes, launches_ins
    achieved = kbytes / (kms / 1e3) / 1e9
    fbytes = filt.storage.num_words * 8
    ceiling, ceiling_src = random_ceiling(fbytes)
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4),
                "traffic": profiled_traffic(args.config, kname),
                "kernel": f"{kname}: {klaunch} launch(es)/step, {kms / klaunch:.3f} ms/launch",
                "algorithmic_bytes_per_launch": kbytes / klaunch,
                "algorithmic_bytes_per_unit": (cfg["lookup_bytes"] if kname == "contains"
                                               else insert_bytes(cfg["c"])),
                "peak_source": peak_src,
                "random_sector_ceiling_gbs": ceiling,
                "frac_of_random_ceiling": round(achieved / ceiling, 4),
                "random_ceiling_source": ceiling_src}
    if fbytes <= 64 * 2**20:
        roofline["note"] = ("filter mostly L2-resident: block traffic is served by L2, so "
                            "algorithmic GB/s can exceed the HBM copy peak")
    elif fbytes <= torch.cuda.get_device_properties(dev).L2_cache_size:
        roofline["note"] = ("filter fits the L2 and its words are launched under a persisting "
                            "L2 access-policy window; block traffic is largely served by L2")

    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "Mkeys/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u64",
        "data": ("synthetic: reference key streams even_keys(n, 11) / odd_keys(., 12 + rank) "
                 "(numpy-identical, generated on the device for cfg3/5), seeded 50/50 mix"),
        "config": {"workload": cfg["workload"], "insert_mode": mode,
                   "lookups_per_rank": plan["per_rank"],
                   "lookup_launches_per_step": plan["nslices"],
                   "resident_query_slices": plan["distinct"],
                   "parallelism": ("single GPU" if world == 1 else
                                   f"build from per-rank key slices + OR all-reduce, "
                                   f"lookups split dp{world}" if split else
                                   f"relaxed build partitioned over the {world} replicas "
                                   f"through peer memory (one kernel per rank) + the owners' "
                                   f"range broadcasts, lookups split dp{world}" if parted else
                                   f"build on rank 0 + NCCL broadcast, lookups split dp{world}"),
                   "l2": "inputs larger than L2 (keys and queries re-read every step); filter "
                         "words L2-persisting only when the filter fits L2"},
        "insert_mkeys_s": round(cfg["n"] / ins_ms / 1e3, 2) if builder else None,
        "lookup_mkeys_s": round(world * plan["per_rank"] / look_ms / 1e3, 2),
        "lookup_ms": round(look_ms, 3), "insert_ms": round(ins_ms, 3) if builder else None,
        "broadcast_ms": round(bc_ms, 3) if DIST else None,
        "replication": ("or_allreduce" if split else "partitioned" if parted else "broadcast")
        if DIST else None,
        "false_negatives": fn, "fpr": fp / max(n_neg, 1), "negatives_checked": n_neg,
        "gpu_launches": int(launches),
        "clocks": clocks,
        "roofline": roofline,
    }

    if not args.no_extras and mode == "relaxed" and rank == 0:
        # the bit-exact alternative (stream-order claim rounds, the Filter
        # default), timed once outside the timed region
        exact = bb.Filter.from_config(bb.FilterConfig(**fkw), insert_mode="ordered")
        exact.insert_many(keys[: min(cfg["n"], 1 << 20)])  # scratch + warm-up
        exact.storage.d_words.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        exact.insert_many(keys)
        e1.record(stream)
        torch.cuda.synchronize()
        ord_ms = e0.elapsed_time(e1)
        line["ordered_insert_mkeys_s"] = round(cfg["n"] / ord_ms / 1e3, 2)
        if world == 1:
            # the whole step with the bit-exact insert in place of the relaxed
            # one: this run's measured lookups plus the exact insert above
            line["bit_exact_step"] = {
                "value": round(keys_per_step / ((ord_ms + look_ms) / 1e3) / 1e6, 2),
                "unit": "Mkeys/s", "insert_ms": round(ord_ms, 3),
                "note": "Filter default (stream order, bits identical to the reference); "
                        "one timed insert + the timed region's lookup phase"}
        del exact
        torch.cuda.empty_cache()
    if not args.no_extras and args.config == 5 and rank == 0:
        line["fpr_curve"] = fpr_curve(filt, keys, dev)
    # e2e through the public API from page-locked host buffers
    if not args.no_e2e:
        del outs, is_pos
        line["e2e"] = run_e2e(args, cfg, plan, filt, keys, queries, world, rank, dev)
    del queries
    torch.cuda.empty_cache()
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args.config, cfg)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if DIST:
        dist.barrier()
        dist.destroy_process_group()


def cpu_baseline(cfgno: int, cfg: dict) -> dict:
    """The reference itself (numba, baseline/_ref) on one bounded sample step,
    else the oracle C port."""
    try:
        r = reference_rate(cfgno, cfg, steps=1, warmup=0)
        return {k: r[k] for k in ("value", "unit", "cores", "kind", "sample", "cpu",
                                  "insert_rate", "lookup_rate", "ms_per_step")}
    except ImportError as e:
        r = port_rate(cfg) or {"value": None}
        r["note"] = f"reference not importable ({e}); oracle port timed instead"
        return r


class HostBuffers:
    """numpy arrays page-locked in place (cudaHostRegister): the copy engines
    read and write them directly, with no staging copy and no power-of-two
    rounding of the pinned allocator."""

    def __init__(self):
        self.arrays = []

    def alloc(self, n: int, dtype) -> np.ndarray:
        import torch

        a = np.empty(n, dtype=dtype)
        if a.nbytes:
            rc = torch.cuda.cudart().cudaHostRegister(a.ctypes.data, a.nbytes, 0)
            if int(rc) != 0:
                raise RuntimeError(f"cudaHostRegister failed ({rc})")
            self.arrays.append(a)
        return a

    def release(self):
        import torch

        for a in self.arrays:
            torch.cuda.cudart().cudaHostUnregister(a.ctypes.data)
        self.arrays = []


def run_e2e(args, cfg, plan, filt, keys, queries, world, rank, dev):
    """The step through Filter.insert_many / contains_many with host (numpy)
    keys and answers: every insert key and every lookup key crosses the host
    link inside the timed region (bc_insert_host / bc_contains_host stage
    them through the copy engines, overlapped with the kernels), and every
    answer comes back to host memory."""
    import torch
    import torch.distributed as dist

    from paper_2501_18977_b200 import distributed as D

    split = DIST and world > 1 and D.order_free(filt)
    builder = split or rank == 0
    lo, hi = D.slice_bounds(cfg["n"], world)[rank] if split else (0, cfg["n"])
    n_mine = hi - lo if builder else 0
    need = 8 * n_mine + 9 * plan["slice"]
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", "1"))
    avail = host_mem_available() // max(1, local_world)
    ok = need <= 0.8 * avail
    if DIST:
        t = torch.tensor([0 if ok else 1], device=dev)
        dist.all_reduce(t)
        ok = int(t.item()) == 0
    if not ok:
        return {"value": None, "unit": "Mkeys/s",
                "note": f"host RAM: {need / 1e9:.0f} GB of page-locked buffers per rank needed, "
                        f"{avail / 1e9:.0f} GB available"}
    hb = HostBuffers()
    t_setup = time.perf_counter()
    try:
        h_keys = hb.alloc(n_mine, np.uint64)
        h_q = hb.alloc(plan["slice"], np.uint64)
        h_out = hb.alloc(plan["slice"], np.uint8)
        if n_mine:
            torch.from_numpy(h_keys.view(np.int64)).copy_(keys[lo:hi].view(torch.int64))
        torch.from_numpy(h_q.view(np.int64)).copy_(queries[0].view(torch.int64))
        setup_s = time.perf_counter() - t_setup
        words = filt.storage.d_words
        nk = h_keys

        def step():
            if builder:
                words.zero_()
                filt.insert_many(nk)                 # H2D of the keys inside the call
            if split:
                D.or_allreduce_(words.view(torch.int64))
            elif DIST:
                dist.broadcast(words.view(torch.int64), src=0)
            for _ in range(plan["nslices"]):
                filt.contains_many(h_q, out=h_out)   # H2D queries, D2H answers

        steps = max(1, min(args.steps, 2 if plan["per_rank"] >= 2**30 else args.steps))
        step()
        torch.cuda.synchronize()
        if DIST:
            dist.barrier()
        stream = torch.cuda.current_stream()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        # CUDA events on the current stream; the host-buffer calls return only
        # after their answers are in host memory, so the bracket covers the copies
        t0.record(stream)
        for _ in range(steps):
            step()
        t1.record(stream)
        torch.cuda.synchronize()
        el = t0.elapsed_time(t1) / 1e3
        if DIST:
            t = torch.tensor([el], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el = float(t.item())
        # positives are even keys: none may be answered False (first 2^24)
        m = min(h_q.shape[0], 1 << 24)
        fn_e2e = int(np.count_nonzero(((h_q[:m] & np.uint64(1)) == 0) & (h_out[:m] == 0)))
    finally:
        hb.release()
    keys_per_step = cfg["n"] + world * plan["per_rank"]
    h2d = int(8 * (n_mine + plan["per_rank"]))
    d2h = int(plan["per_rank"])
    return {"value": round(keys_per_step * steps / el / 1e6, 2), "unit": "Mkeys/s",
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "ms_per_step": round(el / steps * 1e3, 3), "steps": steps, "warmup": 1,
            "link_gbs": round((h2d + d2h) * steps / el / 1e9, 1),
            "host_buffers": ("page-locked numpy (cudaHostRegister): all insert keys, one "
                             f"lookup slice of {plan['slice']} keys re-sent for each of the "
                             f"step's {plan['nslices']} lookup launches, its answers"),
            "setup_s": round(setup_s, 1), "false_negatives_last_slice": fn_e2e,
            "path": "Filter.insert_many/contains_many(numpy) -> bc_insert_host/bc_contains_host"}


def fpr_curve(filt, keys, device, gammas=(0.2, 0.4, 0.6, 0.8, 1.0, 1.2), n_neg=1 << 26):
    """FPR after inserting gamma x design capacity (cfg5: capacity 2^32 keys),
    from n_neg odd keys; keys holds 1.2 x capacity in stream order."""
    import torch

    from paper_2501_18977_b200 import odd_keys

    neg = odd_keys(n_neg, 77, device=device)
    filt.storage.d_words.zero_()
    cap = keys.numel() / 1.2
    done, curve = 0, []
    for gm in gammas:
        upto = min(keys.numel(), int(round(gm * cap)))
        if upto > done:
            filt.insert_many(keys[done:upto])
            done = upto
        curve.append({"gamma": gm, "fpr": filt.count_hits(neg) / n_neg})
    del neg
    torch.cuda.empty_cache()
    return curve


def make_dna(cfg, device, n_reads):
    """Genome (synthetic_genome: PCG64 words, the stream the full-size parity
    fixture was built from), true reads (1% substitutions) and random reads,
    ASCII on the device; reads are laid out 151 bytes apart (150 bases + '\\n')."""
    import torch

    from paper_2501_18977_b200 import synthetic_genome

    L, R, RL = cfg["genome"], n_reads, cfg["read_len"]
    genome = synthetic_genome(L, 4, device=device)
    g = torch.Generator(device=device).manual_seed(4)
    lut = torch.tensor(list(b"ACGT"), dtype=torch.uint8, device=device)
    true_reads = torch.empty((R, RL + 1), dtype=torch.uint8, device=device)
    rand_reads = torch.empty((R, RL + 1), dtype=torch.uint8, device=device)
    true_reads[:, RL] = ord("\n")
    rand_reads[:, RL] = ord("\n")
    off = torch.arange(RL, device=device, dtype=torch.int64)
    chunk = 1 << 20
    for a in range(0, R, chunk):
        b = min(R, a + chunk)
        start = torch.randint(0, L - RL, (b - a, 1), device=device, dtype=torch.int64,
                              generator=g)
        c = genome[start + off]
        sub = torch.rand((b - a, RL), device=device, generator=g) < cfg["sub"]
        shift = torch.randint(1, 4, (b - a, RL), device=device, dtype=torch.uint8, generator=g)
        # substitute to one of the other three bases
        code = ((c >> 1) ^ (c >> 2)) & 3
        true_reads[a:b, :RL] = torch.where(sub, lut[((code + shift) % 4).long()], c)
        rc = torch.randint(0, 4, (b - a, RL), device=device, dtype=torch.uint8, generator=g)
        rand_reads[a:b, :RL] = lut[rc.long()]
    return genome, true_reads.view(-1), rand_reads.view(-1)


def run_dna(args, cfg):
    """Config 4: fused q-gram insert of the genome, fused count-only lookups
    of both read sets; value = k-mers processed per second."""
    import torch
    import torch.distributed as dist

    import paper_2501_18977_b200 as bb

    world, rank, local = dist_env()
    if DIST:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    mode = args.insert_mode or "relaxed"
    q = cfg["q"]
    L = cfg["genome"]
    R = args.reads or cfg["reads"]
    RL = cfg["read_len"]
    filt = bb.Filter.from_config(bb.FilterConfig(kind="blowchoc", k=cfg["k"], choices=cfg["c"],
                                                 size_bits=cfg["k"] * (L - q + 1), seed=1),
                                 insert_mode=mode)
    enc = bb.QGramEncoder(q, True)
    genome, true_reads, rand_reads = make_dna(cfg, dev, R)
    # strong scaling: each rank looks up its share of the reads
    r_lo, r_hi = rank * R // world, (rank + 1) * R // world
    my_true = true_reads[r_lo * (RL + 1):r_hi * (RL + 1)]
    my_rand = rand_reads[r_lo * (RL + 1):r_hi * (RL + 1)]
    words = filt.storage.d_words
    stream = torch.cuda.current_stream()
    builder = rank == 0
    res = {}

    def step(ev):
        ev[0].record(stream)
        if builder:
            words.zero_()
            res["inserted"] = filt.insert_qgrams(enc, genome)
        ev[1].record(stream)
        if DIST:
            dist.broadcast(words.view(torch.int64), src=0)
        ev[2].record(stream)
        res["hits_true"] = filt.count_qgram_hits(enc, my_true)
        res["hits_rand"] = filt.count_qgram_hits(enc, my_rand)
        ev[3].record(stream)

    elapsed, timed, launches, clocks = timed_steps(step, args.steps, args.warmup, stream,
                                                   world, dev)
    ins_ms = phase_ms(timed, 0, 1, dev)
    look_ms = phase_ms(timed, 2, 3, dev)
    ms = elapsed / args.steps
    win_read = RL - q + 1
    kmers_ins = L - q + 1
    kmers_look = 2 * R * win_read
    value = (kmers_ins + kmers_look) / (ms / 1e3) / 1e6
    peak, peak_src = measured_peak()
    my_look = 2 * (r_hi - r_lo) * win_read
    look_bytes = cfg["lookup_bytes"] * my_look + 2 * (r_hi - r_lo) * (RL + 1)
    ins_bytes = insert_bytes(cfg["c"]) * kmers_ins + L
    if look_ms >= ins_ms or not builder:
        kname, kms, kbytes = "contains_qgrams", look_ms, look_bytes
    else:
        kname, kms, kbytes = "insert_qgrams", ins_ms, ins_bytes
    achieved = kbytes / (kms / 1e3) / 1e9
    ceiling, ceiling_src = random_ceiling(filt.storage.num_words * 8)
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "Mk-mers/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic: seeded i.i.d. ACGT genome (PCG64 words) and reads, on the device",
        "config": {"workload": cfg["workload"] + (f" [reads={R}]" if R != cfg["reads"] else ""),
                   "insert_mode": mode, "l2": "inputs larger than L2"},
        "insert_mkmers_s": round(kmers_ins / ins_ms / 1e3, 2) if builder else None,
        "lookup_mkmers_s": round(kmers_look / look_ms / 1e3, 2),
        "inserted_kmers": res.get("inserted"),
        "true_read_kmer_hit_rate": res["hits_true"] / ((r_hi - r_lo) * win_read),
        "expected_true_rate_approx": 0.99 ** q,
        "fpr": res["hits_rand"] / ((r_hi - r_lo) * win_read),
        "gpu_launches": int(launches), "clocks": clocks,
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                     "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": None,
                     "kernel": f"{kname} ({kms:.2f} ms/step)", "peak_source": peak_src,
                     "random_sector_ceiling_gbs": ceiling,
                     "frac_of_random_ceiling": round(achieved / ceiling, 4)},
    }
    if not args.no_e2e:
        line["e2e"] = run_dna_e2e(args, filt, enc, genome, my_true, my_rand, builder,
                                  kmers_ins + kmers_look, world, dev)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(4, cfg)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if DIST:
        dist.destroy_process_group()


def run_dna_e2e(args, filt, enc, genome, true_reads, rand_reads, builder, kmers, world, dev):
    """Config 4 through the public API from page-locked host buffers: the
    genome and both read sets cross the host link every step."""
    import torch
    import torch.distributed as dist

    hb = HostBuffers()
    try:
        h_g = hb.alloc(genome.numel() if builder else 0, np.uint8)
        h_t = hb.alloc(true_reads.numel(), np.uint8)
        h_r = hb.alloc(rand_reads.numel(), np.uint8)
        if builder:
            torch.from_numpy(h_g).copy_(genome)
        torch.from_numpy(h_t).copy_(true_reads)
        torch.from_numpy(h_r).copy_(rand_reads)
        words = filt.storage.d_words

        def step():
            if builder:
                words.zero_()
                filt.insert_qgrams(enc, h_g)
            if DIST:
                dist.broadcast(words.view(torch.int64), src=0)
            filt.count_qgram_hits(enc, h_t)
            filt.count_qgram_hits(enc, h_r)

        step()
        torch.cuda.synchronize()
        stream = torch.cuda.current_stream()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        steps = max(1, min(args.steps, 2))
        t0.record(stream)
        for _ in range(steps):
            step()
        t1.record(stream)
        torch.cuda.synchronize()
        el = t0.elapsed_time(t1) / 1e3
        if DIST:
            t = torch.tensor([el], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el = float(t.item())
    finally:
        hb.release()
    h2d = int(h_g.nbytes + h_t.nbytes + h_r.nbytes)
    return {"value": round(kmers * steps / el / 1e6, 2), "unit": "Mk-mers/s",
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 16,
            "ms_per_step": round(el / steps * 1e3, 3), "steps": steps,
            "path": "Filter.insert_qgrams/count_qgram_hits(numpy bytes)"}


def main():
    args = parse()
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
    elif cfg.get("dna"):
        run_dna(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
