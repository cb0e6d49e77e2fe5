"""Throughput of the insert / lookup hot path on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

A step is one pass of the hot path over one batch of synthetic input:
build the filter from zero (insert the config's n keys) and answer the
config's lookup batch.  The default workload is BASELINE.json configs[1]
(config 2: single-choice blocked filter, 2^26 keys, k=12, 12 bits/key,
2^27 lookups, half inserted / half fresh).  Keys are the reference's own
streams (even_keys(n, 11), odd_keys(., 12), seeded shuffle) for configs 1-2
and seeded device-generated uint64 for the larger configs.

``value``: keys (inserted + looked up) per second over the timed steps,
inputs resident in HBM.  ``e2e``: the same metric through the public API
(Filter.insert_many / contains_many) from pinned host buffers, copies
included.  ``--impl reference`` times the CPU oracle (a C restatement of the
reference's numba kernels, oracle/) on all host cores instead.

Multi-GPU (torchrun, one rank per GPU, NCCL): every rank answers its own
lookup batch (weak scaling); the build is shared for order-free kinds (c = 1,
standard: each rank ORs a slice of the keys into its replica, then the
replicas are OR-all-reduced) and done on rank 0 + NCCL-broadcast for c >= 2
(T = 1, so the reference layout has no subfilters).  value = all keys / max
rank time.
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

METRIC = "insert & lookup Mkeys/s (1/2/4/8 B200); FPR; % of random-sector HBM roofline"

# BASELINE.json configs; bytes/unit from SURVEY §8(d)
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
    5: dict(workload="cfg5: blowchoc c=2 k=11 8 GiB, 1.2*2^32 keys, 2^32 lookups per step "
                     "(50% pos)",
            kind="blowchoc", c=2, k=11, n=int(1.2 * 2**32), size_bits=2**36, nq=2**32,
            ref_keys=False, lookup_bytes=119.6),
}


def insert_bytes(c: int) -> float:
    return 8 + 64 * c + 64  # key + c candidate reads + one block write-back


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=2, choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--insert-mode", default=None, choices=["ordered", "relaxed"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
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


# -- synthetic inputs ---------------------------------------------------------------------

def make_inputs(cfg: dict, rank: int, device):
    """(insert keys, query keys, positive mask) on the device."""
    import torch

    n, nq = cfg["n"], cfg["nq"]
    if cfg["ref_keys"]:
        from paper_2501_18977_b200 import even_keys, odd_keys

        keys = even_keys(n, 11)
        npos = nq // 2
        rng = np.random.default_rng(5 + rank)
        pos = keys[rng.integers(0, n, npos)]
        neg = odd_keys(nq - npos, 12 + rank)
        q = np.concatenate([pos, neg])
        perm = rng.permutation(nq)
        q = q[perm]
        is_pos = perm < npos
        return (torch.from_numpy(keys).to(device), torch.from_numpy(q).to(device),
                torch.from_numpy(is_pos).to(device))
    from paper_2501_18977_b200 import even_keys, odd_keys

    # the reference's own streams (even_keys(n, 11) / odd_keys(., 12)),
    # generated on the device bit-identically to numpy (bc_pcg64_fill)
    g = torch.Generator(device=device).manual_seed(1234 + rank)
    span = 1 << 28  # slices: cfg5 holds 5e9 keys + 4e9 queries (~80 GB)
    keys = even_keys(n, 11, device=device).view(torch.int64)
    # queries: a seeded coin picks a uniform sample of the inserted keys
    # (positive) or the next key of the odd stream (negative)
    q = torch.empty(nq, dtype=torch.int64, device=device)
    sel = torch.empty(nq, dtype=torch.bool, device=device)
    for a in range(0, nq, span):
        b = min(nq, a + span)
        s = torch.randint(0, 2, (b - a,), device=device, dtype=torch.int64, generator=g).bool()
        idx = torch.randint(0, n, (b - a,), device=device, dtype=torch.int64, generator=g)
        neg = odd_keys(b - a, 12 + rank, device=device, offset=a).view(torch.int64)
        q[a:b] = torch.where(s, keys[idx], neg)
        sel[a:b] = s
        del s, idx, neg
    return keys.view(torch.uint64), q.view(torch.uint64), sel


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
        return float(d["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured copy)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


def random_ceiling(filter_bytes: int):
    """Measured random 64-byte-gather ceiling (tools/gather_probe.cu, ld.global.cg,
    profiles/r1/gather_probe_*.txt) for the nearest filter size, in algorithmic
    GB/s of the lookup pattern (64 B block + 8 B key + 1 B answer)."""
    table = [(96 << 20, 7011.0), (512 << 20, 3145.0), (2 << 30, 2551.0), (8 << 30, 2415.0)]
    best = min(table, key=lambda t: abs(np.log2(t[0]) - np.log2(max(filter_bytes, 1))))
    return best[1]


def profiled_traffic(config: int, kernel: str):
    """dram bytes per launch of ``kernel`` from the committed ncu summary."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return d.get(f"cfg{config}", {}).get(kernel)
    except (OSError, ValueError):
        return None


# -- CPU side (oracle: test infrastructure, used only as baseline / reference arm) ------

def oracle_filter(cfg: dict, words_host: np.ndarray | None):
    """A full-size oracle filter holding the workload's bit array: the
    GPU-built words when given, else built on the host (all keys for
    single-choice filters up to 2^26, a 2^22-key prefix otherwise)."""
    from oracle import oracle as orc

    kw = dict(k=cfg["k"], choices=cfg["c"], seed=1,
              size_bits=cfg.get("size_bits", cfg.get("bpk", 0) * cfg["n"]))
    f = orc.make_filter(cfg["kind"], **kw)
    if words_host is not None:
        f.words[:] = words_host
        return f, "GPU-built bit array"
    nb = cfg["n"] if (cfg["c"] == 1 and cfg["n"] <= 2**26) or cfg["n"] <= 2**22 else 2**22
    keys = orc.even_keys(nb, 11)
    if cfg["c"] == 1:
        f.insert_many_mt(keys, host_cores())
    else:
        f.insert_many(keys)
    return f, f"host-built from {nb} keys"


def cpu_sample(cfg: dict, f) -> dict:
    """Oracle rates on a bounded sample: 2^22 fresh inserts (threaded OR for
    c = 1 -- bit-identical to stream order; one writer in stream order for
    c >= 2, as the reference's single-writer rule requires) and 2^23 lookups,
    half positive, split over all host cores (the reference's query
    parallelism, analysis.py:96-107)."""
    from oracle import oracle as orc

    threads = host_cores()
    n_ins = min(cfg["n"], 1 << 22)
    ins = orc.even_keys(n_ins, 13)
    t0 = time.perf_counter()
    if cfg["c"] == 1:
        f.insert_many_mt(ins, threads)
    else:
        f.insert_many(ins)
    t_ins = time.perf_counter() - t0
    n_look = min(cfg["nq"], 1 << 23)
    rng = np.random.default_rng(99)
    q = np.concatenate([ins[rng.integers(0, n_ins, n_look // 2)],
                        orc.odd_keys(n_look - n_look // 2, 12)])
    rng.shuffle(q)
    t0 = time.perf_counter()
    f.contains_many(q, threads=threads)
    t_look = time.perf_counter() - t0
    ins_rate, look_rate = n_ins / t_ins, n_look / t_look
    step_s = cfg["n"] / ins_rate + cfg["nq"] / look_rate
    return dict(value=round((cfg["n"] + cfg["nq"]) / step_s / 1e6, 3), unit="Mkeys/s",
                cores=threads, kind="port",
                sample=(f"{n_ins} inserts ({'threaded OR' if cfg['c'] == 1 else '1 writer, stream order'})"
                        f" + {n_look} lookups ({threads} threads) into the full-size filter; rate "
                        f"weighted to the step's {cfg['n']} inserts + {cfg['nq']} lookups"),
                insert_mkeys_s=round(ins_rate / 1e6, 3), lookup_mkeys_s=round(look_rate / 1e6, 3),
                cpu=cpu_model())


def cpu_rate(cfg: dict, words_host: np.ndarray | None) -> dict:
    f, built = oracle_filter(cfg, words_host)
    r = cpu_sample(cfg, f)
    r["sample"] += f" ({built})"
    return r


def cpu_dna_rate(cfg: dict) -> dict:
    """Oracle k-mers/s for config 4 on a bounded sample: encode + insert a
    4 Mbp genome prefix (one writer, stream order), then encode + look up
    2 x 40 000 reads (joined with separators, all host threads); the rate is
    weighted to the step's mix of inserted and looked-up k-mers."""
    from oracle import oracle as orc

    threads = host_cores()
    q, RL = cfg["q"], cfg["read_len"]
    rng = np.random.default_rng(4)
    Lp, R = 4_000_000, 40_000
    alphabet = np.frombuffer(b"ACGT", dtype=np.uint8)
    codes = rng.integers(0, 4, Lp)
    genome = alphabet[codes].tobytes()
    t0 = time.perf_counter()
    keys = orc.encode_qgrams(genome, q, True)
    f = orc.make_filter("blowchoc", k=cfg["k"], choices=cfg["c"], seed=1,
                        size_bits=cfg["k"] * (Lp - q + 1))
    f.insert_many(keys)
    t_ins = time.perf_counter() - t0
    starts = rng.integers(0, Lp - RL, R)
    reads = codes[starts[:, None] + np.arange(RL)]
    sub = rng.random(reads.shape) < cfg["sub"]
    reads = np.where(sub, (reads + rng.integers(1, 4, reads.shape)) % 4, reads)
    rand = rng.integers(0, 4, (R, RL))
    sep = np.full((R, 1), ord("\n"), dtype=np.uint8)
    blob = np.concatenate([np.concatenate([alphabet[reads], sep], 1).ravel(),
                           np.concatenate([alphabet[rand], sep], 1).ravel()]).tobytes()
    t0 = time.perf_counter()
    qk = orc.encode_qgrams(blob, q, True)
    f.contains_many(qk, threads=threads)
    t_look = time.perf_counter() - t0
    ins_rate, look_rate = keys.shape[0] / t_ins, qk.shape[0] / t_look
    n_ins = cfg["genome"] - q + 1
    n_look = 2 * cfg["reads"] * (RL - q + 1)
    value = (n_ins + n_look) / (n_ins / ins_rate + n_look / look_rate) / 1e6
    return dict(value=round(value, 3), unit="Mk-mers/s", cores=threads, kind="port",
                sample=(f"encode+insert of a {Lp}-bp genome prefix (1 writer) + encode+lookup "
                        f"of 2x{R} reads ({threads} threads); rate weighted to the step's "
                        f"{n_ins} inserted + {n_look} looked-up k-mers"),
                insert_mkmers_s=round(ins_rate / 1e6, 3),
                lookup_mkmers_s=round(look_rate / 1e6, 3), cpu=cpu_model())


def run_reference(args, cfg):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    if cfg.get("dna"):
        vals = [cpu_dna_rate(cfg) for _ in range(args.warmup + args.steps)][args.warmup:]
        r = vals[-1]
        value = statistics.median(v["value"] for v in vals)
        print(json.dumps({
            "impl": "reference", "metric": METRIC, "value": value, "unit": "Mk-mers/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic i.i.d. genome and reads", "config": {"workload": cfg["workload"]},
            "cpu_baseline": dict(r, value=value),
            "e2e": {"value": value, "unit": "Mk-mers/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}), flush=True)
        return
    f, built = oracle_filter(cfg, None)
    vals = []
    r = None
    for i in range(args.warmup + args.steps):
        r = cpu_sample(cfg, f)
        if i >= args.warmup:
            vals.append(r["value"])
    value = statistics.median(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "Mkeys/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round((cfg["n"] + cfg["nq"]) / value / 1e3, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic (reference key streams: even_keys/odd_keys)",
        "config": {"workload": cfg["workload"], "l2": "inputs larger than L2"},
        "cpu_baseline": {"value": value, "unit": "Mkeys/s", "cores": r["cores"],
                         "kind": "port", "sample": r["sample"] + f" ({built})", "cpu": r["cpu"],
                         "insert_mkeys_s": r["insert_mkeys_s"],
                         "lookup_mkeys_s": r["lookup_mkeys_s"]},
        "e2e": {"value": value, "unit": "Mkeys/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# -- GPU arm -----------------------------------------------------------------------------

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
    keys, queries, is_pos = make_inputs(cfg, rank, dev)
    out = torch.empty(queries.numel(), dtype=torch.uint8, device=dev)
    words = filt.storage.d_words
    stream = torch.cuda.current_stream()
    # N > 1: order-free kinds (c = 1, standard) build from per-rank key slices
    # and OR-all-reduce the replicas; c >= 2 builds on rank 0 and broadcasts
    split = DIST and world > 1 and D.order_free(filt)
    builder = split or rank == 0
    lo, hi = D.slice_bounds(cfg["n"], world)[rank] if split else (0, cfg["n"])
    my_keys = keys[lo:hi]

    def step(ev):
        ev[0].record(stream)
        if builder:
            words.zero_()
            filt.insert_many(my_keys)
        ev[1].record(stream)
        if split:
            D.or_allreduce_(words.view(torch.int64))
        elif DIST:
            dist.broadcast(words.view(torch.int64), src=0)
        ev[2].record(stream)
        filt.contains_many(queries, out=out)
        ev[3].record(stream)

    events = [[torch.cuda.Event(enable_timing=True) for _ in range(4)]
              for _ in range(args.warmup + args.steps)]
    sampler = ClockSampler(torch.cuda.current_device())
    sampler.start()
    for i in range(args.warmup):
        step(events[i])
    torch.cuda.synchronize()
    if DIST:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = _native.launch_count()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for i in range(args.warmup, args.warmup + args.steps):
        step(events[i])
    t1.record(stream)
    torch.cuda.synchronize()
    launches = _native.launch_count() - l0
    if DIST:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = sampler.stop()
    elapsed_ms = t0.elapsed_time(t1)
    timed = events[args.warmup:]
    ins_ms = sum(e[0].elapsed_time(e[1]) for e in timed) / args.steps
    bc_ms = sum(e[1].elapsed_time(e[2]) for e in timed) / args.steps
    look_ms = sum(e[2].elapsed_time(e[3]) for e in timed) / args.steps
    if DIST:
        t = torch.tensor([elapsed_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms = float(t.item())
    ms_per_step = elapsed_ms / args.steps
    keys_per_step = cfg["n"] + world * cfg["nq"]
    value = keys_per_step / (ms_per_step / 1e3) / 1e6

    # correctness of the measured run (outside the timed region)
    found = out.bool()
    fn = int((is_pos & ~found).sum().item())
    n_neg = int((~is_pos).sum().item())
    fp = int((~is_pos & found).sum().item())
    if DIST:
        t = torch.tensor([fn, fp, n_neg], device=dev, dtype=torch.int64)
        dist.all_reduce(t)
        fn, fp, n_neg = (int(v) for v in t.tolist())

    # roofline of the dominant kernel
    peak, peak_src = measured_peak()
    # kernel launches of one insert call (outside the timed region)
    l0 = _native.launch_count()
    if builder:
        words.zero_()
        filt.insert_many(my_keys)
    torch.cuda.synchronize()
    launches_ins = max(1, _native.launch_count() - l0)
    ins_bytes = insert_bytes(cfg["c"]) * (hi - lo)
    look_bytes = cfg["lookup_bytes"] * cfg["nq"]
    if look_ms >= ins_ms:
        kname, kms, kbytes, klaunch = "contains", look_ms, look_bytes, 1
    else:
        kname, kms, kbytes, klaunch = "insert", ins_ms, ins_bytes, launches_ins
    achieved = kbytes / (kms / 1e3) / 1e9
    traffic = profiled_traffic(args.config, kname)
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic,
                "kernel": f"{kname} ({klaunch} launch(es)/step, {kms:.3f} ms/step)",
                "algorithmic_bytes_per_launch": kbytes / klaunch, "peak_source": peak_src}
    if filt.storage.num_words * 8 <= 64 * 2**20:
        roofline["note"] = ("filter mostly L2-resident: block traffic is served by L2, so "
                            "algorithmic GB/s can exceed the HBM copy peak")
    elif filt.storage.num_words * 8 <= torch.cuda.get_device_properties(dev).L2_cache_size:
        roofline["note"] = ("filter fits the L2 and its words are launched under a persisting "
                            "L2 access-policy window (keys stream past it); block traffic is "
                            "largely served by L2 (profiles/r1)")
    roofline["random_sector_ceiling_gbs"] = random_ceiling(filt.storage.num_words * 8)

    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "Mkeys/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
        "data": ("synthetic: reference key streams even_keys/odd_keys, seeded shuffle"
                 if cfg["ref_keys"] else
                 "synthetic: reference key streams even_keys(n, 11) / odd_keys(., 12) "
                 "generated on the device (bit-identical to numpy), seeded 50/50 mix"),
        "config": {"workload": cfg["workload"], "insert_mode": mode,
                   "parallelism": ("single GPU" if world == 1 else
                                   f"build from per-rank key slices + OR all-reduce "
                                   f"(all-to-all, OR fold, all-gather), lookups dp{world}"
                                   if split else
                                   f"build on rank 0 + NCCL broadcast, lookups dp{world}"),
                   "l2": "inputs larger than L2 (keys re-read every step); filter words "
                         "L2-persisting when the filter fits L2 (BC_L2_PERSIST)"},
        "insert_mkeys_s": round(cfg["n"] / ins_ms / 1e3, 2) if builder else None,
        "lookup_mkeys_s": round(cfg["nq"] / look_ms / 1e3, 2),
        "broadcast_ms": round(bc_ms, 3) if DIST else None,
        "replication": ("or_allreduce" if split else "broadcast") if DIST else None,
        "false_negatives": fn, "fpr": fp / max(n_neg, 1),
        "gpu_launches": int(launches),
        "clocks": clocks,
        "roofline": roofline,
    }

    if mode == "relaxed" and rank == 0:
        # the bit-exact alternative (stream-order claim rounds), timed once
        # outside the timed region, for reference next to the relaxed rate
        exact = bb.Filter.from_config(bb.FilterConfig(**fkw), insert_mode="ordered")
        exact.insert_many(keys[: min(cfg["n"], 1 << 20)])  # scratch + warm-up
        exact.storage.d_words.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        exact.insert_many(keys)
        e1.record(stream)
        torch.cuda.synchronize()
        line["ordered_insert_mkeys_s"] = round(cfg["n"] / e0.elapsed_time(e1) / 1e3, 2)
        del exact
        torch.cuda.empty_cache()
    if args.config == 5 and builder:
        line["fpr_curve"] = fpr_curve(filt, keys, dev)
    # e2e through the public API from pinned host buffers
    if not args.no_e2e:
        line["e2e"] = run_e2e(args, cfg, filt, keys, queries, world, rank, dev)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_rate(cfg, filt.storage.words)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if DIST:
        dist.barrier()
        dist.destroy_process_group()


def run_e2e(args, cfg, filt, keys, queries, world, rank, dev):
    import torch
    import torch.distributed as dist

    if cfg["nq"] > 2**28:
        return {"value": None, "unit": "Mkeys/s", "note": "e2e skipped above 2^28 lookups"}
    h_keys = torch.empty(keys.numel(), dtype=torch.uint64, pin_memory=True)
    h_keys.copy_(keys.cpu())
    h_q = torch.empty(queries.numel(), dtype=torch.uint64, pin_memory=True)
    h_q.copy_(queries.cpu())
    h_out = torch.empty(queries.numel(), dtype=torch.uint8, pin_memory=True)
    nk, nq, no = h_keys.numpy(), h_q.numpy(), h_out.numpy()
    from paper_2501_18977_b200 import distributed as D

    split = DIST and world > 1 and D.order_free(filt)
    builder = split or rank == 0
    lo, hi = D.slice_bounds(cfg["n"], world)[rank] if split else (0, cfg["n"])
    nk_mine = nk[lo:hi]
    words = filt.storage.d_words

    def step():
        if builder:
            words.zero_()
            filt.insert_many(nk_mine)            # H2D of the keys inside the call
        if split:
            D.or_allreduce_(words.view(torch.int64))
        elif DIST:
            dist.broadcast(words.view(torch.int64), src=0)
        filt.contains_many(nq, out=no)           # H2D queries, D2H answers

    # large batches: 5 steps are seconds of PCIe traffic; small ones use all steps
    steps = max(1, min(args.steps, 5) if cfg["nq"] >= 2**26 else args.steps)
    for _ in range(max(1, min(args.warmup, 3))):
        step()
    torch.cuda.synchronize()
    if DIST:
        dist.barrier()
    # CUDA events on the current stream; the host-buffer calls return only
    # after their answers are in host memory, so the bracket covers the copies
    stream = torch.cuda.current_stream()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
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
    keys_per_step = cfg["n"] + world * cfg["nq"]
    h2d = int(8 * ((hi - lo if builder else 0) + cfg["nq"]))
    d2h = int(cfg["nq"])
    return {"value": round(keys_per_step * steps / el / 1e6, 2), "unit": "Mkeys/s",
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "ms_per_step": round(el / steps * 1e3, 3), "steps": steps,
            "link_gbs": round((h2d + d2h) * steps / el / 1e9, 1),
            "note": "bound by the host link: keys and queries cross PCIe every step",
            "path": "Filter.insert_many/contains_many(pinned numpy) -> bc_*_host"}


def fpr_curve(filt, keys, device, gammas=(0.2, 0.4, 0.6, 0.8, 1.0, 1.2), n_neg=1 << 26):
    """FPR after inserting gamma x design capacity (cfg5: capacity 2^32 keys),
    from n_neg odd keys; keys holds 1.2 x capacity in stream order."""
    import torch

    g = torch.Generator(device=device).manual_seed(77)
    neg = (torch.randint(-2**63, 2**63 - 1, (n_neg,), device=device, dtype=torch.int64,
                         generator=g) | 1).view(torch.uint64)
    filt.storage.d_words.zero_()
    cap = keys.numel() / 1.2
    done, curve = 0, []
    for gm in gammas:
        upto = min(keys.numel(), int(round(gm * cap)))
        if upto > done:
            filt.insert_many(keys[done:upto])
            done = upto
        curve.append({"gamma": gm, "fpr": filt.count_hits(neg) / n_neg})
    return curve


def make_dna(cfg, device, n_reads):
    """Genome, true reads (1% substitutions) and random reads, ASCII on the
    device; reads are laid out 151 bytes apart (150 bases + '\\n')."""
    import torch

    L, R, RL = cfg["genome"], n_reads, cfg["read_len"]
    g = torch.Generator(device=device).manual_seed(4)
    lut = torch.tensor(list(b"ACGT"), dtype=torch.uint8, device=device)
    codes = torch.empty(L, dtype=torch.uint8, device=device)
    span = 1 << 27
    for a in range(0, L, span):
        b = min(L, a + span)
        codes[a:b] = torch.randint(0, 4, (b - a,), device=device, dtype=torch.uint8, generator=g)
    genome = torch.empty(L, dtype=torch.uint8, device=device)
    for a in range(0, L, span):
        b = min(L, a + span)
        genome[a:b] = lut[codes[a:b].long()]
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
        c = codes[start + off]
        sub = torch.rand((b - a, RL), device=device, generator=g) < cfg["sub"]
        shift = torch.randint(1, 4, (b - a, RL), device=device, dtype=torch.uint8, generator=g)
        c = torch.where(sub, (c + shift) % 4, c)
        true_reads[a:b, :RL] = lut[c.long()]
        rc = torch.randint(0, 4, (b - a, RL), device=device, dtype=torch.uint8, generator=g)
        rand_reads[a:b, :RL] = lut[rc.long()]
    del codes
    return genome, true_reads.view(-1), rand_reads.view(-1)


def run_dna(args, cfg):
    """Config 4: fused q-gram insert of the genome, fused count-only lookups
    of both read sets; value = k-mers processed per second."""
    import torch
    import torch.distributed as dist

    import paper_2501_18977_b200 as bb
    from paper_2501_18977_b200 import _native

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
        res["hits_true"] = filt.count_qgram_hits(enc, true_reads)
        res["hits_rand"] = filt.count_qgram_hits(enc, rand_reads)
        ev[3].record(stream)

    events = [[torch.cuda.Event(enable_timing=True) for _ in range(4)]
              for _ in range(args.warmup + args.steps)]
    sampler = ClockSampler(torch.cuda.current_device())
    sampler.start()
    for i in range(args.warmup):
        step(events[i])
    torch.cuda.synchronize()
    if DIST:
        dist.barrier()
    l0 = _native.launch_count()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for i in range(args.warmup, args.warmup + args.steps):
        step(events[i])
    t1.record(stream)
    torch.cuda.synchronize()
    launches = _native.launch_count() - l0
    clocks = sampler.stop()
    elapsed = t0.elapsed_time(t1)
    if DIST:
        t = torch.tensor([elapsed], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed = float(t.item())
    timed = events[args.warmup:]
    ins_ms = sum(e[0].elapsed_time(e[1]) for e in timed) / args.steps
    look_ms = sum(e[2].elapsed_time(e[3]) for e in timed) / args.steps
    ms = elapsed / args.steps
    win_read = RL - q + 1
    kmers_ins = L - q + 1
    kmers_look = 2 * R * win_read
    value = (kmers_ins + world * kmers_look) / (ms / 1e3) / 1e6
    peak, peak_src = measured_peak()
    look_bytes = cfg["lookup_bytes"] * kmers_look + 2 * R * (RL + 1)
    ins_bytes = insert_bytes(cfg["c"]) * kmers_ins + L
    if look_ms >= ins_ms:
        kname, kms, kbytes = "contains_qgrams", look_ms, look_bytes
    else:
        kname, kms, kbytes = "insert_qgrams", ins_ms, ins_bytes
    achieved = kbytes / (kms / 1e3) / 1e9
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "Mk-mers/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic: seeded i.i.d. ACGT genome and reads generated on the device",
        "config": {"workload": cfg["workload"] + (f" [reads={R}]" if R != cfg["reads"] else ""),
                   "insert_mode": mode, "l2": "inputs larger than L2"},
        "insert_mkmers_s": round(kmers_ins / ins_ms / 1e3, 2),
        "lookup_mkmers_s": round(kmers_look / look_ms / 1e3, 2),
        "inserted_kmers": res["inserted"],
        "true_read_kmer_hit_rate": res["hits_true"] / (R * win_read),
        "expected_true_rate_approx": 0.99 ** q,
        "fpr": res["hits_rand"] / (R * win_read),
        "gpu_launches": int(launches), "clocks": clocks,
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                     "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": None,
                     "kernel": f"{kname} ({kms:.2f} ms/step)", "peak_source": peak_src},
        "e2e": {"value": None, "unit": "Mk-mers/s",
                "note": "DNA inputs are generated on the device; see configs 1-2 for e2e"},
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_dna_rate(cfg)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if DIST:
        dist.destroy_process_group()


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
