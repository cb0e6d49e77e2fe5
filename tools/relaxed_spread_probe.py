import os, sys
sys.path.insert(0, os.getcwd())
import json, numpy as np
import paper_2501_18977_b200 as bb
meta = json.load(open("tests/golden/golden.json"))
for name in ["cfg1", "bc3_k12_20k", "bc2_k6_t4", "bc3_dist_k10", "bc8_k5", "bc2_b1024", "cfg3_small", "cfg5_small_k11"]:
    case = meta[name]
    cfg = bb.FilterConfig(**case["config"])
    keys = bb.even_keys(case["n_insert"], case["insert_seed"])
    neg = bb.odd_keys(case["n_neg"], case["neg_seed"])
    exact = bb.Filter.from_config(cfg); exact.insert_many(keys)
    he = bb.block_load_histogram(exact).counts
    tvs, hs, vs = [], [], []
    for r in range(10):
        f = bb.Filter.from_config(cfg, insert_mode="relaxed"); f.insert_many(keys)
        h = bb.block_load_histogram(f)
        tvs.append(bb.histogram_distance(h.counts, he)); hs.append(f.count_hits(neg)); vs.append(h.variance / case["variance"] - 1)
    print(name, f.num_blocks, "TV max %.4f" % max(tvs), "hits", min(hs), max(hs), "ref", case["hits_neg"], "var dev max %.3f" % max(abs(v) for v in vs))
