#!/bin/bash
# ordered1_kernel: split phase B (checks, then full-tile commits; variant since removed, see
# profiles/r2/ordered_l2_sweeps.txt) vs fused; set-aside above the claims' size
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
run() { c=$1; lab=$2; shift 2; env "$@" python tools/ordered_probe.py $c 2>&1 | grep -E "mkeys|rror" | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l); print('$c', '$lab', d['ms_median'], d['mkeys_s'], d['bits_equal_reference'])
    except Exception: print(l.strip())"; }
python - <<'PY'
import torch
p = torch.cuda.get_device_properties(0)
print("L2", p.L2_cache_size, "persisting max", getattr(p, "persisting_l2_cache_max_size", None), "window max", getattr(p, "access_policy_max_window_size", None))
PY
for c in 3 5 16800000000:1200000000:2:14 17179869184:536870912:3:16; do
  run $c "split" A=1
  run $c "fused" BC_LIBRARY=$PWD/paper_2501_18977_b200/libbbchoc_nosplit.so
done
for mb in 36 40 48 64; do
  run 3 "split set-aside=$mb" BC_ORDERED_PERSIST_MB=$mb
  run 5 "split set-aside=$mb" BC_ORDERED_PERSIST_MB=$mb
done
