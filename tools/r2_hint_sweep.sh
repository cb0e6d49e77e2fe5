#!/bin/bash
# L2 eviction-priority hints (createpolicy + .L2::cache_hint) on the exact-order
# rounds: claims evict_last (hc), + candidate block loads evict_first (hcb), + the
# commits' REDs evict_first (hcbr), blocks only (hb); with and without the persisting window
# (the BC_HINT_* code paths were removed after the measurement: profiles/r2/ordered_l2_sweeps.txt)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
run() { c=$1; lab=$2; shift 2; env "$@" python tools/ordered_probe.py $c 2>&1 | grep -E "mkeys|rror" | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l); print('$c', '$lab', d['ms_median'], d['mkeys_s'], d['bits_equal_reference'])
    except Exception: print(l.strip())"; }
for c in 3 5; do
  run $c "default" A=1
  for v in hc hcb hcbr hb; do
    run $c "$v + window" BC_LIBRARY=$PWD/paper_2501_18977_b200/libbbchoc_$v.so
    run $c "$v, no window" BC_LIBRARY=$PWD/paper_2501_18977_b200/libbbchoc_$v.so BC_L2_PERSIST=0
  done
done
LIBS="cur hb" CONFIGS="3" STEPS=5 bash tools/ab_libs.sh
