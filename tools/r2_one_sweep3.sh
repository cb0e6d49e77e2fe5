#!/bin/bash
# ordered1_kernel: load steps per commit tile x CTAs per SM
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
run() { c=$1; lab=$2; shift 2; env "$@" python tools/ordered_probe.py $c 2>&1 | grep -E "mkeys|rror" | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l); print('$c', '$lab', d['ms_median'], d['mkeys_s'], d['bits_equal_reference'])
    except Exception: print(l.strip())"; }
for c in 3 5 16800000000:1200000000:2:14 17179869184:536870912:3:16; do
  run $c "default (3 CTAs/SM)" A=1
  run $c "2 CTAs/SM" BC_LIBRARY=$PWD/paper_2501_18977_b200/libbbchoc_minb2.so
  run $c "2 CTAs/SM, one load step" BC_LIBRARY=$PWD/paper_2501_18977_b200/libbbchoc_minb2unr4.so
  run $c "3 CTAs/SM, one key per load step" BC_LIBRARY=$PWD/paper_2501_18977_b200/libbbchoc_unr1.so
done
