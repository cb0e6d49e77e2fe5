#!/bin/bash
# ordered1_kernel: per-round profile, persisting window, CTAs per SM
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
run() { c=$1; lab=$2; shift 2; env "$@" python tools/ordered_probe.py $c 2>&1 | grep -E "mkeys|rror" | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l); print('$c', '$lab', d['ms_median'], d['mkeys_s'], d['bits_equal_reference'])
    except Exception: print(l.strip())"; }
for c in 3 5; do
  BC_LIBRARY=$PWD/paper_2501_18977_b200/libbbchoc_prof.so python tools/ordered_probe.py $c 2>&1 | grep "ord1 prof" | awk 'NR%7==1' | head -4
  run $c "nopersist" BC_L2_PERSIST=0
  run $c "set-aside=16" BC_ORDERED_PERSIST_MB=16
  run $c "set-aside=24" BC_ORDERED_PERSIST_MB=24
  run $c "2 CTAs/SM (122 regs)" BC_LIBRARY=$PWD/paper_2501_18977_b200/libbbchoc_minb2.so
  run $c "4 CTAs/SM (64 regs)" BC_LIBRARY=$PWD/paper_2501_18977_b200/libbbchoc_minb4.so
  run $c "default" A=1
done
