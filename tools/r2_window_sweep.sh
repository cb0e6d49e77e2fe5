#!/bin/bash
# one-array claim rounds on mid-size filters (2^20 .. 2^22 blocks, 16 bits/key): window as a fraction of M
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
run() { c=$1; lab=$2; shift 2; env "$@" python tools/ordered_probe.py $c 2>&1 | grep -E "mkeys|rror" | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l); print('$c', '$lab', d['ms_median'], d['mkeys_s'])
    except Exception: print(l.strip())"; }
for ck in 2:14 3:16; do
for lg in 20 21 22; do
  M=$((1 << lg)); bits=$((512 << lg)); nk=$((bits / 16))
  for div in 2 4 8 16; do
    ch=$((M / div)); [ $ch -gt 786432 ] && continue
    run $bits:$nk:$ck "M=2^$lg c:k=$ck window=M/$div" BC_ORDERED_TICKET=0 BC_ORDERED_CHUNK=$ch
  done
done; done
