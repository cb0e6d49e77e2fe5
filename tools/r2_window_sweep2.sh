#!/bin/bash
# one-array claim rounds: the window rule's constant for c = 3 and c = 4 (default M / (2 c^2))
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
run() { c=$1; lab=$2; shift 2; env "$@" python tools/ordered_probe.py $c 2>&1 | grep -E "mkeys|rror" | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l); print('$c', '$lab', d['ms_median'], d['mkeys_s'])
    except Exception: print(l.strip())"; }
for lg in 20 22; do
  M=$((1 << lg)); bits=$((512 << lg)); nk=$((bits / 16))
  run $bits:$nk:3:16 "M=2^$lg c=3 default (M/18)" BC_ORDERED_TICKET=0
  for div in 12 24 32; do run $bits:$nk:3:16 "M=2^$lg c=3 window=M/$div" BC_ORDERED_TICKET=0 BC_ORDERED_CHUNK=$((M / div)); done
  run $bits:$nk:4:16 "M=2^$lg c=4 default (M/32)" BC_ORDERED_TICKET=0
  for div in 16 24 48; do run $bits:$nk:4:16 "M=2^$lg c=4 window=M/$div" BC_ORDERED_TICKET=0 BC_ORDERED_CHUNK=$((M / div)); done
done
