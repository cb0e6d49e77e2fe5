#!/bin/bash
# ticket dataflow vs one-array claim rounds by filter size (exact order, 16 bits/key)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
run() { c=$1; lab=$2; shift 2; env "$@" python tools/ordered_probe.py $c 2>&1 | grep -E "mkeys|rror" | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l); print('$c', '$lab', d['ms_median'], d['mkeys_s'], d['bits_equal_reference'])
    except Exception: print(l.strip())"; }
for lg in 15 16 17 18 19 20; do
  bits=$((512 << lg)); n=$((bits / 16))
  run $bits:$n:2:14 "ticket" A=1
  run $bits:$n:2:14 "claims" BC_ORDERED_TICKET=0
done
for lg in 15 17 18 19 20 21; do
  bits=$((512 << lg)); n=$((bits / 16))
  run $bits:$n:3:16 "ticket" A=1
  run $bits:$n:3:16 "claims" BC_ORDERED_TICKET=0
done
