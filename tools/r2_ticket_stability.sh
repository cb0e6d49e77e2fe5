#!/bin/bash
# run-to-run spread of the ticket dataflow near its upper size limit (c = 3, 16 bits/key)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
for M in 262144 393216 458752 524287; do
  bits=$((M * 512)); nk=$((bits / 16))
  for rep in 1 2 3 4; do
    python tools/ordered_probe.py $bits:$nk:3:16 2>&1 | grep mkeys | python -c "
import json,sys
for l in sys.stdin: d=json.loads(l); print('M=$M c=3 run $rep', d['ms_median'], d['mkeys_s'])"
  done
done
