#!/bin/bash
# exact-order claim rounds: claim slots x window x L2 persistence (env knobs only)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
run() { c=$1; lab=$2; shift 2; env "$@" python tools/ordered_probe.py $c 2>&1 | grep mkeys | python -c "
import json,sys
for l in sys.stdin: d=json.loads(l); print('cfg$c', '$lab', d['ms_median'], d['mkeys_s'], d['bits_equal_reference'])"; }
for sl in 2097152 4194304 8388608; do for ch in 262144 524288 786432 1048576; do
  run 5 "nopersist slots=$sl chunk=$ch" BC_L2_PERSIST=0 BC_ORDERED_SLOTS=$sl BC_ORDERED_CHUNK=$ch
done; done
for pe in 0 -1; do for ch in 262144 393216 524288 786432; do
  run 3 "persist=$pe chunk=$ch" BC_L2_PERSIST=$pe BC_ORDERED_CHUNK=$ch
done; done
