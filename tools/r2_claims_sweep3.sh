#!/bin/bash
# exact-order claim rounds: right-sized persisting set-aside vs none
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
run() { c=$1; lab=$2; shift 2; env "$@" python tools/ordered_probe.py $c 2>&1 | grep mkeys | python -c "
import json,sys
for l in sys.stdin: d=json.loads(l); print('cfg$c', '$lab', d['ms_median'], d['mkeys_s'], d['bits_equal_reference'])"; }
for sl in 1048576 2097152 4194304 8388608; do
  run 5 "fit slots=$sl" BC_ORDERED_PERSIST_FIT=1 BC_ORDERED_SLOTS=$sl
done
run 5 "nopersist slots=1048576" BC_L2_PERSIST=0 BC_ORDERED_SLOTS=1048576
for sl in 2097152 4194304 8388608; do
  run 3 "fit slots=$sl" BC_ORDERED_PERSIST_FIT=1 BC_ORDERED_SLOTS=$sl
done
run 3 "nopersist slots=2097152" BC_L2_PERSIST=0 BC_ORDERED_SLOTS=2097152
