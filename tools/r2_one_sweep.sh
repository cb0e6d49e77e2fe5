#!/bin/bash
# one-array same-round claim rounds (ordered1_kernel) vs the two-array rounds; claim slots
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
run() { c=$1; lab=$2; shift 2; env "$@" python tools/ordered_probe.py $c 2>&1 | grep -E "mkeys|rror" | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l); print('$c', '$lab', d['ms_median'], d['mkeys_s'], d['bits_equal_reference'])
    except Exception: print(l.strip())"; }
run 3 "two-array" BC_ORDERED_ONE=0
run 3 "one-array" BC_ORDERED_ONE=1
run 5 "two-array" BC_ORDERED_ONE=0
for sl in 4194304 8388608 16777216; do run 5 "one-array slots=$sl" BC_ORDERED_SLOTS=$sl; done
for ch in 393216 786432 1048576; do run 3 "one-array chunk=$ch" BC_ORDERED_CHUNK=$ch; done
run 16800000000:1200000000:2:14 "c2 cfg4-geometry two-array" BC_ORDERED_ONE=0
for sl in 4194304 8388608 16777216; do run 16800000000:1200000000:2:14 "c2 cfg4-geometry one-array slots=$sl" BC_ORDERED_SLOTS=$sl; done
run 17179869184:536870912:3:16 "c3 2GiB two-array" BC_ORDERED_ONE=0
for sl in 8388608 16777216; do run 17179869184:536870912:3:16 "c3 2GiB one-array slots=$sl" BC_ORDERED_SLOTS=$sl; done
