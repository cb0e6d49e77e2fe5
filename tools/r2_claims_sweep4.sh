#!/bin/bash
# exact-order claim rounds: size of the persisting set-aside under the claims
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
run() { c=$1; lab=$2; shift 2; env "$@" python tools/ordered_probe.py $c 2>&1 | grep mkeys | python -c "
import json,sys
for l in sys.stdin: d=json.loads(l); print('$c', '$lab', d['ms_median'], d['mkeys_s'], d['bits_equal_reference'])"; }
for mb in 32 48 56; do run 3 "slots=2^23 set-aside=$mb" BC_ORDERED_PERSIST_FIT=1 BC_ORDERED_PERSIST_MB=$mb; done
for mb in 16 24; do run 5 "slots=2^22 set-aside=$mb" BC_ORDERED_PERSIST_FIT=1 BC_ORDERED_PERSIST_MB=$mb BC_ORDERED_SLOTS=4194304; done
for mb in 32 48; do run 5 "slots=2^23 set-aside=$mb" BC_ORDERED_PERSIST_FIT=1 BC_ORDERED_PERSIST_MB=$mb; done
for ch in 393216 786432; do run 5 "slots=2^22 fit chunk=$ch" BC_ORDERED_PERSIST_FIT=1 BC_ORDERED_SLOTS=4194304 BC_ORDERED_CHUNK=$ch; done
for ch in 393216 786432; do run 3 "fit chunk=$ch" BC_ORDERED_PERSIST_FIT=1 BC_ORDERED_CHUNK=$ch; done
# c = 3 above 2^23 blocks (2 GiB), c = 2 at cfg4's geometry
for sl in 4194304 8388608; do
  run 17179869184:536870912:3:16 "c3 2GiB fit slots=$sl" BC_ORDERED_PERSIST_FIT=1 BC_ORDERED_SLOTS=$sl
  run 16800000000:1200000000:2:14 "c2 cfg4-geometry fit slots=$sl" BC_ORDERED_PERSIST_FIT=1 BC_ORDERED_SLOTS=$sl
done
run 16800000000:1200000000:2:14 "c2 cfg4-geometry old default" A=1
