#!/bin/bash
# Exact-order window sweep (BC_ORDERED_CHUNK keys per round) on configs 3 and 5.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
for ch in ${CHUNKS:-393216 524288 786432 1048576}; do
  BC_ORDERED_CHUNK=$ch python tools/ordered_probe.py ${CFGS:-3 5} 2>&1 | grep mkeys | python -c "
import json,sys
for l in sys.stdin: d=json.loads(l); print($ch, d['config'], d['ms_median'], d['mkeys_s'], d['bits_equal_reference'])"
done
