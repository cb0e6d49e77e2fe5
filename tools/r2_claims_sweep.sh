#!/bin/bash
# exact-order claim rounds vs claim-array footprint and L2 persistence (env knobs only)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
run() { lab=$1; shift; env "$@" python tools/ordered_probe.py ${CFGS:-3 5} 2>&1 | grep mkeys | python -c "
import json,sys
for l in sys.stdin: d=json.loads(l); print('$lab', d['config'], d['ms_median'], d['mkeys_s'], d['bits_equal_reference'])"; }
run default A=1
run nopersist BC_L2_PERSIST=0
run slots22 BC_ORDERED_SLOTS=4194304
run slots21 BC_ORDERED_SLOTS=2097152
run slots20 BC_ORDERED_SLOTS=1048576
run slots22_nopersist BC_ORDERED_SLOTS=4194304 BC_L2_PERSIST=0
