#!/bin/bash
# A/B of exact-order kernel variants (paper_2501_18977_b200/libbbchoc_<v>.so,
# tools/build_variant.sh), interleaved, with the bits checked each time.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
for rep in 1 2; do for lib in ${LIBS:-cur}; do
  L=paper_2501_18977_b200/libbbchoc.so; [ "$lib" != cur ] && L=paper_2501_18977_b200/libbbchoc_$lib.so
  BC_LIBRARY=$PWD/$L python tools/ordered_probe.py ${CFGS:-3 5} 2>&1 | grep mkeys | python -c "
import json,sys
for l in sys.stdin: d=json.loads(l); print('$lib', d['config'], d['ms_median'], d['mkeys_s'], d['bits_equal_reference'])"
done; done
