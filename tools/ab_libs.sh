#!/bin/bash
# A/B of library builds on the GPU box: bench each config with each variant
# (LIBS="rmw ''" -> paper_2501_18977_b200/libbbchoc_rmw.so and libbbchoc.so),
# interleaved so box drift hits both.  Variants come from tools/build_variant.sh.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
[ "${TESTS:-0}" = "1" ] && timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -2
for c in ${CFGS:-2}; do for rep in $(seq ${REPS:-1}); do for lib in ${LIBS:-""}; do
  [ "$lib" = "cur" ] && lib=""
  L=paper_2501_18977_b200/libbbchoc${lib:+_$lib}.so
  BC_LIBRARY=$PWD/$L timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline --steps ${STEPS:-20} ${EXTRA:-} 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print($c, '${lib:-cur}', d['value'], d['insert_mkeys_s'], d['lookup_mkeys_s'], d['fpr'], d['false_negatives'])"
done; done; done
