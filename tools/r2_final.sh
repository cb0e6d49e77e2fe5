#!/bin/bash
# Round-2 final evidence on one GPU: the whole -m gpu suite, every bench line
# (tools/r2_refresh.sh), the exact-order kernel's DRAM traffic under
# application replay and its --set full capture.  Output: gpurun_out/$1/
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=${1:-final4}; mkdir -p gpurun_out/$O
timeout 3000 python -m pytest tests -m gpu -x -q -rs --durations=10 > gpurun_out/$O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/$O/pytest_gpu.log
bash tools/r2_refresh.sh $O
for c in 3 5; do
  bash tools/r2_ncu_app.sh ordered1_kernel $O/ord1_cfg${c}_app -- python tools/ordered_probe.py $c > gpurun_out/$O/ord1_cfg${c}_app.txt 2>&1; echo "app replay cfg$c rc=$?"
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ordered1_kernel -c 1 -o gpurun_out/$O/prof_cfg3_ordered1 python tools/ordered_probe.py 3 > gpurun_out/$O/full3_ord1.log 2>&1; echo "full3 ordered1 rc=$?"
