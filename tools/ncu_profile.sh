#!/bin/bash
# ncu captures of the bench command (1 GPU): launch list + full set of the
# blocks512 kernels.  Usage: tools/ncu_profile.sh <config> <tag> [extra ncu args]
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
C=${1:-2}; TAG=${2:-r1}; shift 2
mkdir -p gpurun_out
CMD="python bench.py --config $C --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none --csv \
    --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1
echo "launch list rc=$?"
$CMD > gpurun_out/plain2_$TAG.log 2>&1 && \
ncu --set full --clock-control none --cache-control none --import-source on -k regex:${KREGEX:-blocks512} -s ${SKIP:-2} -c ${COUNT:-2} "$@" \
    -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo "full rc=$?"; tail -2 gpurun_out/ncu_full_$TAG.log
