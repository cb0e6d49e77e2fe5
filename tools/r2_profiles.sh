#!/bin/bash
# Round-2 ncu evidence (1 GPU): launch list of the default bench command
# (config 5) and --set full captures of its two kernels, of the exact-order
# config-3 claim-round kernel, and of the config-1 ticket dataflow.
# Output: gpurun_out/$1/
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/${1:-prof}; mkdir -p $O
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-extras"
$CMD > $O/plain.json 2> $O/plain.err; echo "plain rc=$?"
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $O/launches_cfg5.csv $CMD > $O/launch.log 2>&1; echo "launch list rc=$?"
for k in relaxed512 lookup512; do
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o $O/prof_cfg5_$k $CMD > $O/full5_$k.log 2>&1; echo "full5 $k rc=$?"
done
python tools/ordered_probe.py 3 > $O/ordered3.json 2>&1; echo "ordered3 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ordered1_kernel -c 1 -o $O/prof_cfg3_ordered python tools/ordered_probe.py 3 > $O/full3_ord.log 2>&1; echo "full3 ordered rc=$?"
python tools/ordered_probe.py 1 > $O/ordered1.json 2>&1; echo "ordered1 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg1_ordered.csv python tools/ordered_probe.py 1 > /dev/null 2>&1; echo "launch1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ticket_exec -c 1 -o $O/prof_cfg1_ticket python tools/ordered_probe.py 1 > $O/full1_ticket.log 2>&1; echo "full1 ticket rc=$?"
