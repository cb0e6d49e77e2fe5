#!/bin/bash
# ncu evidence for configs 4 and 5 (1 GPU): launch lists of the bench command
# and one --set full capture of each dominant kernel.  Output: gpurun_out/ncu45/
cd $GRAFT_REPO_ROOT; O=gpurun_out/ncu45; mkdir -p $O
for c in 5 4; do
  CMD="python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
  [ $c = 4 ] && CMD="$CMD --reads 4000000"
  $CMD > $O/plain$c.log 2>&1; echo "plain$c rc=$?"
  timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_cfg$c.csv $CMD > $O/launch$c.log 2>&1; echo "launch$c rc=$?"
done
C5="python bench.py --config 5 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
C4="python bench.py --config 4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --reads 4000000"
for k in relaxed512 lookup512; do
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o $O/prof_cfg5_$k $C5 > $O/full5_$k.log 2>&1; echo "full5 $k rc=$?"
done
for k in qgram_blocks qgram_lookup; do
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o $O/prof_cfg4_$k $C4 > $O/full4_$k.log 2>&1; echo "full4 $k rc=$?"
done
