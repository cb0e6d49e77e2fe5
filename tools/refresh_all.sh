#!/bin/bash
# Round-end evidence on one GPU: every bench line, the reference arm, a
# torchrun (1 rank) sanity run, the ncu launch list of the default command and
# a --set full capture of its two kernels.  Output: gpurun_out/final/
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/final; mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
for c in 2 1 3 4 5; do
  timeout 1200 python bench.py --config $c > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err; echo "cfg$c rc=$?"
done
for c in 1 3 5; do
  timeout 1200 python bench.py --config $c --insert-mode ordered > $O/bench_cfg${c}_ordered.json 2> $O/bo$c.err; echo "cfg$c ordered rc=$?"
done
timeout 900 python bench.py --impl reference > $O/bench_reference_cfg2.json 2> $O/ref.err; echo "ref rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu-baseline > $O/torchrun1.json 2> $O/torchrun1.err; echo "torchrun rc=$?"
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > $O/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file $O/launches_cfg2.csv $CMD > $O/ncu_launch.log 2>&1; echo "launch list rc=$?"
$CMD > $O/plain2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"blocks512|lookup512" -s 6 -c 2 \
      -o $O/prof_cfg2 $CMD > $O/ncu_full.log 2>&1; echo "full rc=$?"
