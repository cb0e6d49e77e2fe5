#!/bin/bash
# Round-2 bench evidence on one GPU: every config's bench line (default
# relaxed mode for c >= 2, then the bit-exact mode), the reference arm, a
# one-rank torchrun launch of the default command, and the §8(f) rows.
# Output: gpurun_out/$1/
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/${1:-refresh}; mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
for c in 5 1 2 3 4; do
  timeout 1500 python bench.py --config $c > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err; echo "cfg$c rc=$?"
done
for c in 1 3 4 5; do
  timeout 1500 python bench.py --config $c --insert-mode ordered --no-cpu-baseline > $O/bench_cfg${c}_ordered.json 2> $O/bo$c.err; echo "cfg$c ordered rc=$?"
done
timeout 900 python bench.py --impl reference > $O/bench_reference_cfg5.json 2> $O/ref.err; echo "ref rc=$?"
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/torchrun1.json 2> $O/torchrun1.err; echo "torchrun rc=$?"
timeout 1500 python tools/bench_next.py > $O/bench_next.jsonl 2> $O/bench_next.err; echo "bench_next rc=$?"
