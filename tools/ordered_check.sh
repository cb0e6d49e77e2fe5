set -o pipefail
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "ordered or hashed or several" 2>&1 | tail -3
for c in 1 3 5; do
  timeout 600 python bench.py --config $c --insert-mode ordered --no-e2e --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/ord_cfg$c.json 2>gpurun_out/ord_cfg$c.err
  python -c "import json;d=json.loads(open('gpurun_out/ord_cfg$c.json').read().strip().splitlines()[-1]);print('cfg$c', d['insert_mkeys_s'], d['lookup_mkeys_s'], d['fpr'])" || tail -5 gpurun_out/ord_cfg$c.err
done
for sl in 8388608 16777216; do
  BC_ORDERED_SLOTS=$sl timeout 600 python bench.py --config 5 --insert-mode ordered --no-e2e --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/ord5_$sl.json 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/ord5_$sl.json').read().strip().splitlines()[-1]);print('cfg5 slots $sl', d['insert_mkeys_s'])"
done
