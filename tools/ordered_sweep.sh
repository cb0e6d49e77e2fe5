# exact-order insert rate by claim slots / window (bench.py --insert-mode ordered)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
run() {  # config, label, env...
  c=$1; lab=$2; shift 2
  env "$@" timeout 600 python bench.py --config $c --insert-mode ordered --no-e2e --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/sw.json 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/sw.json').read().strip().splitlines()[-1]);print('cfg$c $lab', d['insert_mkeys_s'])" || tail -3 gpurun_out/sw.json
}
for c in 3 5; do
  run $c default
  run $c slots22 BC_ORDERED_SLOTS=4194304
  run $c win18 BC_ORDERED_CHUNK=262144
  run $c win20 BC_ORDERED_CHUNK=1048576
done
run 1 default
run 1 win14 BC_ORDERED_CHUNK=16384
run 1 win13 BC_ORDERED_CHUNK=8192
