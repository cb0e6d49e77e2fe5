#!/bin/bash
# one gpurun call: GPU tests (quick subset unless FULL=1), then the default bench
set -o pipefail
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
if [ "${FULL:-0}" = "1" ]; then
  timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -15
else
  timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "ordered_build or device_tensor or qgram or dna or empty or relaxed" 2>&1 | tail -8
fi
for c in ${CONFIGS:-2}; do
  timeout 600 python bench.py --config $c ${BENCH_ARGS:-} > gpurun_out/bench_cfg$c.json 2> gpurun_out/bench_cfg$c.err
  echo "cfg$c rc=$?"; python - "$c" <<'PY'
import json, sys
c = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/bench_cfg{c}.json").read().strip().splitlines()[-1])
except Exception as e:
    print("no bench line:", e); print(open(f"gpurun_out/bench_cfg{c}.err").read()[-2000:]); sys.exit()
keys = ["value", "insert_mkeys_s", "lookup_mkeys_s", "false_negatives", "fpr", "gpu_launches"]
print({k: d.get(k) for k in keys})
print("roofline", d.get("roofline"))
print("e2e", d.get("e2e"), "clocks", d.get("clocks"))
print("cpu", (d.get("cpu_baseline") or {}).get("value"))
PY
done
