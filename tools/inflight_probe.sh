# relaxed multi-choice inserts: rate and parity statistics against the keys-in-flight cap
cd $GRAFT_REPO_ROOT
for pct in 25 50 100 200; do
  echo "== BC_RELAXED_INFLIGHT_PCT=$pct"
  BC_RELAXED_INFLIGHT_PCT=$pct timeout 300 python bench.py --config 1 --no-e2e --no-cpu-baseline --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg1 insert', d['insert_mkeys_s'], 'fpr', d['fpr'])"
  BC_RELAXED_INFLIGHT_PCT=$pct timeout 300 python tools/relaxed_spread_probe.py 2>&1 | grep -E "^cfg1|cfg5_small|cfg3_small"
done
