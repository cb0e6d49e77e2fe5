cd $GRAFT_REPO_ROOT
run() { c=$1; lab=$2; shift 2; env "$@" python tools/ordered_probe.py $c 2>&1 | grep -E "mkeys|rror" | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l); print('$c', '$lab', d['ms_median'], d['mkeys_s'])
    except Exception: print(l.strip())"; }
for ch in 786432 917504 1048576 1212416; do
  run 5 "chunk=$ch" BC_ORDERED_CHUNK=$ch
  run 16800000000:1200000000:2:14 "cfg4-geometry chunk=$ch" BC_ORDERED_CHUNK=$ch
done
