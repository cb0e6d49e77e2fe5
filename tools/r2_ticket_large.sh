#!/bin/bash
# Ticket dataflow forced onto large filters: total rate, bits, and the
# per-kernel split (sort vs execution) from an ncu launch list.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
python tools/ordered_probe.py 3 2>&1 | grep mkeys
BC_TICKET_MAX_BLOCKS=1073741824 python tools/ordered_probe.py 3 5 2>&1 | grep mkeys
BC_TICKET_MAX_BLOCKS=1073741824 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none \
  --csv --log-file gpurun_out/ticket_cfg3_launches.csv python tools/ordered_probe.py 3 > gpurun_out/ticket_ncu.log 2>&1
python - <<'PY'
import csv, collections
rows = [r for r in csv.reader(open("gpurun_out/ticket_cfg3_launches.csv")) if len(r) > 10]
h = rows[0]; ki = h.index("Kernel Name"); vi = h.index("Metric Value")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    try: v = float(r[vi].replace(",", ""))
    except ValueError: continue
    k = r[ki][:60]; agg[k][0] += 1; agg[k][1] += v
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{n:6d} {t/1e6:10.3f} ms  {k}")
PY
