#!/bin/bash
# ncu with APPLICATION replay (the whole probe re-run per pass), so the
# ordered launch's persisting L2 window on the claim arrays is intact in every
# pass -- kernel replay loses it and inflates the DRAM traffic.
#   tools/r2_ncu_app.sh KERNEL_REGEX OUTNAME -- command...
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
K=$1; OUT=$2; shift 3
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_requests_srcunit_tex_op_atom.sum,lts__t_requests_srcunit_tex_op_red.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_write.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,smsp__inst_executed.sum,breakdown:lts__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active
mkdir -p gpurun_out
timeout 1500 ncu --replay-mode application --cache-control none --clock-control none -k "regex:$K" -c 1 \
  --metrics $M --csv --log-file gpurun_out/$OUT.csv "$@" > gpurun_out/$OUT.log 2>&1
echo "ncu rc=$?"
python - gpurun_out/$OUT.csv <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
for r in rows[1:]:
    print(f"{r[h.index('Metric Name')]:75s} {r[h.index('Metric Value')]:>20} {r[h.index('Metric Unit')]}")
PY
