#!/bin/bash
# A/B probes: TMA gather4 vs LDGSTS block staging (tools/tma_gather_probe.cu),
# and the two-phase exact-order kernel (libbbchoc_tp.so) vs the default.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/${1:-probe}; mkdir -p $O
nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -o /tmp/tma_gather_probe tools/tma_gather_probe.cu
for mib in 96 512 8192; do
  /tmp/tma_gather_probe $mib 27 2>&1 | tee -a $O/tma_probe.txt
  PROBE_PERSIST=1 /tmp/tma_gather_probe $mib 27 2>&1 | sed 's/^/persist /' | tee -a $O/tma_probe.txt
done
cuobjdump -sass /tmp/tma_gather_probe | grep -E "UTMALDG|LDGSTS" | sort | uniq -c > $O/tma_probe_sass.txt
for lib in "" _tp; do
  echo "== lib$lib"; BC_LIBRARY=$PWD/paper_2501_18977_b200/libbbchoc$lib.so python tools/ordered_probe.py 3 5 2>&1 | tail -2
done
