#!/bin/bash
# SASS evidence of the hot kernels in libbbchoc.so (no GPU needed): per kernel,
# the instruction count and the memory-instruction mix (LDG/LDGSTS/STG/RED/
# ATOM/UTMALDG/...), plus the full listing.  Output: profiles/<tag>/sass/
cd "$(dirname "$0")/.."
TAG=${1:-r2}; O=profiles/$TAG/sass; mkdir -p $O
LIB=paper_2501_18977_b200/libbbchoc.so
KERNELS="_ZN2bc27lookup512_pipe_multi_kernelILi2ELi11EEEvNS_7KParamsEPKmS3_mPhPy
_ZN2bc27lookup512_pipe_multi_kernelILi3ELi16EEEvNS_7KParamsEPKmS3_mPhPy
_ZN2bc17relaxed512_kernelILi2EEEvNS_7KParamsEPmPKmm
_ZN2bc15ordered1_kernelILi3ENS_9ArrayKeysEEEvNS_7KParamsEPmT0_mjPjmjS5_Pyj
_ZN2bc15ordered1_kernelILi2ENS_9ArrayKeysEEEvNS_7KParamsEPmT0_mjPjmjS5_Pyj
_ZN2bc17ordered512_kernelILi3ENS_9ArrayKeysEEEvNS_7KParamsEPmT0_mjPjmjS5_Py
_ZN2bc18ticket_exec_kernelILi2ENS_9ArrayKeysEEEvNS_7KParamsEPmT0_mPKjPjS7_Py
_ZN2bc16blocks512_kernelILi1ELi1EEEvNS_7KParamsEPmPKmmPhPy"
: > $O/summary.txt
for k in $KERNELS; do
  short=$(echo $k | sed -E 's/_ZN2bc[0-9]+//; s/EEEv.*//; s/ILi/_/g; s/ENS_9ArrayKeys/_keys/; s/Li//g; s/E/_/g')
  cuobjdump -sass -fun "$k" $LIB > $O/$short.sass 2>/dev/null
  n=$(grep -cE "^\s+/\*[0-9a-f]{4}\*/" $O/$short.sass)
  { echo "== $k ($n instructions)";
    grep -oE "^\s+/\*[0-9a-f]{4}\*/\s+(@!?U?P[0-9T] )?[A-Z0-9_.]+" $O/$short.sass | awk '{print $NF}' |
      grep -E "^(LDG|LDGSTS|STG|RED|ATOM|UTMA|UBLK|LDS|STS|ATOMS|SHFL|MEMBAR|BAR|SYNCS|POPC|IMAD|LOP3)" |
      sed -E 's/\..*//' | sort | uniq -c | sort -rn | tr '\n' ' '; echo; } >> $O/summary.txt
done
cat $O/summary.txt
