#!/bin/bash
# Full ncu captures of single launches of the hot kernels (one GPU, run under gpurun):
#   tools/ncu_capture.sh <tag> [workload]   (NCU_NAME/NCU_REGEX/NCU_SKIP or NCU_SPECS)
# Writes gpurun_out/<tag>_<kernel>.ncu-rep.  The compiled circuit is cached
# under /tmp for the duration of the call (PCB_CIRCUIT_CACHE).
set -u
tag=$1; wl=${2:-hclt256}
export PCB_CIRCUIT_CACHE=/tmp/pcbcache
python tools/ncu_step.py $wl 1 > /dev/null 2>&1   # warm the circuit cache
cap() {  # name regex skip
  timeout 600 ncu --set full --import-source on --clock-control none -k "regex:$2" --launch-skip $3 -c 1 \
    -o gpurun_out/${tag}_$1 -f python tools/ncu_step.py $wl 1 > gpurun_out/${tag}_$1.log 2>&1
  echo "$1 rc=$?"
}
# NCU_SPECS="name:regex:skip ..." captures several kernels in one call
if [ -n "${NCU_SPECS:-}" ]; then
  for spec in $NCU_SPECS; do
    IFS=: read -r n r k <<< "$spec"
    cap "$n" "$r" "$k"
  done
else
  cap ${NCU_NAME:-sum_fwd_leaf} "${NCU_REGEX:-k_sum_ws}" ${NCU_SKIP:-0}
fi
