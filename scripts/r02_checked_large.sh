#!/bin/bash
# the bounds-checked library (GM_LIB=checked: device bounds / layout checks, run-time
# compiled kernels checked too) over the full-size workloads, 1-2 steps each
for a in "C2b 2" "C5 2" "C1 2" "C4 1" "C4p 1" "C3b 2" "C2a 4" "C3n 4" "C3u 2"; do
  set -- $a
  s=$(date +%s)
  GM_LIB=checked timeout 900 python scripts/prof_run.py --workload $1 --horizon $2 > gpurun_out/chk_$1.log 2>&1
  echo "$1 T=$2 rc=$? $(( $(date +%s) - s )) s: $(tail -1 gpurun_out/chk_$1.log | cut -c1-120)"
done
