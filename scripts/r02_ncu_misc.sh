#!/bin/bash
# ncu --set full: k_step_warp on C2a (one warp per state), k_build_ws on C1 (shape-specialised, pitch 172)
ncu --set full --clock-control none --import-source on -k regex:k_step_warp -s 4 -c 1 \
  -o gpurun_out/ncu_step_warp_C2a -f python scripts/prof_run.py --workload C2a --horizon 8 > gpurun_out/ncu_sw.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_build_ws -c 1 \
  -o gpurun_out/ncu_build_C1 -f python scripts/prof_run.py --workload C1 --horizon 1 > gpurun_out/ncu_c1.log 2>&1
