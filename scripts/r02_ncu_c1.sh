#!/bin/bash
# ncu --set full of the C1 (robot reach-avoid, R = 169) stored-matrix build
GM_JIT_CACHE=0 GM_JIT_VERBOSE=1 ncu --set full --clock-control none --import-source on -k regex:k_build_ws -c 1 \
  -o gpurun_out/ncu_build_c1 -f python scripts/prof_run.py --workload C1 --horizon 1 > gpurun_out/ncu_build_c1.log 2>&1
cp /tmp/gm_jit_kind*.cubin gpurun_out/ 2>/dev/null
