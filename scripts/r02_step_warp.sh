#!/bin/bash
# one warp per state (k_step_warp) vs expect_matrix + maxmin on the small stored-matrix sweeps, then parity
for w in C2a C3n; do
  python scripts/c3b_repeat.py $w 4 | tail -1 | sed "s/^/k_step_warp /"
  GM_STEP_WARP=0 python scripts/c3b_repeat.py $w 3 | tail -1 | sed "s/^/expect_matrix+maxmin /"
done > gpurun_out/sw_t.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_variants.py tests/test_gpu_parity.py tests/test_gpu_fullhorizon.py tests/test_gpu_checked.py tests/test_gpu_multi.py -x -q 2>&1 | tail -3 >> gpurun_out/sw_t.log
