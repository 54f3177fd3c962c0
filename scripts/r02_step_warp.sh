#!/bin/bash
# one warp per state (k_step_warp) vs expect_matrix + maxmin on the small stored-matrix sweeps, then the GPU suite
for w in C2a C3n; do
  python scripts/c3b_repeat.py $w 4 | tail -1 | sed "s/^/k_step_warp /"
  GM_STEP_WARP=0 python scripts/c3b_repeat.py $w 3 | tail -1 | sed "s/^/expect_matrix+maxmin /"
done > gpurun_out/sw_t.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 >> gpurun_out/sw_t.log
python scripts/configs_table.py --only C2a,C3n --cpu-from profiles/r02/configs.md > gpurun_out/cfg_small.log 2>&1
