#!/bin/bash
# C4 OFA (k_expect_ofa_pk, TAB_P): shared-memory carveout (more L1 for the V gathers)
for c in default 25 50 75; do
  if [ $c = default ]; then python scripts/c3b_repeat.py C4 2 1 | tail -1 | sed "s/^/$c /";
  else GM_OFA_CARVEOUT=$c python scripts/c3b_repeat.py C4 2 1 | tail -1 | sed "s/^/$c /"; fi
done > gpurun_out/c4co.log 2>&1
