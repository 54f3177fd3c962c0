#!/bin/bash
# k_expect_matrix_small: gathers in flight (GM_SMALL_U) x shared-memory budget per CTA
# (GM_SMALL_SMEM_KB; a smaller budget leaves more L1 for the V gathers)
for w in C2a C3n; do
  for u in 8 16 32; do for kb in 56 112 28; do
    echo "== $w U=$u KB=$kb"
    GM_MATRIX_SMALL=1 GM_SMALL_U=$u GM_SMALL_SMEM_KB=$kb python scripts/c3b_repeat.py $w 3 | tail -2
  done; done
  echo "== $w default"; python scripts/c3b_repeat.py $w 3 | tail -2
done
