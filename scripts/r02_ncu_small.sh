#!/bin/bash
# ncu --set full of the small-row stored-matrix sweep kernels (C2a, R = 27; C3n, R = 32)
mkdir -p gpurun_out
python scripts/c3b_repeat.py C2a 2 > gpurun_out/c2a_plain.log 2>&1 || exit 1
for w in C2a C3n; do
ncu --set full --clock-control none --import-source on -k regex:"k_expect_matrix_small|k_maxmin" -s 6 -c 4 \
  -o gpurun_out/ncu_small_$w -f python scripts/c3b_repeat.py $w 1 > gpurun_out/ncu_small_$w.log 2>&1
done
