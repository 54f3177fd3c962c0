#!/bin/bash
# row-shape specialised fill for pitches that are not a multiple of 32 / long cell periods
# (C1: R = 169, pitch 172, period 13 in 6 chunks; C3u / C3e: R = 243): on vs off
for w in C1 C3u C3e C2b; do
  GM_JIT=1 python scripts/c3b_repeat.py $w 4 1 | tail -1 | sed "s/^/shape /"
  GM_JIT=1 GM_JIT_SHAPE=0 python scripts/c3b_repeat.py $w 4 1 | tail -1 | sed "s/^/noshape /"
done > gpurun_out/fs.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_jit.py tests/test_gpu_variants.py tests/test_gpu_fullhorizon.py -x -q 2>&1 | tail -3 >> gpurun_out/fs.log
