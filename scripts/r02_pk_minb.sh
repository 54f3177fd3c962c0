#!/bin/bash
# k_expect_ofa_pk register cap experiment: the hoisted-cell OFA kernel under a
# 3-CTA (80 registers), 2-CTA (128) cap; rebuilds the kernel object on the box.
mkdir -p gpurun_out
run() {
  python scripts/c3b_repeat.py C4 3 1
  GM_JIT=0 python scripts/c3b_repeat.py C5 3 4
  python scripts/c3b_repeat.py tests/golden/large/bmw7_mid.cfg 3 8
  GM_JIT=0 python scripts/c3b_repeat.py C4p 2 1
}
for b in 3 2; do
  rm -f paper_2005_06191_b200/_build/gm_kernels.o
  make -s -C paper_2005_06191_b200/csrc NVEXTRA=-DGM_OFA_PK_MINB=$b ../libgridmdp_b200.so > /dev/null 2>&1
  run 2>&1 | sed "s/^/minb$b /"
done
