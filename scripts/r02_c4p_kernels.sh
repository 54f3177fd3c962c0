#!/bin/bash
# C4p / C5 OFA consumer choice: per-group NVRTC kernel vs batched shape kernel vs the
# ahead-of-time hoisted-cell kernel
for w in C4p C5; do
  python scripts/c3b_repeat.py $w 2 2
  GM_OFA_GROUP=0 python scripts/c3b_repeat.py $w 2 2
  GM_JIT=0 python scripts/c3b_repeat.py $w 2 2
  GM_JIT=0 GM_OFA_PK=1 python scripts/c3b_repeat.py $w 2 2
done
