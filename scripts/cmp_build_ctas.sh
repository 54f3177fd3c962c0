#!/bin/bash
# k_build_ws residency (GM_BUILD_CTAS) with the run-time compiled kernels: C2b (bench,
# shape-specialised fill), the C5 half-matrix shard and C1 (generic fill)
for c in 3 2 3 2; do
  GM_BUILD_CTAS=$c python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --extra "" 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('C2b ctas $c', round(d['build_ms_per_step'],3), d['clocks']['sm_mhz'])"
  GM_BUILD_CTAS=$c python scripts/c5_build_shard.py 3 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('C5 shard ctas $c', d['build_ms'], d['kernel_variant'])"
  GM_BUILD_CTAS=$c python scripts/c3b_repeat.py C1 4 | tail -2 | sed "s/^/ctas $c /"
done
