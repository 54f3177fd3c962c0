# k_expect_ofa: terms in flight per lane (GM_OFA_U) on C5
for u in 4 6 8 4; do
  GM_OFA_U=$u timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/co.json 2>gpurun_out/co.err
  python3 -c "
import json; d=json.loads(open('gpurun_out/co.json').read().strip().splitlines()[-1])
print('U $u', d['extra']['C5']['sweep_s'], round(d['extra']['C5']['hbm_equiv_frac'],3), d['clocks']['sm_mhz'])"
done
