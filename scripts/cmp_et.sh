# k_expect_matrix_et(2): loads in flight per lane x residency (GM_ET_VARIANT) on the bench sweep
for v in 0 1 2 3 4 5 0; do
  GM_ET_VARIANT=$v timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --extra "" > gpurun_out/ce.json 2>gpurun_out/ce.err
  python3 -c "
import json; d=json.loads(open('gpurun_out/ce.json').read().strip().splitlines()[-1])
print('variant $v', round(d['roofline']['avg_launch_ms'],3), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['roofline']['kernel'])"
done
