# k_expect_matrix_et: loads in flight per lane x residency (GM_ET_VARIANT)
#timeout 900 python -m pytest tests -q -m gpu -x -k "matrix" > gpurun_out/pt.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pt.log
for v in 0 5 0 5; do
  GM_ET_VARIANT=$v timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --extra "" > gpurun_out/ce.json 2>gpurun_out/ce.err
  python3 -c "
import json; d=json.loads(open('gpurun_out/ce.json').read().strip().splitlines()[-1])
print('variant $v', round(d['roofline']['avg_launch_ms'],3), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"
done
