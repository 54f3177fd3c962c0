timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for o in 8 8; do
  GM_BUILD_OPTS=$o timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --extra "" > gpurun_out/cmpb_$o.json 2>gpurun_out/cmpb_$o.err
  echo "opts=$o rc=$?"; python3 -c "
import json; d=json.loads(open('gpurun_out/cmpb_$o.json').read().strip().splitlines()[-1])
print({a:round(b,2) for a,b in d['kernel_ms_per_step'].items()}, round(d['value']/1e9,1), d['clocks']['sm_mhz'])"
done
