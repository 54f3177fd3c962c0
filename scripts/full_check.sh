timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest gpu rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/b12.json 2>gpurun_out/b12.err; echo "bench rc=$?"
python3 -c "
import json; d=json.loads(open('gpurun_out/b12.json').read().strip().splitlines()[-1])
print({a:round(b,2) for a,b in d['kernel_ms_per_step'].items()}, d['clocks']['sm_mhz'], round(d['value']/1e9,1), d['extra']['C5']['sweep_s'])"
