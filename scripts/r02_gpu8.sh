mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_checked.py -q -m gpu --timeout 900 -rf > gpurun_out/pytest_checked.log 2>&1; echo "checked rc=$?"; tail -15 gpurun_out/pytest_checked.log
timeout 900 python bench.py --no-cpu --extra "" --no-e2e > gpurun_out/bench8.json 2> gpurun_out/bench8.err; echo "bench rc=$?"
python3 -c "
import json; d=json.loads(open('gpurun_out/bench8.json').read().strip().splitlines()[-1])
print({a:round(b,2) for a,b in d['kernel_ms_per_step'].items()}, d['clocks'], round(d['value']/1e9,1), round(d['roofline']['frac'],3), d['roofline_build'], d['store_ceiling'])"
