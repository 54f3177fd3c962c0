mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_large.py tests/test_gpu_jit.py tests/test_gpu_checked.py -q -m gpu --timeout 900 -rf > gpurun_out/pytest_gpu14.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu14.log
for d in 1 0; do
GM_BUILD_HOST_DIRECT=$d timeout 900 python bench.py --no-cpu --extra "" > gpurun_out/bench14_$d.json 2> gpurun_out/bench14_$d.err; echo "bench direct=$d rc=$?"
python3 -c "
import json; d=json.loads(open('gpurun_out/bench14_$d.json').read().strip().splitlines()[-1])
print({a:round(b,2) for a,b in d['kernel_ms_per_step'].items()}, d['clocks']['sm_mhz'], round(d['value']/1e9,1), 'e2e', d['e2e']['value']/1e9, d['e2e']['seconds_per_step'], d['e2e_synthesize'])"
done
