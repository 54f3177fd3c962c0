mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu --timeout 900 -rf > gpurun_out/pytest_gpu12.log 2>&1; echo "pytest rc=$?"; tail -8 gpurun_out/pytest_gpu12.log
timeout 900 python bench.py > gpurun_out/bench12.json 2> gpurun_out/bench12.err; echo "bench rc=$?"; tail -3 gpurun_out/bench12.err
python3 -c "
import json; d=json.loads(open('gpurun_out/bench12.json').read().strip().splitlines()[-1])
print({a:round(b,2) for a,b in d['kernel_ms_per_step'].items()}, d['clocks'], round(d['value']/1e9,1), round(d['roofline']['frac'],3), d['roofline_build']['frac'], d['roofline_build'].get('frac_of_store_ceiling'), d['store_ceiling']['ms'], d['e2e']['value']/1e9, d['cpu_baseline']['value']/1e9)
print(d['extra']['C5'])"
