mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_variants.py tests/test_gpu_fullhorizon.py tests/test_gpu_parity.py tests/test_gpu_large.py tests/test_gpu_multi.py -q -m gpu --timeout 900 -rf -x > gpurun_out/pytest_gpu10.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu10.log
timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/bench10.json 2> gpurun_out/bench10.err; echo "bench rc=$?"; tail -3 gpurun_out/bench10.err
python3 -c "
import json; d=json.loads(open('gpurun_out/bench10.json').read().strip().splitlines()[-1])
print({a:round(b,2) for a,b in d['kernel_ms_per_step'].items()}, d['clocks'], round(d['value']/1e9,1), round(d['roofline']['frac'],3), d['roofline_build']['frac'], d['roofline_build'].get('frac_of_store_ceiling'), d['store_ceiling'])
print(d['extra']['C5'])"
for c in 1 0; do GM_OFA_CACHE=$c timeout 600 python scripts/configs_table.py --only C5,C3b,C4p --no-cpu > gpurun_out/ofa_cache$c.log 2>&1; echo "cache=$c"; grep '^| C' gpurun_out/ofa_cache$c.log; done
