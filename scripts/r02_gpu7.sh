mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu --timeout 900 -rf -x > gpurun_out/pytest_gpu7.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu7.log
timeout 900 python bench.py --no-cpu --extra "" --no-e2e > gpurun_out/bench7.json 2> gpurun_out/bench7.err; echo "bench rc=$?"
python3 -c "
import json; d=json.loads(open('gpurun_out/bench7.json').read().strip().splitlines()[-1])
print({a:round(b,2) for a,b in d['kernel_ms_per_step'].items()}, d['clocks'], round(d['value']/1e9,1), round(d['roofline']['frac'],3), round(d['roofline_build']['frac'],3))"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_build_ws -c 1 \
  -o gpurun_out/ncu_build_r02c -f python scripts/prof_run.py --workload C2b --horizon 1 > gpurun_out/ncu_build_r02c.log 2>&1; echo "ncu build rc=$?"
