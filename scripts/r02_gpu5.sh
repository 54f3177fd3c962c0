mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu --timeout 900 -rf -x > gpurun_out/pytest_gpu5.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu5.log
timeout 900 python bench.py --no-cpu --extra C5 > gpurun_out/bench5.json 2> gpurun_out/bench5.err; echo "bench rc=$?"
python3 -c "
import json; d=json.loads(open('gpurun_out/bench5.json').read().strip().splitlines()[-1])
print({a:round(b,2) for a,b in d['kernel_ms_per_step'].items()}, d['clocks'], round(d['value']/1e9,1), round(d['roofline']['frac'],3), round(d['roofline_build']['frac'],3), d['extra']['C5']['sweep_s'], d['e2e']['value']/1e9)"
timeout 900 python scripts/configs_table.py --only C1,C2a,C3n,C3u,C3b,C5 --no-cpu > gpurun_out/configs5.log 2>&1; echo "configs rc=$?"; grep "^| C" gpurun_out/configs5.log
for co in 100 75 50; do
  GM_OFA_CARVEOUT=$co timeout 600 python scripts/configs_table.py --only C5 --no-cpu > gpurun_out/c5_carve$co.log 2>&1; echo "carveout $co: $(grep '^| C5' gpurun_out/c5_carve$co.log)"
done
