mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu --timeout 900 -rf > gpurun_out/pytest_gpu23.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu23.log
for gr in 0 1 0 1; do GM_OFA_GROUP=$gr timeout 900 python scripts/configs_table.py --only C3b --no-cpu > gpurun_out/c3b_$gr.log 2>&1; echo "group=$gr $(grep '^| C3b' gpurun_out/c3b_$gr.log)"; done
timeout 900 python bench.py > gpurun_out/bench23.json 2> gpurun_out/bench23.err; echo "bench rc=$?"
python3 -c "
import json; d=json.loads(open('gpurun_out/bench23.json').read().strip().splitlines()[-1])
print({a:round(b,2) for a,b in d['kernel_ms_per_step'].items()}, d['clocks'], round(d['value']/1e9,1), round(d['roofline']['frac'],3), d['roofline_build']['frac'], d['roofline_build'].get('frac_of_store_ceiling'), d['e2e']['value']/1e9, d['cpu_baseline']['value']/1e9)
print(d['extra']['C5']['sweep_s'], d['extra']['C5']['kernel_variant'])"
