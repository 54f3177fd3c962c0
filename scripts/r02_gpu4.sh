mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench4.json 2> gpurun_out/bench4.err; echo "bench rc=$?"
python3 -c "
import json; d=json.loads(open('gpurun_out/bench4.json').read().strip().splitlines()[-1])
print({a:round(b,2) for a,b in d['kernel_ms_per_step'].items()}, d['clocks'], round(d['value']/1e9,1), round(d['roofline']['frac'],3), round(d['roofline_build']['frac'],3), d['extra']['C5']['sweep_s'], d['cpu_baseline']['value'])"
timeout 2400 python scripts/configs_table.py --out gpurun_out/configs.md > gpurun_out/configs.log 2>&1; echo "configs rc=$?"; tail -14 gpurun_out/configs.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_build_ws -c 1 \
  -o gpurun_out/ncu_build_r02b -f python scripts/prof_run.py --workload C2b --horizon 1 > gpurun_out/ncu_build_r02b.log 2>&1; echo "ncu build rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_maxmin -c 1 \
  -o gpurun_out/ncu_maxmin_r02 -f python scripts/prof_run.py --workload C2b --horizon 1 > gpurun_out/ncu_maxmin_r02.log 2>&1; echo "ncu maxmin rc=$?"
