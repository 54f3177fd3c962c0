mkdir -p gpurun_out
timeout 900 python bench.py --no-cpu --extra "" --no-e2e > gpurun_out/bench9.json 2> gpurun_out/bench9.err; echo "bench rc=$?"; tail -3 gpurun_out/bench9.err
python3 -c "
import json; d=json.loads(open('gpurun_out/bench9.json').read().strip().splitlines()[-1])
print({a:round(b,2) for a,b in d['kernel_ms_per_step'].items()}, d['clocks'], round(d['value']/1e9,1), round(d['roofline']['frac'],3), d['roofline_build']['frac'], d['roofline_build'].get('frac_of_store_ceiling'), d['store_ceiling'])"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/launches_bench.log 2>&1; echo "ncu launches rc=$?"
