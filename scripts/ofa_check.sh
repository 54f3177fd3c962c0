timeout 900 python -m pytest tests -q -m gpu -x -k "ofa or synthesis or step or bmw or jit" > gpurun_out/pt.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pt.log
for i in 1 2; do timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/b14.json 2>&1; python3 -c "
import json; d=json.loads(open('gpurun_out/b14.json').read().strip().splitlines()[-1])
print({a:round(b,2) for a,b in d['kernel_ms_per_step'].items()}, d['clocks']['sm_mhz'], d['extra']['C5']['sweep_s'], d['extra']['C5']['hbm_equiv_frac'])"; done
