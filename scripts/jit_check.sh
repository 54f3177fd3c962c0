# JIT parity tests, full GPU suite, then the C2b / C5 bench with JIT (auto) vs interpreter
timeout 900 python -m pytest tests/test_gpu_jit.py -q -x > gpurun_out/pytest_jit.log 2>&1; echo "pytest jit rc=$?"; tail -15 gpurun_out/pytest_jit.log
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest gpu rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for j in auto 0; do
  unset GM_JIT; [ $j = 0 ] && export GM_JIT=0
  timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/cmpj_$j.json 2>gpurun_out/cmpj_$j.err
  echo "jit=$j rc=$?"; python3 -c "
import json; d=json.loads(open('gpurun_out/cmpj_$j.json').read().strip().splitlines()[-1])
print({a:round(b,2) for a,b in d['kernel_ms_per_step'].items()}, d['clocks']['sm_mhz'], d['extra']['C5']['sweep_s'], d['extra']['C5']['kernel_ms'])"
done
