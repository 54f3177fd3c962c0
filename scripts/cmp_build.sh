GM_BUILD_OPTS=128 timeout 900 python -m pytest tests -q -m gpu -x -k "matrix or build or cli" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest(staged) rc=$?"; tail -1 gpurun_out/pytest_gpu.log
GM_BUILD_OPTS=144 timeout 300 python scripts/prof_run.py --workload C2b --horizon 1 2>&1 | grep -E "k_build|rror" | head -5
for o in 0 128 0 128; do
  GM_BUILD_OPTS=$o timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --extra "" > gpurun_out/cmpb_$o.json 2>gpurun_out/cmpb_$o.err
  echo "opts=$o rc=$?"; python3 -c "
import json; d=json.loads(open('gpurun_out/cmpb_$o.json').read().strip().splitlines()[-1])
print({a:round(b,2) for a,b in d['kernel_ms_per_step'].items()}, d['clocks']['sm_mhz'])"
done
