# A/B: 8-byte (0) vs 16-byte pair (2) stores in the k_build_ws fill (JIT dynamics)
GM_BUILD_OPTS=2 GM_JIT=1 timeout 900 python -m pytest tests/test_gpu_jit.py -q -x -k build > gpurun_out/pytest_p2.log 2>&1; echo "pytest(pairs) rc=$?"; tail -1 gpurun_out/pytest_p2.log
GM_BUILD_OPTS=2 timeout 900 python -m pytest tests -q -m gpu -x -k "matrix or build or cli" > gpurun_out/pytest_p2b.log 2>&1; echo "pytest(pairs, interp) rc=$?"; tail -1 gpurun_out/pytest_p2b.log
for o in 0 2 0 2; do
  GM_BUILD_OPTS=$o timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --extra "" > gpurun_out/cmpb_$o.json 2>gpurun_out/cmpb_$o.err
  echo "opts=$o rc=$?"; python3 -c "
import json; d=json.loads(open('gpurun_out/cmpb_$o.json').read().strip().splitlines()[-1])
print({a:round(b,2) for a,b in d['kernel_ms_per_step'].items()}, d['clocks']['sm_mhz'])"
done
