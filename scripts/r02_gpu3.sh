# GPU suite (all), then the C2b bench with / without the shape-specialised build
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu --timeout 900 --durations=40 -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -50 gpurun_out/pytest_gpu.log
for shp in 1 0; do
  GM_JIT_SHAPE=$shp timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --extra "" > gpurun_out/bench_shape$shp.json 2> gpurun_out/bench_shape$shp.err; echo "bench shape=$shp rc=$?"
  python3 -c "
import json; d=json.loads(open('gpurun_out/bench_shape$shp.json').read().strip().splitlines()[-1])
print('shape=$shp', {a:round(b,2) for a,b in d['kernel_ms_per_step'].items()}, d['clocks'], round(d['value']/1e9,1), round(d['roofline_build']['frac'],3))"
done
