# build in 1 / 4 / 16 slices (GM_BUILD_SLICES) inside the bench loop
for sl in 1 4 16 1 4; do
  GM_BUILD_SLICES=$sl timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --extra "" > gpurun_out/cs.json 2>gpurun_out/cs.err
  python3 -c "
import json; d=json.loads(open('gpurun_out/cs.json').read().strip().splitlines()[-1])
print('slices $sl', {a:round(b,2) for a,b in d['kernel_ms_per_step'].items()}, d['build_ms_per_step'], d['clocks']['sm_mhz'])"
done
