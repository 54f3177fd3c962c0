# row pitch A/B: unpadded (GM_PITCH_GRANULE=1) vs 256-byte rows (default), full and constant-store builds
for gr in 1 32 1 32; do
  for o in 0 32; do
    GM_PITCH_GRANULE=$gr GM_BUILD_OPTS=$o timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --extra "" > gpurun_out/cp.json 2>gpurun_out/cp.err
    python3 -c "
import json; d=json.loads(open('gpurun_out/cp.json').read().strip().splitlines()[-1])
print('granule $gr opts $o', {a:round(b,2) for a,b in d['kernel_ms_per_step'].items()}, d['clocks']['sm_mhz'])"
  done
done
