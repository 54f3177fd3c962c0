# Power experiment: the bench step with the build's fill replaced by constant stores
# (GM_BUILD_OPTS=32) or with no stores (64); results are wrong, timings only.
for o in 0 32 64 0; do
  GM_BUILD_OPTS=$o timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --extra "" > gpurun_out/cc.json 2>gpurun_out/cc.err
  python3 -c "
import json; d=json.loads(open('gpurun_out/cc.json').read().strip().splitlines()[-1])
print('opts $o', round(d['build_ms_per_step'],2), round(d['roofline']['avg_launch_ms'],2), d['clocks']['sm_mhz'])"
done
