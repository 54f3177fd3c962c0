# k_build_ws residency (GM_BUILD_CTAS) with the interpreter kernels (GM_JIT=0), then JIT default
for c in 4 3 4 3; do
  GM_BUILD_CTAS=$c timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --extra "" > gpurun_out/cc.json 2>gpurun_out/cc.err
  python3 -c "
import json; d=json.loads(open('gpurun_out/cc.json').read().strip().splitlines()[-1])
print('ctas $c', round(d['build_ms_per_step'],2), round(d['roofline']['avg_launch_ms'],2), d['clocks']['sm_mhz'])"
done
