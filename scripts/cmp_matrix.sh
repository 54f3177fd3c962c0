# staged-V chunk size / box capacity sweep (GM_SV_ROWS / GM_SV_CAP) against the element table
for cfg in "96 6144" "200 9000" "400 12000" "800 20000" "et"; do
  unset GM_MATRIX_KERNEL GM_SV_ROWS GM_SV_CAP
  if [ "$cfg" = et ]; then export GM_MATRIX_KERNEL=et; else set -- $cfg; export GM_SV_ROWS=$1 GM_SV_CAP=$2; fi
  timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --extra "" > gpurun_out/cmp.json 2>gpurun_out/cmp.err
  echo "$cfg rc=$?"; python3 -c "
import json; d=json.loads(open('gpurun_out/cmp.json').read().strip().splitlines()[-1])
print({a:round(b,2) for a,b in d['kernel_ms_per_step'].items()}, round(d['roofline']['avg_launch_ms'],2), d['clocks']['sm_mhz'])"
done
