# k_expect_ofa on C4 (R = 78,125; the line table does not fit shared memory):
# leading-prefix offset table in shared memory (default) vs line offsets from global memory
for t in default global default global; do
  if [ $t = default ]; then unset GM_OFA_TABLE; else export GM_OFA_TABLE=$t; fi
  timeout 400 python scripts/configs_table.py --only C4 --no-cpu > gpurun_out/cot_$t.log 2>&1
  echo "table=$t"; grep '"workload": "C4"' gpurun_out/cot_$t.log | python3 -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l[l.index('{'):]); print(' sweep_s', round(d['gpu_sweep_s'],3), 'hbm_equiv', round(d['hbm_equiv_frac'],3), 'ofa_ms', round(d['kernel_ms']['expect_ofa'],1))"
done
unset GM_OFA_TABLE
