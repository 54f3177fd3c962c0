# k_expect_ofa offset-table variants per OFA workload (default plan vs forced
# GM_OFA_TABLE=global|prefix on the leading-prefix product table; pk / nopk = GM_OFA_PK=1 / 0)
#   bash scripts/cmp_ofa_table.sh "C4 C4p C3b C5" "default global prefix"
WLS=${1:-C4}
TABS=${2:-"default global default global"}
for w in $WLS; do
for t in $TABS; do
  unset GM_OFA_TABLE GM_OFA_PK
  case $t in default) ;; nopk) export GM_OFA_PK=0 ;; pk) export GM_OFA_PK=1 ;; *) export GM_OFA_TABLE=$t ;; esac
  timeout 400 python scripts/configs_table.py --only $w --no-cpu > gpurun_out/cot_${w}_$t.log 2>&1
  echo "$w table=$t"; grep "\"workload\": \"$w\"" gpurun_out/cot_${w}_$t.log | python3 -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l[l.index('{'):]); print(' sweep_s', round(d['gpu_sweep_s'],4), 'hbm_equiv', round(d['hbm_equiv_frac'],3), 'ofa_ms', round(d['kernel_ms']['expect_ofa'],1))"
done
done
unset GM_OFA_TABLE GM_OFA_PK
