mkdir -p gpurun_out
for cfg in "1 56" "1 64" "2 64" "1 110" "2 110" "2 80"; do
  set -- $cfg
  GM_OFA_ROWS=$1 GM_OFA_SMEM_KB=$2 timeout 600 python scripts/configs_table.py --only C5 --no-cpu > gpurun_out/ofa_t_$1_$2.log 2>&1; echo "rows=$1 smem=$2 $(grep '^| C5' gpurun_out/ofa_t_$1_$2.log)"
done
