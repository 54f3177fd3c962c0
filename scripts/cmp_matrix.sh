# A/B of the stored-matrix stage-(ii) kernels on C2b (GM_MATRIX_KERNEL / GM_ER_MINB / GM_CONTIG)
for k in et etc er4 er4c; do
  unset GM_MATRIX_KERNEL GM_ER_MINB GM_CONTIG
  case $k in er4) export GM_ER_MINB=4;; er4c) export GM_ER_MINB=4 GM_CONTIG=1;; et) export GM_MATRIX_KERNEL=et;; etc) export GM_MATRIX_KERNEL=et GM_CONTIG=1;; esac
  timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --extra "" > gpurun_out/cmp_$k.json 2>gpurun_out/cmp_$k.err
  echo "$k rc=$?"
done
