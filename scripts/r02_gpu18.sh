mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none -k regex:k_expect_matrix -c 2 -s 4 \
  -o gpurun_out/ncu_c2a_matrix -f python scripts/prof_run.py --workload C2a --horizon 8 > gpurun_out/ncu_c2a.log 2>&1; echo "ncu rc=$?"
GM_MATRIX_SMALL=0 timeout 900 ncu --set full --clock-control none -k regex:k_expect_matrix -c 2 -s 4 \
  -o gpurun_out/ncu_c2a_matrix_et -f python scripts/prof_run.py --workload C2a --horizon 8 > gpurun_out/ncu_c2a_et.log 2>&1; echo "ncu rc=$?"
