# GPU tests, then one ncu --set full capture of each stage-(ii)/(i) kernel on C2b
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_expect_matrix_et -c 1 \
  -o gpurun_out/ncu_em_et -f python scripts/prof_run.py --workload C2b --horizon 1 > gpurun_out/ncu_em_et.log 2>&1; echo "ncu em rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on --replay-mode application -k regex:k_build -c 1 \
  -o gpurun_out/ncu_build -f python scripts/prof_run.py --workload C2b --horizon 1 > gpurun_out/ncu_build.log 2>&1; echo "ncu build rc=$?"
