mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_variants.py tests/test_gpu_fullhorizon.py tests/test_gpu_jit.py -q -m gpu --timeout 900 -rf -x > gpurun_out/pytest_gpu22.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu22.log
for gr in 1 0; do GM_OFA_GROUP=$gr timeout 900 python scripts/configs_table.py --only C5,C3b,C4p --no-cpu > gpurun_out/ofa_group$gr.log 2>&1; echo "group=$gr"; grep '^| C' gpurun_out/ofa_group$gr.log; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_expect_ofa -c 1 -s 30 \
  -o gpurun_out/ncu_ofa_group_C5 -f python scripts/prof_run.py --workload C5 --horizon 2 > gpurun_out/ncu_ofa_group.log 2>&1; echo "ncu rc=$?"
