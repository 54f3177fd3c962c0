mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_jit.py tests/test_gpu_variants.py tests/test_gpu_fullhorizon.py -q -m gpu --timeout 900 -rf -x > gpurun_out/pytest_gpu11.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu11.log
for sh in 1 0; do GM_OFA_SHAPE=$sh timeout 600 python scripts/configs_table.py --only C5,C3b --no-cpu > gpurun_out/ofa_shape$sh.log 2>&1; echo "shape=$sh"; grep '^| C' gpurun_out/ofa_shape$sh.log; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_expect_ofa -c 1 -s 5 \
  -o gpurun_out/ncu_ofa_shape_C5 -f python scripts/prof_run.py --workload C5 --horizon 2 > gpurun_out/ncu_ofa_shape.log 2>&1; echo "ncu rc=$?"
