# GPU suite + source-level ncu capture of the C2b build kernel
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu --timeout 900 --durations=40 -rf -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -60 gpurun_out/pytest_gpu.log
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_build_ws -c 1 \
  -o gpurun_out/ncu_build_r02 -f python scripts/prof_run.py --workload C2b --horizon 1 > gpurun_out/ncu_build_r02.log 2>&1; echo "ncu build rc=$?"; tail -3 gpurun_out/ncu_build_r02.log
