mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu --timeout 900 -rf > gpurun_out/pytest_gpu15.log 2>&1; echo "pytest rc=$?"; tail -6 gpurun_out/pytest_gpu15.log
timeout 900 python scripts/configs_table.py --only C1,C2a,C3n,C3u,C3e --no-cpu > gpurun_out/configs15.log 2>&1; echo "configs rc=$?"; grep "^| C" gpurun_out/configs15.log
GM_STEP_FUSED=0 timeout 900 python scripts/configs_table.py --only C2a,C3n --no-cpu > gpurun_out/configs15b.log 2>&1; echo "unfused:"; grep "^| C" gpurun_out/configs15b.log
