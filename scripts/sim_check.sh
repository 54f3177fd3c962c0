timeout 900 python -m pytest tests/test_gpu_sim.py -q -x > gpurun_out/pytest_sim.log 2>&1; echo "pytest sim rc=$?"; tail -25 gpurun_out/pytest_sim.log
