mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_variants.py tests/test_gpu_parity.py tests/test_gpu_fullhorizon.py tests/test_gpu_checked.py -q -m gpu --timeout 900 -rf -x > gpurun_out/pytest_gpu17.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu17.log
timeout 900 python scripts/configs_table.py --only C2a,C3n,C1,C3u --no-cpu > gpurun_out/configs17.log 2>&1; echo "configs rc=$?"; grep "^| C" gpurun_out/configs17.log
grep '"C2a"\|"C3n"' gpurun_out/configs17.log | python3 -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['workload'], d['gpu_sweep_s'], d['kernel_ms'])"
