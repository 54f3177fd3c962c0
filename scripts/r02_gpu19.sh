mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_variants.py tests/test_gpu_parity.py -q -m gpu --timeout 900 -rf -x > gpurun_out/pytest_gpu19.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu19.log
for ms in 1 0; do GM_MATRIX_SMALL=$ms timeout 900 python scripts/configs_table.py --only C2a,C3n --no-cpu > gpurun_out/configs19_$ms.log 2>&1; echo "small=$ms"; grep "^| C" gpurun_out/configs19_$ms.log
grep '"C2a"\|"C3n"' gpurun_out/configs19_$ms.log | python3 -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['workload'], d['gpu_sweep_s'], d['kernel_ms'])"; done
timeout 900 ncu --set full --clock-control none -k regex:k_expect_matrix -c 1 -s 4 \
  -o gpurun_out/ncu_c2a_small -f python scripts/prof_run.py --workload C2a --horizon 8 > gpurun_out/ncu_c2a_small.log 2>&1; echo "ncu rc=$?"
