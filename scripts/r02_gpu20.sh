mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_variants.py tests/test_gpu_fullhorizon.py tests/test_gpu_parity.py -q -m gpu --timeout 900 -rf -x > gpurun_out/pytest_gpu20.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu20.log
for ms in 1 0; do GM_MATRIX_SMALL=$ms timeout 900 python scripts/configs_table.py --only C2a,C3n --no-cpu > gpurun_out/configs20_$ms.log 2>&1; echo "small=$ms"; grep "^| C" gpurun_out/configs20_$ms.log; done
for pk in 1 0; do GM_OFA_PACK=$pk timeout 600 python scripts/configs_table.py --only C5 --no-cpu > gpurun_out/c5_pack$pk.log 2>&1; echo "pack=$pk $(grep '^| C5' gpurun_out/c5_pack$pk.log)"; done
