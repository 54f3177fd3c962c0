python -m pytest tests/test_gpu_large.py -k "chains or traffic" -x -q -s 2>&1 | tail -15 > gpurun_out/t_large.log
python -m pytest tests/test_gpu_variants.py -x -q 2>&1 | tail -15 > gpurun_out/t_var.log
bash scripts/r02_pk_minb.sh > gpurun_out/minb.log 2>&1
