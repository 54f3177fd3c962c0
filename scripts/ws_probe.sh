GM_MATRIX_KERNEL=cp timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -2
python scripts/prof_run.py --workload C2b --horizon 2 > gpurun_out/p1.log 2>&1
for k in plain cp; do GM_MATRIX_KERNEL=$k timeout 120 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:expect_matrix --log-file gpurun_out/lk_$k.csv python scripts/prof_run.py --workload C2b --horizon 2 > /dev/null 2>&1; done
cat gpurun_out/p1.log
