python scripts/prof_run.py --workload C2b --horizon 1 > gpurun_out/p1.log 2>&1
for b in 0 1 2; do GM_BUILD_BULK=$b timeout 120 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k_build --log-file gpurun_out/lbb$b.csv python scripts/prof_run.py --workload C2b --horizon 1 > /dev/null 2>&1; done
GM_BUILD_BULK=2 timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py -q -m gpu -x 2>&1 | tail -1
cat gpurun_out/p1.log
