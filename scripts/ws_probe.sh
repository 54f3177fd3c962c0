timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -1
python scripts/prof_run.py --workload C5 --horizon 1 > gpurun_out/p2.log 2>&1
timeout 120 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_c5.csv python scripts/prof_run.py --workload C5 --horizon 1 > /dev/null 2>&1
cat gpurun_out/p2.log
