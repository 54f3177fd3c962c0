GM_BUILD_PIPE=1 GM_BUILD_OPTS=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_prologue|k_expand|k_build" --csv --log-file gpurun_out/pipe_launches.csv python scripts/prof_run.py --workload C2b --horizon 1 > gpurun_out/pipe_ncu.log 2>&1; echo rc=$?
python scripts/launches.py gpurun_out/pipe_launches.csv
