timeout 1500 ncu --set full --clock-control none --import-source on --replay-mode application -k regex:k_build -c 1 \
  -o gpurun_out/ncu_build_ws -f python scripts/prof_run.py --workload C2b --horizon 1 > gpurun_out/ncu_build_ws.log 2>&1; echo "ncu build rc=$?"
