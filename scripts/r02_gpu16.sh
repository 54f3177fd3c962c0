mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_build_ws -c 1 \
  -o gpurun_out/ncu_build_r02d -f python scripts/prof_run.py --workload C2b --horizon 1 > gpurun_out/ncu_build_r02d.log 2>&1; echo "ncu build rc=$?"
