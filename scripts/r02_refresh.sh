# Round-2 evidence refresh after the late changes: GPU suite, bench line, configs table
# (GPU columns re-measured, CPU columns reused from the first table), launch list,
# ncu --set full of the bench's top kernels
set -u
O=gpurun_out/r02d
mkdir -p $O
timeout 2400 python -m pytest tests -q -m gpu --timeout 900 -rf > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
timeout 1800 python scripts/configs_table.py --cpu-from profiles/r02/configs.md --out $O/configs.md > $O/configs.log 2>&1; echo "configs rc=$?"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file $O/launches_bench.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu > $O/launches_bench.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_expect_matrix_et -c 1 \
  -o $O/ncu_expect_matrix -f python scripts/prof_run.py --workload C2b --horizon 1 > $O/ncu_em.log 2>&1; echo "ncu em rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_expect_ofa -c 1 -s 30 \
  -o $O/ncu_expect_ofa_C5 -f python scripts/prof_run.py --workload C5 --horizon 2 > $O/ncu_ofa.log 2>&1; echo "ncu ofa rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_build_ws -c 1 \
  -o $O/ncu_build -f python scripts/prof_run.py --workload C2b --horizon 1 > $O/ncu_build.log 2>&1; echo "ncu build rc=$?"
