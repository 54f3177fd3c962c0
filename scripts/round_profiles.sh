# Round evidence: bench line, launch list of the bench command, ncu --set full of the top kernels.
set -u
O=gpurun_out/r01
mkdir -p $O
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_bench.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu > $O/launches_bench.log 2>&1; echo "ncu launches rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C5_T1.csv \
  python scripts/prof_run.py --workload C5 --horizon 1 > $O/launches_C5.log 2>&1; echo "ncu C5 launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_expect_matrix_et -c 1 \
  -o $O/ncu_expect_matrix -f python scripts/prof_run.py --workload C2b --horizon 1 > $O/ncu_em.log 2>&1; echo "ncu em rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_expect_ofa -c 1 \
  -o $O/ncu_expect_ofa -f python scripts/prof_run.py --workload C5 --horizon 1 > $O/ncu_ofa.log 2>&1; echo "ncu ofa rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on --replay-mode application -k regex:k_build -c 1 \
  -o $O/ncu_build -f python scripts/prof_run.py --workload C2b --horizon 1 > $O/ncu_build.log 2>&1; echo "ncu build rc=$?"
