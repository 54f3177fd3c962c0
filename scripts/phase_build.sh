# per-role cycle totals of k_build_ws (GM_BUILD_OPTS bit 4) on C2b, JIT and interpreter dynamics
for j in 1 0; do
  echo "== GM_JIT=$j"; GM_JIT=$j GM_BUILD_OPTS=16 timeout 300 python scripts/prof_run.py --workload C2b --horizon 1 2>&1 | grep -E "k_build|rror" | head -4
done
