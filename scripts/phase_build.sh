# per-phase cycle totals of k_build (GM_BUILD_OPTS bit 2) for each option set
for o in 4 6; do
  echo "== opts $o"; GM_BUILD_OPTS=$o timeout 300 python scripts/prof_run.py --workload C2b --horizon 1 2>&1 | grep -E "k_build|Error|error" | head -4
done
