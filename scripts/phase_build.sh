# per-role cycle totals of k_build_ws (GM_BUILD_OPTS bit 4) on C2b
for o in 24; do
  echo "== opts $o"; GM_BUILD_OPTS=$o timeout 300 python scripts/prof_run.py --workload C2b --horizon 1 2>&1 | grep -E "k_build|Error|error" | head -4
done
