# compute-sanitizer over every kernel family: memcheck, racecheck
# (shared-memory hazards: named barriers, row-claim counters, warp roles), synccheck.
# Summaries -> gpurun_out/sanitize/ (copied to profiles/r02/ by hand).
O=gpurun_out/sanitize
mkdir -p $O
CS=/usr/local/cuda/bin/compute-sanitizer
run() { # tool scenario env...
  local tool=$1 sc=$2; shift 2
  local tag=${tool}_${sc}${*:+_$(echo "$*" | tr ' =' '__')}
  env "$@" timeout 600 $CS --tool $tool --error-exitcode 99 --print-limit 20 \
      python scripts/sanitize_cases.py $sc > $O/$tag.log 2>&1
  echo "$tag rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|scenario .* ok' $O/$tag.log | tr '\n' ' ')"
}
for tool in memcheck racecheck synccheck; do
  run $tool core GM_JIT=0
  run $tool jit GM_JIT=1
  run $tool et2 GM_JIT=0
  run $tool et2 GM_JIT=0 GM_ET_VARIANT=5
  run $tool ofa_pk GM_JIT=0 GM_OFA_PK=1
  run $tool ofa_pk GM_JIT=0 GM_OFA_TABLE=global
  run $tool ofa_pk GM_JIT=0 GM_OFA_TABLE=prefix GM_OFA_PK=1
  run $tool custom GM_JIT=0
  run $tool sim GM_JIT=0
  run $tool multi GM_JIT=0
  run $tool build_single GM_JIT=0 GM_BUILD_WS=0 GM_MATRIX_KERNEL=walk
done
