#!/bin/bash
# both bench arms back to back with default arguments, as the driver runs them
s=$(date +%s); python bench.py --impl reference > gpurun_out/arm_ref.json 2> gpurun_out/arm_ref.err; echo "reference rc=$? $(( $(date +%s) - s )) s"
s=$(date +%s); python bench.py > gpurun_out/arm_b200.json 2> gpurun_out/arm_b200.err; echo "b200 rc=$? $(( $(date +%s) - s )) s"
s=$(date +%s); python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/arm_smoke.log 2>&1; echo "smoke rc=$? $(( $(date +%s) - s )) s"
