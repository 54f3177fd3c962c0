# round-2 GPU check: full GPU suite, default bench, torchrun (NCCL) bench, CLI multi-GPU
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 2400 python -m pytest tests -q -m gpu --timeout 900 --durations=30 -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -45 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -c 3000 gpurun_out/bench.json
NCCL_DEBUG=INFO timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29531 bench.py --no-cpu --no-e2e > gpurun_out/bench_torchrun1.json 2> gpurun_out/bench_torchrun1.err; echo "torchrun rc=$?"; tail -c 1500 gpurun_out/bench_torchrun1.json
NCCL_DEBUG=INFO timeout 300 paper_2005_06191_b200/gridmdp synthesize -c tests/golden/large/C5.cfg --gpus 1 -o /tmp/c5.bin > gpurun_out/cli_c5_gpus1.log 2>&1; echo "cli rc=$?"; grep -v NCCL gpurun_out/cli_c5_gpus1.log
timeout 300 paper_2005_06191_b200/gridmdp synthesize -c tests/golden/large/C5.cfg --devices 0,0,0,0 --transport peer -o /tmp/c5p.bin > gpurun_out/cli_c5_peer4.log 2>&1; echo "cli peer rc=$?"; cat gpurun_out/cli_c5_peer4.log; cmp /tmp/c5.bin /tmp/c5p.bin && echo same-bytes
