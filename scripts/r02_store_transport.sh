#!/bin/bash
# multi-device synthesis with the store transport (pass-2 epilogue writes into the peers'
# value tables) on one GPU listed several times, vs peer copies: parity + timing
timeout 1500 python -m pytest tests/test_gpu_multi.py tests/test_integration.py -x -q 2>&1 | tail -3 > gpurun_out/store_t.log
for t in peer store; do
  for d in 0,0 0,0,0,0; do
    s=$(date +%s%N); paper_2005_06191_b200/gridmdp synthesize -c tests/golden/large/C5.cfg -o /tmp/r_$t.bin --devices $d --transport $t > /tmp/o_$t.txt 2>&1
    echo "C5 $t devices=$d rc=$? $(grep -E 'time_sweep_s|v_exchange' /tmp/o_$t.txt | tr '\n' ' ')" >> gpurun_out/store_t.log
  done
done
cmp /tmp/r_peer.bin /tmp/r_store.bin && echo "containers identical" >> gpurun_out/store_t.log
