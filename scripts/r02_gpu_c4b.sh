#!/bin/bash
python -m pytest tests/test_gpu_variants.py tests/test_gpu_large.py -x -q 2>&1 | tail -5 > gpurun_out/t_c4b.log
python scripts/configs_table.py --only C4,C4p,C5 --no-cpu > gpurun_out/cfg_c4.log 2>&1
