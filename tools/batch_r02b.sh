#!/usr/bin/env bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m pytest tests/test_gpu_persistent.py tests/test_gpu_fused_lambda.py -q -x > gpurun_out/b_tests.log 2>&1
python tools/lanes_timing.py 32 31 30 32 > gpurun_out/lanes.txt 2>&1
timeout 600 python tools/timeline_partition.py --agents 2000000 --days 4 > gpurun_out/timeline2.txt 2>&1
echo done > gpurun_out/b_done.txt
