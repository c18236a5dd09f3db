#!/usr/bin/env bash
# k_fused_run: colleague shifts of t + 2 from the previous day's table entry (no read after the wait): repeated tests, parity, config-1 A/B
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${AB_TAG:-s}
LIBS=B REPS=12 K="reset_after or deterministic" TAG=$T bash tools/flaky_check.sh
EPI_B200_LIB=build/ab/libB.so timeout 1200 python -m pytest tests/test_gpu_persistent.py tests/test_gpu_fused_lambda.py tests/test_gpu_confignet.py -q -x > gpurun_out/${T}_tests.txt 2>&1
bash tools/ab_timing.sh build/ab/libA.so build/ab/libB.so > gpurun_out/${T}_c1.txt 2>&1
