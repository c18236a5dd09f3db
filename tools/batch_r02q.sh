#!/usr/bin/env bash
# k_fused_run wtab race fix: repeated equality tests with libB, parity tests, config-1 and config-2 A/B timings
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${AB_TAG:-w}
LIBS=B REPS=12 TAG=$T bash tools/flaky_check.sh
EPI_B200_LIB=build/ab/libB.so timeout 1200 python -m pytest tests/test_gpu_persistent.py tests/test_gpu_fused_lambda.py tests/test_gpu_confignet.py tests/test_gpu_partition.py -q -x > gpurun_out/${T}_tests.txt 2>&1
bash tools/ab_timing.sh build/ab/libA.so build/ab/libB.so > gpurun_out/${T}_c1.txt 2>&1
bash tools/ab_timing.sh build/ab/libA.so build/ab/libB.so --iv > gpurun_out/${T}_c2.txt 2>&1
