#!/usr/bin/env bash
# A/B of build/ab/libA.so (HEAD) vs build/ab/libB.so: k_iv_run without the end barrier on notifier-free days
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${AB_TAG:-p}
EPI_B200_LIB=build/ab/libB.so timeout 1200 python -m pytest tests/test_gpu_persistent.py tests/test_gpu_fused_lambda.py tests/test_gpu_confignet.py tests/test_gpu_partition.py -q -x > gpurun_out/${T}_tests.txt 2>&1
bash tools/ab_timing.sh build/ab/libA.so build/ab/libB.so --iv > gpurun_out/${T}_c2.txt 2>&1
echo done > gpurun_out/${T}_done.txt
