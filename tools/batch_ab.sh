#!/usr/bin/env bash
# A/B of build/ab/libA.so (before) vs build/ab/libB.so (after): parity tests of the
# persistent kernels with libB, then alternating timings of config 1 and config 2
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${AB_TAG:-ab}
EPI_B200_LIB=build/ab/libB.so timeout 900 python -m pytest tests/test_gpu_persistent.py tests/test_gpu_fused_lambda.py -q -x > gpurun_out/${T}_tests.txt 2>&1
bash tools/ab_timing.sh build/ab/libA.so build/ab/libB.so > gpurun_out/${T}_c1.txt 2>&1
bash tools/ab_timing.sh build/ab/libA.so build/ab/libB.so --iv > gpurun_out/${T}_c2.txt 2>&1
echo done > gpurun_out/${T}_done.txt
