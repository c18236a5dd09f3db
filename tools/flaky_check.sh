#!/usr/bin/env bash
# Repeat the persistent-kernel equality tests with several builds (EPI_B200_LIB=build/ab/lib$X.so): a race shows as an intermittent failure
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for lib in ${LIBS:-O A B}; do for i in $(seq ${REPS:-8}); do
EPI_B200_LIB=build/ab/lib$lib.so timeout 600 python -m pytest tests/test_gpu_persistent.py -q -rf -k "${K:-reset_after or deterministic or intervention_day}" 2>&1 | grep -E "passed|failed|FAILED" | sed "s/^/$lib $i: /"
done; done > gpurun_out/${TAG:-u}_flaky.txt
