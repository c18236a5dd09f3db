#!/usr/bin/env bash
# A/B timing of two builds of the library (EPI_B200_LIB), alternating processes:
#   bash tools/ab_timing.sh libA.so libB.so [args for fused_run_timing.py]
cd "$(dirname "$0")/.."
A=$1; B=$2; shift 2
for i in 1 2 3; do
  for v in "$A" "$B"; do
    echo "== $v"; EPI_B200_LIB=$v python tools/fused_run_timing.py 15 "$@" 2>&1 | grep ms/sim
  done
done
