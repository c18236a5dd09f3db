#!/usr/bin/env bash
# tools/iv_phase_cost.py over several builds of the library (EPI_B200_LIB)
cd "$(dirname "$0")/.."
for i in 1 2; do
  for v in "$@"; do
    echo "== $v"; EPI_B200_LIB=$v python tools/iv_phase_cost.py 2>&1 | grep ms/sim
  done
done
