#!/usr/bin/env bash
# message pass alone at 10M agents (tools/msgpass_timing.py) for several builds (EPI_B200_LIB)
cd "$(dirname "$0")/.."
for i in 1 2 3; do
  for v in "$@"; do
    echo "== $v"; EPI_B200_LIB=$v python tools/msgpass_timing.py 2>&1 | tail -1
  done
done
