#!/usr/bin/env bash
# config 3 (10M agents, 1 GPU) ms per simulation for several builds (EPI_B200_LIB)
cd "$(dirname "$0")/.."
for i in 1 2; do
  for v in "$@"; do
    echo "== $v"; EPI_B200_LIB=$v python bench.py --workload config3 --steps 3 --warmup 1 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], 'ms/sim')"
  done
done
