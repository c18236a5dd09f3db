#!/usr/bin/env bash
# refresh after the config-3 changes: full GPU suite + smoke, config 3 bench + ncu of its day kernel, launch list
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/l_full.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/l_smoke.txt 2>&1
python bench.py --workload config3 --steps 5 --warmup 2 > gpurun_out/l_c3.json 2> gpurun_out/l_c3.err
python tools/profile_c3.py --days 62 > gpurun_out/l_pc3.log 2>&1 && ncu --set full --import-source on --clock-control none -k regex:k_fused_step --launch-skip 60 --launch-count 1 -o gpurun_out/l_fused10M -f python tools/profile_c3.py --days 62 > gpurun_out/l_ncu3.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_c3_launches.csv python tools/profile_c3.py --days 180 > gpurun_out/l_ncu4.log 2>&1
echo done > gpurun_out/l_done.txt
