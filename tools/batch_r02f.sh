#!/usr/bin/env bash
# config 3 with sparse push rows: launch list of one simulation, ncu of the day kernel at day 60
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python tools/profile_c3.py --days 62 > gpurun_out/f_pc3.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f_c3_launches.csv python tools/profile_c3.py --days 180 > gpurun_out/f_ncu1.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_fused_step --launch-skip 60 --launch-count 1 -o gpurun_out/f_fused10M -f python tools/profile_c3.py --days 62 > gpurun_out/f_ncu2.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_fused_step --launch-skip 60 --launch-count 1 -o gpurun_out/f_fused10M_inv -f python tools/profile_c3.py --days 62 --no-sparse > gpurun_out/f_ncu3.log 2>&1
echo done > gpurun_out/f_done.txt
