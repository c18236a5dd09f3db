#!/usr/bin/env bash
# ncu captures of the round-2 build (after the plain runs exit 0)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --no-partition --no-message-pass --no-cpu-baseline --mode fused"
$B > gpurun_out/c_plain.json 2> gpurun_out/c_plain.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/c_launches.csv $B > gpurun_out/c_ncu1.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_fused_run -c 1 -o gpurun_out/c_fusedrun -f $B > gpurun_out/c_ncu2.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_iv_run -c 1 -o gpurun_out/c_ivrun -f python bench.py --steps 1 --warmup 1 --no-partition --no-message-pass --no-cpu-baseline --mode fused --workload config2 > gpurun_out/c_ncu3.log 2>&1
python tools/profile_day.py --agents 10000000 --days 4 > gpurun_out/c_pd.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_fused_step --launch-skip 2 --launch-count 1 -o gpurun_out/c_fused10M -f python tools/profile_day.py --agents 10000000 --days 4 > gpurun_out/c_ncu4.log 2>&1
echo done > gpurun_out/c_done.txt
