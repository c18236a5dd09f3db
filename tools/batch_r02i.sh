#!/usr/bin/env bash
# refresh after the last kernel changes: full GPU suite + smoke, config 3 bench, the fused launch list
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/i_full.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/i_smoke.txt 2>&1
python bench.py --workload config3 --steps 5 --warmup 2 > gpurun_out/i_c3.json 2> gpurun_out/i_c3.err
B="python bench.py --steps 2 --warmup 1 --no-partition --no-message-pass --no-cpu-baseline --mode fused"
$B > gpurun_out/i_plain.json 2> gpurun_out/i_plain.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/i_launches.csv $B > gpurun_out/i_ncu0.log 2>&1
python tools/profile_c3.py --days 180 > gpurun_out/i_pc3.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/i_c3_launches.csv python tools/profile_c3.py --days 180 > gpurun_out/i_ncu1.log 2>&1
echo done > gpurun_out/i_done.txt
