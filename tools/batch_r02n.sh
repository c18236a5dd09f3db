#!/usr/bin/env bash
# round-2 re-entry final measurements: full GPU suite + smoke, bench lines
# (config 1 default, config 2 at 21 / 84, config 3), launch list, ncu of
# k_fused_run and of config 3's day kernel, k_iv_run timeline
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/p_full.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/p_smoke.txt 2>&1
python bench.py > gpurun_out/p_bench.json 2> gpurun_out/p_bench.err
python bench.py --workload config2 --steps 10 --warmup 3 > gpurun_out/p_c2_21.json 2> gpurun_out/p_c2_21.err
python bench.py --workload config2 --dose-gap 84 --steps 10 --warmup 3 > gpurun_out/p_c2_84.json 2> gpurun_out/p_c2_84.err
python bench.py --workload config3 --steps 5 --warmup 2 > gpurun_out/p_c3.json 2> gpurun_out/p_c3.err
B="python bench.py --steps 2 --warmup 1 --no-partition --no-message-pass --no-cpu-baseline --mode fused"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/p_launches.csv $B > gpurun_out/p_ncu0.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_fused_run -c 1 -o gpurun_out/p_fusedrun -f $B > gpurun_out/p_ncu1.log 2>&1
python tools/profile_c3.py --days 62 > gpurun_out/p_pc3.log 2>&1 && ncu --set full --import-source on --clock-control none -k regex:k_fused_step --launch-skip 60 --launch-count 1 -o gpurun_out/p_fused10M -f python tools/profile_c3.py --days 62 > gpurun_out/p_ncu3.log 2>&1
EPI_B200_LIB=build/trace/libepib200.so python tools/iv_timeline.py > gpurun_out/p_ivtl.txt 2>&1
echo done > gpurun_out/p_done.txt
