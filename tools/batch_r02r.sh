#!/usr/bin/env bash
# round-2 final measurements (after the k_fused_run barrier-window fix and the k_iv_run end-barrier skip):
# full GPU suite + smoke, bench lines, launch list, ncu of k_fused_run and k_iv_run, k_iv_run timeline
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${TAG:-z}
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/${T}_full.txt 2>&1; echo "rc=$?" >> gpurun_out/${T}_full.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 900 python bench.py --workload config2 --steps 10 --warmup 3 > gpurun_out/${T}_c2_21.json 2> gpurun_out/${T}_c2_21.err
timeout 900 python bench.py --workload config2 --dose-gap 84 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_c2_84.json 2> gpurun_out/${T}_c2_84.err
timeout 900 python bench.py --workload config3 --steps 5 --warmup 3 > gpurun_out/${T}_c3.json 2> gpurun_out/${T}_c3.err
B="python bench.py --steps 2 --warmup 1 --no-partition --no-message-pass --no-cpu-baseline --mode fused"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches.csv $B > gpurun_out/${T}_ncu0.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_fused_run -c 1 -o gpurun_out/${T}_fusedrun -f $B > gpurun_out/${T}_ncu1.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_iv_run -c 1 -o gpurun_out/${T}_ivrun -f python bench.py --steps 1 --warmup 1 --no-partition --no-message-pass --no-cpu-baseline --mode fused --workload config2 > gpurun_out/${T}_ncu2.log 2>&1
EPI_B200_LIB=build/trace/libepib200.so timeout 600 python tools/iv_timeline.py > gpurun_out/${T}_ivtl.txt 2>&1
echo done > gpurun_out/${T}_done.txt
