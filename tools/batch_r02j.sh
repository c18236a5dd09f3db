#!/usr/bin/env bash
# round-2 final measurements (bench lines of every workload, launch lists, ncu
# of the timed kernels: each capture after its plain run exited 0)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python bench.py > gpurun_out/j_default.json 2> gpurun_out/j_default.err
python bench.py --impl reference > gpurun_out/j_ref.json 2> gpurun_out/j_ref.err
python bench.py --workload config2 --dose-gap 21 --steps 20 --warmup 5 --no-partition --no-message-pass > gpurun_out/j_c2_21.json 2> gpurun_out/j_c2_21.err
python bench.py --workload config2 --dose-gap 84 --steps 20 --warmup 5 --no-partition --no-message-pass > gpurun_out/j_c2_84.json 2> gpurun_out/j_c2_84.err
python bench.py --workload config0 --steps 20 --warmup 5 --no-partition --no-message-pass > gpurun_out/j_c0.json 2> gpurun_out/j_c0.err
python bench.py --workload config3 --steps 5 --warmup 2 > gpurun_out/j_c3.json 2> gpurun_out/j_c3.err
python bench.py --workload config4 --steps 2 --warmup 1 > gpurun_out/j_c4.json 2> gpurun_out/j_c4.err
python bench.py --workload refnet --steps 5 --warmup 2 > gpurun_out/j_refnet.json 2> gpurun_out/j_refnet.err
python bench.py --precision f64 --mode csr --steps 10 --warmup 3 --no-partition --no-message-pass --no-cpu-baseline > gpurun_out/j_f64.json 2> gpurun_out/j_f64.err
B="python bench.py --steps 2 --warmup 1 --no-partition --no-message-pass --no-cpu-baseline --mode fused"
$B > gpurun_out/j_plain.json 2> gpurun_out/j_plain.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/j_launches.csv $B > gpurun_out/j_ncu0.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_fused_run -c 1 -o gpurun_out/j_fusedrun -f $B > gpurun_out/j_ncu1.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_iv_run -c 1 -o gpurun_out/j_ivrun -f python bench.py --steps 1 --warmup 1 --no-partition --no-message-pass --no-cpu-baseline --mode fused --workload config2 > gpurun_out/j_ncu2.log 2>&1
python tools/profile_c3.py --days 62 > gpurun_out/j_pc3.log 2>&1 && ncu --set full --import-source on --clock-control none -k regex:k_fused_step --launch-skip 60 --launch-count 1 -o gpurun_out/j_fused10M -f python tools/profile_c3.py --days 62 > gpurun_out/j_ncu3.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/j_c3_launches.csv python tools/profile_c3.py --days 180 > gpurun_out/j_ncu4.log 2>&1
echo done > gpurun_out/j_done.txt
