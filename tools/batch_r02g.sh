#!/usr/bin/env bash
# ncu captures of the persistent kernels and the 10M sparse day kernel (after the plain runs exit 0)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --no-partition --no-message-pass --no-cpu-baseline --mode fused"
$B > gpurun_out/g_plain.json 2> gpurun_out/g_plain.err || exit 1
ncu --set full --import-source on --clock-control none -k regex:k_fused_run -c 1 -o gpurun_out/g_fusedrun -f $B > gpurun_out/g_ncu1.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_iv_run -c 1 -o gpurun_out/g_ivrun -f python bench.py --steps 1 --warmup 1 --no-partition --no-message-pass --no-cpu-baseline --mode fused --workload config2 > gpurun_out/g_ncu2.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_fused_step --launch-skip 60 --launch-count 1 -o gpurun_out/g_fused10M -f python tools/profile_c3.py --days 62 > gpurun_out/g_ncu3.log 2>&1
echo done > gpurun_out/g_done.txt
