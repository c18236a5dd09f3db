#!/usr/bin/env bash
# ncu captures of the persistent kernels (after the plain run exits 0)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --no-partition --no-message-pass --no-cpu-baseline --mode fused"
$B > gpurun_out/e_plain.json 2> gpurun_out/e_plain.err || exit 1
ncu --set full --import-source on --clock-control none -k regex:k_fused_run -c 1 -o gpurun_out/e_fusedrun -f $B > gpurun_out/e_ncu2.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_iv_run -c 1 -o gpurun_out/e_ivrun -f python bench.py --steps 1 --warmup 1 --no-partition --no-message-pass --no-cpu-baseline --mode fused --workload config2 > gpurun_out/e_ncu3.log 2>&1
echo done > gpurun_out/e_done.txt
