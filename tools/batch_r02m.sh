#!/usr/bin/env bash
# per-line profiles of HEAD's persistent kernels (k_fused_run, k_iv_run)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --no-partition --no-message-pass --no-cpu-baseline --mode fused"
ncu --set full --import-source on --clock-control none -k regex:k_fused_run -c 1 -o gpurun_out/n_fusedrun -f $B > gpurun_out/n_ncu1.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_iv_run -c 1 -o gpurun_out/n_ivrun -f python bench.py --steps 1 --warmup 1 --no-partition --no-message-pass --no-cpu-baseline --mode fused --workload config2 > gpurun_out/n_ncu2.log 2>&1
echo done > gpurun_out/n_done.txt
