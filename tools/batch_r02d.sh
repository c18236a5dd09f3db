#!/usr/bin/env bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python bench.py --steps 20 --warmup 5 > gpurun_out/k_default.json 2> gpurun_out/k_default.err
python bench.py --workload refnet --steps 5 --warmup 2 > gpurun_out/k_refnet.json 2> gpurun_out/k_refnet.err
python bench.py --impl reference --workload refnet --steps 6 --warmup 1 > gpurun_out/k_refnet_ref.json 2> gpurun_out/k_refnet_ref.err
python bench.py --workload config4 --steps 2 --warmup 1 > gpurun_out/k_c4.json 2> gpurun_out/k_c4.err
python bench.py --workload config2 --dose-gap 84 --steps 20 --warmup 5 --no-partition --no-message-pass > gpurun_out/k_c2_84.json 2> gpurun_out/k_c2_84.err
python bench.py --workload config2 --dose-gap 21 --steps 20 --warmup 5 --no-partition --no-message-pass > gpurun_out/k_c2_21.json 2> gpurun_out/k_c2_21.err
python bench.py --workload config3 --steps 5 --warmup 2 > gpurun_out/k_c3.json 2> gpurun_out/k_c3.err
echo done > gpurun_out/k_done.txt
