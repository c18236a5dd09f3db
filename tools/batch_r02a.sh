#!/usr/bin/env bash
# round-2 GPU batch: sanitizers, timeline, extra bench lines (outputs -> gpurun_out/)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m pytest tests/test_gpu_fused_lambda.py tests/test_gpu_persistent.py tests/test_gpu_partition.py -q > gpurun_out/a_tests.log 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_run.py > gpurun_out/san_$tool.txt 2>&1
  echo "rc=$?" >> gpurun_out/san_$tool.txt
done
timeout 600 python tools/timeline_partition.py --agents 2000000 --days 5 > gpurun_out/timeline.txt 2>&1
python bench.py --precision f64 --mode csr --steps 10 --warmup 3 --no-partition --no-message-pass --no-cpu-baseline > gpurun_out/bench_f64.json 2> gpurun_out/bench_f64.err
python bench.py --workload config0 --steps 20 --warmup 5 --no-partition --no-message-pass > gpurun_out/bench_c0.json 2> gpurun_out/bench_c0.err
python bench.py --workload config2 --dose-gap 84 --steps 20 --warmup 5 --no-partition --no-message-pass > gpurun_out/bench_c2_84.json 2> gpurun_out/bench_c2_84.err
python bench.py --workload config2 --dose-gap 21 --steps 20 --warmup 5 --no-partition --no-message-pass > gpurun_out/bench_c2_21.json 2> gpurun_out/bench_c2_21.err
python bench.py --impl reference --workload config0 --steps 10 --warmup 2 > gpurun_out/bench_c0_ref.json 2> gpurun_out/bench_c0_ref.err
python bench.py --impl reference --workload config2 --dose-gap 84 --steps 10 --warmup 2 > gpurun_out/bench_c2_84_ref.json 2> gpurun_out/bench_c2_84_ref.err
echo done > gpurun_out/a_done.txt
