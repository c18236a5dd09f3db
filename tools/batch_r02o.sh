#!/usr/bin/env bash
# Re-entry check of HEAD: full GPU suite, smoke(), default bench line, config 2 and config 3 lines
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${TAG:-o}
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/${T}_gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_gpu_tests.log
timeout 300 python -c 'import __graft_entry__ as g; g.smoke(); print("smoke ok")' > gpurun_out/${T}_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/${T}_bench_c1.json 2> gpurun_out/${T}_bench_c1.err
timeout 900 python bench.py --workload config2 --steps 20 --warmup 5 --no-partition --no-message-pass --no-cpu-baseline > gpurun_out/${T}_bench_c2.json 2> gpurun_out/${T}_bench_c2.err
timeout 900 python bench.py --workload config3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_bench_c3.json 2> gpurun_out/${T}_bench_c3.err
echo done > gpurun_out/${T}_done.txt
