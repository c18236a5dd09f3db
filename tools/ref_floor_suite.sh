#!/usr/bin/env bash
# the reference's fast suite under the plugin, with runner.bench wall times logged
cd "$(dirname "$0")/.."
export PYTHONPATH="$PWD/baseline/_ref:$PWD/tests/reference_suite:$PWD:$PYTHONPATH"
for i in 1 2 3; do
  export B200_PLUGIN_BENCH_LOG=$PWD/gpurun_out/bench_log_$i.txt
  (cd baseline/_ref && python -m pytest -p no:cacheprovider -p b200_plugin tests -q -m "not slow" -o addopts= --rootdir tests > ../../gpurun_out/suite_$i.txt 2>&1)
  tail -n 2 gpurun_out/suite_$i.txt
done
