#!/usr/bin/env bash
# re-entry check of HEAD: full GPU suite + smoke + default bench line
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x > gpurun_out/m_full.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/m_smoke.txt 2>&1
python bench.py > gpurun_out/m_bench.json 2> gpurun_out/m_bench.err
python bench.py --workload config2 --steps 10 --warmup 3 > gpurun_out/m_c2.json 2> gpurun_out/m_c2.err
echo done > gpurun_out/m_done.txt
