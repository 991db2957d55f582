#!/bin/bash
# re-entry check of HEAD: the full GPU suite, smoke, both bench arms, the timed-region launch list
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/d1_tests.log 2>&1; echo "rc=$?" >> gpurun_out/d1_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/d1_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/d1_smoke.log
timeout 900 python bench.py > gpurun_out/d1_bench.json 2> gpurun_out/d1_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/d1_ref.json 2> gpurun_out/d1_ref.err
echo done > gpurun_out/D1DONE
