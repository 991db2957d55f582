#!/bin/bash
# final HEAD check: smoke, retrieval + probe/limiter tests, default bench line
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/d13_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/d13_smoke.log
timeout 1200 python -m pytest -q tests/test_gpu_probe.py tests/test_gpu_retrieval.py tests/test_gpu_config.py tests/test_gpu_api.py -x > gpurun_out/d13_t.log 2>&1; echo "rc=$?" >> gpurun_out/d13_t.log
timeout 900 python bench.py > gpurun_out/d13_bench.json 2> gpurun_out/d13_bench.err
echo done > gpurun_out/D13DONE
