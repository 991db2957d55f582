#!/bin/bash
# round 2 (session 3): re-verify HEAD on a fresh box: GPU tests, smoke, default bench, reference arm
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > gpurun_out/c1_gpu.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/c1_tests.log 2>&1; echo "rc=$?" >> gpurun_out/c1_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/c1_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/c1_bench.json 2> gpurun_out/c1_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/c1_ref.json 2> gpurun_out/c1_ref.err
echo done > gpurun_out/C1DONE
