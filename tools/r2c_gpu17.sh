#!/bin/bash
# final-code robustness: retrieval fuzz (document blocks, both pair-kernel variants), fixed-seed slice, racecheck / memcheck
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python tools/fuzz_retrieval.py 900 6 > gpurun_out/c17_fuzz6.log 2>&1; echo "rc=$?" >> gpurun_out/c17_fuzz6.log
timeout 900 python -m pytest -q tests/test_gpu_fuzz.py tests/test_gpu_bursts.py > gpurun_out/c17_t.log 2>&1; echo "rc=$?" >> gpurun_out/c17_t.log
timeout 1200 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest -q tests/test_gpu_bursts.py -x -k "mixed and bfloat16 and 0" > gpurun_out/c17_racecheck.log 2>&1; echo "rc=$?" >> gpurun_out/c17_racecheck.log
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest -q tests/test_gpu_bursts.py -x -k "lean" > gpurun_out/c17_memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/c17_memcheck.log
echo done > gpurun_out/C17DONE
