#!/bin/bash
# retrieval fuzz with document blocks recorded (seed 6 again, seed 8), racecheck of the cooperative merge
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python tools/fuzz_retrieval.py 840 6 > gpurun_out/c18_fuzz6.log 2>&1; echo "rc=$?" >> gpurun_out/c18_fuzz6.log
timeout 1200 python tools/fuzz_retrieval.py 600 8 > gpurun_out/c18_fuzz8.log 2>&1; echo "rc=$?" >> gpurun_out/c18_fuzz8.log
timeout 1500 compute-sanitizer --tool racecheck python -m pytest -q "tests/test_gpu_bursts.py::test_mixed_burst_sizes_in_one_warp[0-dtype0]" > gpurun_out/c18_racecheck.log 2>&1; echo "rc=$?" >> gpurun_out/c18_racecheck.log
echo done > gpurun_out/C18DONE
