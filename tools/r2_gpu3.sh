#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest -q -x tests/test_gpu_reference_sim.py -s > gpurun_out/f4.log 2>&1
echo "f4 rc=$?" >> gpurun_out/f4.log
timeout 900 python tools/dropin_sim.py > gpurun_out/dropin_sim.jsonl 2> gpurun_out/dropin_sim.err
timeout 2400 python -m pytest -q tests -m gpu -x --ignore=tests/test_gpu_reference_sim.py --ignore=tests/test_gpu_fullsize.py > gpurun_out/gputests.log 2>&1
echo "gpu tests rc=$?" >> gpurun_out/gputests.log
