#!/bin/bash
# one round trip per admission chunk (admit + plan expansion in stream order): parity + timings
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest -q tests/test_gpu_api.py tests/test_gpu_config.py tests/test_gpu_scheduler.py tests/test_gpu_reference_sim.py tests/test_gpu_mapping_a1.py -x > gpurun_out/c26_t.log 2>&1; echo "rc=$?" >> gpurun_out/c26_t.log
timeout 600 python tools/scalar_latency.py > gpurun_out/c26_scalar.txt 2>&1
timeout 900 python tools/dropin_sim.py > gpurun_out/c26_dropin_sim.jsonl 2> gpurun_out/c26_dropin_sim.err
echo done > gpurun_out/C26DONE
