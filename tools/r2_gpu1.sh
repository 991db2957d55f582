#!/bin/bash
# round-2 first GPU pass: new parity tests + the default bench line
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest -q -x tests/test_gpu_synth.py tests/test_gpu_workload.py tests/test_bench_contract.py -m gpu > gpurun_out/t1.log 2>&1
echo "tests rc=$?" >> gpurun_out/t1.log
timeout 900 python bench.py > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err
echo "bench rc=$?" >> gpurun_out/bench_cfg4.err
