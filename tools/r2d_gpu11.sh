#!/bin/bash
# retrieval fuzz on the final kernels (drift limiter on by plan, probe pass on half the cases): seeds 9 and 10
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python tools/fuzz_retrieval.py 600 9 > gpurun_out/d11_fuzz9.log 2>&1; echo "rc=$?" >> gpurun_out/d11_fuzz9.log
timeout 900 python tools/fuzz_retrieval.py 600 10 > gpurun_out/d11_fuzz10.log 2>&1; echo "rc=$?" >> gpurun_out/d11_fuzz10.log
echo done > gpurun_out/D11DONE
