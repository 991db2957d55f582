#!/bin/bash
# probe pass: parity (on / off / auto bit-identical + oracle), then timing A/B per workload
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest -q tests/test_gpu_probe.py -x > gpurun_out/d2_t.log 2>&1; echo "rc=$?" >> gpurun_out/d2_t.log
if grep -q "rc=0" gpurun_out/d2_t.log; then
  for rep in 1 2; do
    for p in off on; do
      for w in cfg1 cfg2 cfg3; do
        timeout 300 python bench.py --workload $w --probe $p --steps 20 --warmup 5 --no-cpu-baseline >> gpurun_out/d2_ab.jsonl 2>> gpurun_out/d2_ab.err
      done
      timeout 300 python bench.py --workload cfg4 --queries 1024 --probe $p --steps 10 --warmup 3 --no-cpu-baseline >> gpurun_out/d2_ab.jsonl 2>> gpurun_out/d2_ab.err
    done
  done
  timeout 1500 python -m pytest -q tests/test_gpu_retrieval.py tests/test_gpu_retrieval_golden.py tests/test_gpu_fuzz.py tests/test_gpu_bursts.py tests/test_gpu_fp32_edges.py -x > gpurun_out/d2_t2.log 2>&1; echo "rc=$?" >> gpurun_out/d2_t2.log
fi
echo done > gpurun_out/D2DONE
