#!/bin/bash
# e2e warm-up of every host ring slot: re-measure the lines whose e2e lagged (cfg3, mid/small batches)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
: > gpurun_out/c13_workloads.jsonl
for args in "--workload cfg3" "--workload cfg4 --queries 1024" "--workload cfg4 --queries 256" "--workload cfg4 --queries 128" \
            "--workload cfg4 --queries 64" "--workload cfg4 --queries 16" "--workload cfg2 --data doc_contiguous"; do
  timeout 900 python bench.py --no-cpu-baseline --steps 10 --warmup 3 $args 2>>gpurun_out/c13_workloads.err | tail -1 >> gpurun_out/c13_workloads.jsonl
done
echo done > gpurun_out/C13DONE
