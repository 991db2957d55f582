#!/bin/bash
# One bench line per BASELINE config shape + the HBM-bound small-batch regime
# + the config-path-only throughput (cfg5); GPU box.  Output: gpurun_out/workloads.jsonl
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
: > gpurun_out/workloads.jsonl
for args in "--workload cfg1" "--workload cfg2" "--workload cfg3" "--workload cfg4" \
            "--workload cfg4 --queries 256" "--workload cfg4 --queries 128" "--workload cfg4 --queries 64"; do
  timeout 900 python bench.py --no-cpu-baseline $args 2>/dev/null | tail -1 >> gpurun_out/workloads.jsonl
done
timeout 300 python tools/select_bench.py > gpurun_out/select_bench.log 2>&1
