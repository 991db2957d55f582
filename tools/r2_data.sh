#!/bin/bash
# data-robustness: the same cfg4 / cfg2 step on the mixture corpus families
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for W in cfg4 cfg2; do for D in iso clustered doc_contiguous; do
  timeout 900 python bench.py --workload $W --data $D --steps 10 --warmup 3 --no-e2e --no-cpu-baseline \
    > gpurun_out/data_${W}_${D}.json 2> gpurun_out/data_${W}_${D}.err
done; done
