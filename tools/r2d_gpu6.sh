#!/bin/bash
# drift limiter on by default (2-4 query tiles, window 2): full GPU suite, then A/B vs sync0 on the affected shapes
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/d6_tests.log 2>&1; echo "rc=$?" >> gpurun_out/d6_tests.log
for rep in 1 2; do
for lib in libragsched_b200.so _variants/sync0.so; do
  tag=$(basename $lib .so); L=$PWD/paper_2412_10543_b200/$lib
  RAGSCHED_B200_LIB=$L timeout 300 python bench.py --workload cfg1 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e | sed "s/^/$tag cfg1 /" >> gpurun_out/d6_ab.txt 2>> gpurun_out/d6_ab.err
  for q in 384 512 768 1024; do
    RAGSCHED_B200_LIB=$L timeout 300 python bench.py --workload cfg4 --queries $q --steps 20 --warmup 5 --no-cpu-baseline --no-e2e | sed "s/^/$tag q$q /" >> gpurun_out/d6_ab.txt 2>> gpurun_out/d6_ab.err
  done
done
done
echo done > gpurun_out/D6DONE
