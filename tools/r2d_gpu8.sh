#!/bin/bash
# final rule (limiter only for exactly one round of units): parity + A/B at the affected and neighbouring shapes
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest -q tests/test_gpu_probe.py tests/test_gpu_retrieval.py tests/test_gpu_bursts.py tests/test_gpu_fuzz.py -x > gpurun_out/d8_t.log 2>&1; echo "rc=$?" >> gpurun_out/d8_t.log
for rep in 1 2; do
for lib in libragsched_b200.so _variants/sync0.so; do
  tag=$(basename $lib .so); L=$PWD/paper_2412_10543_b200/$lib
  for q in 320 512 768 1024; do
    RAGSCHED_B200_LIB=$L timeout 300 python bench.py --workload cfg4 --queries $q --steps 20 --warmup 5 --no-cpu-baseline | sed "s/^/$tag q$q /" >> gpurun_out/d8_ab.txt 2>> gpurun_out/d8_ab.err
  done
  RAGSCHED_B200_LIB=$L timeout 300 python bench.py --workload cfg2 --queries 512 --steps 20 --warmup 5 --no-cpu-baseline | sed "s/^/$tag cfg2q512 /" >> gpurun_out/d8_ab.txt 2>> gpurun_out/d8_ab.err
done
done
echo done > gpurun_out/D8DONE
