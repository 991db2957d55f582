#!/bin/bash
# experiment: one-round plans for 3-4 query tiles (72 units on 74 pairs via --segment-rows) with the drift limiter
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for rep in 1 2; do
for lib in libragsched_b200.so _variants/syncpr.so; do
  tag=$(basename $lib .so); L=$PWD/paper_2412_10543_b200/$lib
  RAGSCHED_B200_LIB=$L timeout 300 python bench.py --workload cfg4 --queries 1024 --steps 20 --warmup 5 --no-cpu-baseline | sed "s/^/$tag q1024 /" >> gpurun_out/d12_ab.txt 2>> gpurun_out/d12_ab.err
  RAGSCHED_B200_LIB=$L timeout 300 python bench.py --workload cfg4 --queries 1024 --segment-rows 555776 --steps 20 --warmup 5 --no-cpu-baseline | sed "s/^/$tag q1024s18 /" >> gpurun_out/d12_ab.txt 2>> gpurun_out/d12_ab.err
  RAGSCHED_B200_LIB=$L timeout 300 python bench.py --workload cfg4 --queries 768 --steps 20 --warmup 5 --no-cpu-baseline | sed "s/^/$tag q768 /" >> gpurun_out/d12_ab.txt 2>> gpurun_out/d12_ab.err
  RAGSCHED_B200_LIB=$L timeout 300 python bench.py --workload cfg4 --queries 768 --segment-rows 416768 --steps 20 --warmup 5 --no-cpu-baseline | sed "s/^/$tag q768s24 /" >> gpurun_out/d12_ab.txt 2>> gpurun_out/d12_ab.err
  RAGSCHED_B200_LIB=$L timeout 300 python bench.py --workload cfg1 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e | sed "s/^/$tag cfg1 /" >> gpurun_out/d12_ab.txt 2>> gpurun_out/d12_ab.err
done
done
echo done > gpurun_out/D12DONE
