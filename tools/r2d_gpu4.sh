#!/bin/bash
# L2 prefetch of the corpus tiles ahead of the TMA loads in the HBM / ridge regime (nq 128-1024), A/B vs default
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for rep in 1 2; do
for lib in libragsched_b200.so _variants/pf1.so _variants/pf2.so; do
  tag=$(basename $lib .so); L=$PWD/paper_2412_10543_b200/$lib
  for q in 128 256 512 1024; do
    RAGSCHED_B200_LIB=$L timeout 300 python bench.py --workload cfg4 --queries $q --steps 20 --warmup 5 --no-cpu-baseline --no-e2e | sed "s/^/$tag q$q /" >> gpurun_out/d4_ab.txt 2>> gpurun_out/d4_ab.err
  done
  if [ $rep -eq 1 ]; then
    RAGSCHED_B200_LIB=$L timeout 300 python bench.py --workload cfg4 --queries 8192 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e | sed "s/^/$tag q8192 /" >> gpurun_out/d4_ab.txt 2>> gpurun_out/d4_ab.err
  fi
done
done
echo done > gpurun_out/D4DONE
