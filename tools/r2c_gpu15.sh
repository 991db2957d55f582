#!/bin/bash
# rank merge: lower burst thresholds (MIN 4 / GAIN 3, MIN 4 / GAIN 2) vs the default (MIN 6 / GAIN 5)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for rep in 1 2 3; do
for lib in libragsched_b200.so _variants/g3.so _variants/g2.so; do
  tag=$(basename $lib .so); L=$PWD/paper_2412_10543_b200/$lib
  RAGSCHED_B200_LIB=$L timeout 600 python bench.py --workload cfg2 --data doc_contiguous --steps 40 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/c15_${tag}_cfg2doc_$rep.json 2>/dev/null
  RAGSCHED_B200_LIB=$L timeout 600 python bench.py --workload cfg1 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/c15_${tag}_cfg1_$rep.json 2>/dev/null
  RAGSCHED_B200_LIB=$L timeout 600 python bench.py --workload cfg2 --data iso --burst-merge on --steps 40 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/c15_${tag}_cfg2isoon_$rep.json 2>/dev/null
done
done
echo done > gpurun_out/C15DONE
