#!/bin/bash
# TMA multicast of the corpus tile across 2 / 4 pairs (RS_PAIR_GROUP) in the mid-batch regime (nq 512-2048),
# where the pairs of a segment drift apart and re-read it from DRAM
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for rep in 1 2; do
for lib in libragsched_b200.so _variants/g2.so _variants/g4.so; do
  tag=$(basename $lib .so); L=$PWD/paper_2412_10543_b200/$lib
  for q in 512 1024 2048; do
    RAGSCHED_B200_LIB=$L timeout 600 python bench.py --workload cfg4 --queries $q --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c19_${tag}_q${q}_$rep.json 2>/dev/null
  done
  if [ $rep = 1 ]; then
    RAGSCHED_B200_LIB=$L timeout 600 python bench.py --workload cfg4 --steps 8 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c19_${tag}_q8192_$rep.json 2>/dev/null
  fi
done
done
for lib in libragsched_b200.so _variants/g4.so; do
  tag=$(basename $lib .so)
  RAGSCHED_B200_LIB=$PWD/paper_2412_10543_b200/$lib timeout 600 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none --csv \
    --log-file gpurun_out/c19_${tag}_q1024_dram.csv -k regex:score_topk_pair --launch-skip 2 -c 1 python tools/one_search.py --workload cfg4 --queries 1024 > /dev/null 2>&1
done
echo done > gpurun_out/C19DONE
