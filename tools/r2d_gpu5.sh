#!/bin/bash
# drift limiter (RS_PAIR_SYNC_TILES) in the 2-8 query-tile regime: parity, DRAM bytes, A/B timing
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
V=$PWD/paper_2412_10543_b200/_variants
RAGSCHED_B200_LIB=$V/sync2.so timeout 900 python -m pytest -q tests/test_gpu_retrieval.py tests/test_gpu_fuzz.py tests/test_gpu_bursts.py tests/test_gpu_retrieval_golden.py -x > gpurun_out/d5_t.log 2>&1; echo "rc=$?" >> gpurun_out/d5_t.log
grep -q "rc=0" gpurun_out/d5_t.log || { echo done > gpurun_out/D5DONE; exit 0; }
for lib in libragsched_b200.so _variants/sync2.so _variants/sync4.so; do
  tag=$(basename $lib .so); L=$PWD/paper_2412_10543_b200/$lib
  for q in 512 1024; do
    RAGSCHED_B200_LIB=$L timeout 600 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:score_topk_pair --launch-skip 2 -c 1 --csv \
      python tools/one_search.py --workload cfg4 --queries $q > gpurun_out/d5_ncu_${tag}_q$q.csv 2>&1
  done
done
for rep in 1 2; do
for lib in libragsched_b200.so _variants/sync2.so _variants/sync4.so; do
  tag=$(basename $lib .so); L=$PWD/paper_2412_10543_b200/$lib
  for q in 512 1024 2048; do
    RAGSCHED_B200_LIB=$L timeout 300 python bench.py --workload cfg4 --queries $q --steps 20 --warmup 5 --no-cpu-baseline --no-e2e | sed "s/^/$tag q$q /" >> gpurun_out/d5_ab.txt 2>> gpurun_out/d5_ab.err
  done
done
done
echo done > gpurun_out/D5DONE
