#!/bin/bash
# drift limiter enabled by the plan (2-4 query tiles, whole rounds): parity, A/B vs sync0, default bench
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest -q tests/test_gpu_probe.py tests/test_gpu_retrieval.py tests/test_gpu_fuzz.py tests/test_gpu_bursts.py tests/test_gpu_fullsize.py tests/test_gpu_dist_multirank.py -x > gpurun_out/d7_t.log 2>&1; echo "rc=$?" >> gpurun_out/d7_t.log
for rep in 1 2; do
for lib in libragsched_b200.so _variants/sync0.so; do
  tag=$(basename $lib .so); L=$PWD/paper_2412_10543_b200/$lib
  RAGSCHED_B200_LIB=$L timeout 300 python bench.py --workload cfg1 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e | sed "s/^/$tag cfg1 /" >> gpurun_out/d7_ab.txt 2>> gpurun_out/d7_ab.err
  for q in 384 512 768 1024; do
    RAGSCHED_B200_LIB=$L timeout 300 python bench.py --workload cfg4 --queries $q --steps 20 --warmup 5 --no-cpu-baseline | sed "s/^/$tag q$q /" >> gpurun_out/d7_ab.txt 2>> gpurun_out/d7_ab.err
  done
done
done
timeout 600 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:score_topk_pair --launch-skip 2 -c 1 --csv \
      python tools/one_search.py --workload cfg4 --queries 512 > gpurun_out/d7_ncu_q512.csv 2>&1
timeout 900 python bench.py > gpurun_out/d7_bench.json 2> gpurun_out/d7_bench.err
echo done > gpurun_out/D7DONE
