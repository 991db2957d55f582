#!/bin/bash
# cooperative flush of heavy lanes: A/B (same box) vs sweep-only and a higher threshold, + counters
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest -q tests/test_gpu_bursts.py tests/test_gpu_retrieval.py -x > gpurun_out/t4.log 2>&1
echo "rc=$?" >> gpurun_out/t4.log
for rep in 1 2; do
for lib in libragsched_b200.so _variants/nocoop.so _variants/coop8.so; do
  for D in doc_contiguous iso; do
    tag=$(basename $lib .so)
    RAGSCHED_B200_LIB=$PWD/paper_2412_10543_b200/$lib timeout 600 python bench.py --workload cfg2 --data $D --steps 50 --warmup 5 --no-e2e --no-cpu-baseline \
      > gpurun_out/c4_${tag}_cfg2_${D}_$rep.json 2> gpurun_out/c4_${tag}_cfg2_${D}_$rep.err
  done
done
done
for D in iso doc_contiguous; do
  RAGSCHED_B200_LIB=$PWD/paper_2412_10543_b200/_variants/prof.so timeout 600 python tools/pair_profile.py \
    --workload cfg2 --data $D > gpurun_out/c4_prof_cfg2_${D}.txt 2>&1
done
echo done > gpurun_out/ALLDONE4
