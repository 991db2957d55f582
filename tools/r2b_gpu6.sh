#!/bin/bash
# multi-rank cascade bound (RS_PAIR_CAS_MULTI): A/B on one box, two passes
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for rep in 1 2; do
for lib in libragsched_b200.so _variants/m4.so _variants/m7.so _variants/m9.so; do
  tag=$(basename $lib .so)
  for D in doc_contiguous iso clustered; do
    RAGSCHED_B200_LIB=$PWD/paper_2412_10543_b200/$lib timeout 600 python bench.py --workload cfg2 --data $D --steps 50 --warmup 5 --no-e2e --no-cpu-baseline \
      > gpurun_out/c6_${tag}_cfg2_${D}_$rep.json 2> gpurun_out/c6_${tag}_cfg2_${D}_$rep.err
  done
  if [ $rep = 1 ]; then
    RAGSCHED_B200_LIB=$PWD/paper_2412_10543_b200/$lib timeout 600 python bench.py --workload cfg4 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline \
      > gpurun_out/c6_${tag}_cfg4.json 2> gpurun_out/c6_${tag}_cfg4.err
    RAGSCHED_B200_LIB=$PWD/paper_2412_10543_b200/$lib timeout 600 python bench.py --workload cfg3 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline \
      > gpurun_out/c6_${tag}_cfg3.json 2> gpurun_out/c6_${tag}_cfg3.err
  fi
done
done
for D in iso doc_contiguous; do
  RAGSCHED_B200_LIB=$PWD/paper_2412_10543_b200/_variants/m7prof.so timeout 600 python tools/pair_profile.py \
    --workload cfg2 --data $D > gpurun_out/c6_prof_cfg2_${D}.txt 2>&1
done
RAGSCHED_B200_LIB=$PWD/paper_2412_10543_b200/_variants/m7.so timeout 900 python -m pytest -q tests/test_gpu_bursts.py tests/test_gpu_retrieval.py tests/test_gpu_fuzz.py -x > gpurun_out/t6.log 2>&1
echo "rc=$?" >> gpurun_out/t6.log
echo done > gpurun_out/ALLDONE6
