#!/bin/bash
# cooperative burst flush: parity tests, cfg2 data families, counters, cfg4 line
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest -q tests/test_gpu_bursts.py tests/test_gpu_retrieval.py tests/test_gpu_retrieval_golden.py -x > gpurun_out/t3.log 2>&1
echo "rc=$?" >> gpurun_out/t3.log
for D in iso doc_contiguous clustered; do
  timeout 600 python bench.py --workload cfg2 --data $D --steps 50 --warmup 5 --no-e2e --no-cpu-baseline \
    > gpurun_out/c3_cfg2_${D}.json 2> gpurun_out/c3_cfg2_${D}.err
done
for D in iso doc_contiguous; do
  RAGSCHED_B200_LIB=$PWD/paper_2412_10543_b200/_variants/prof.so timeout 600 python tools/pair_profile.py \
    --workload cfg2 --data $D > gpurun_out/c3_prof_cfg2_${D}.txt 2>&1
done
timeout 600 python bench.py --workload cfg4 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/c3_cfg4.json 2> gpurun_out/c3_cfg4.err
timeout 600 python bench.py --workload cfg4 --data doc_contiguous --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c3_cfg4_doc.json 2> gpurun_out/c3_cfg4_doc.err
timeout 1500 python -m pytest -q tests -m gpu -x > gpurun_out/t3_all.log 2>&1
echo "rc=$?" >> gpurun_out/t3_all.log
echo done > gpurun_out/ALLDONE3
