#!/bin/bash
# live per-list slots in the pair kernel's shared bound: parity, A/B vs RS_PAIR_LIVE=0, epilogue counters
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest -q tests/test_gpu_bursts.py tests/test_gpu_retrieval.py tests/test_gpu_fp32_edges.py tests/test_gpu_fuzz.py tests/test_gpu_retrieval_golden.py tests/test_gpu_dist_multirank.py tests/test_gpu_fullsize.py -x > gpurun_out/c12_t.log 2>&1; echo "rc=$?" >> gpurun_out/c12_t.log
for rep in 1 2 3; do
for lib in libragsched_b200.so _variants/live0.so; do
  tag=$(basename $lib .so); L=$PWD/paper_2412_10543_b200/$lib
  RAGSCHED_B200_LIB=$L timeout 600 python bench.py --workload cfg1 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/c12_${tag}_cfg1_$rep.json 2>/dev/null
  RAGSCHED_B200_LIB=$L timeout 600 python bench.py --workload cfg2 --steps 40 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/c12_${tag}_cfg2_$rep.json 2>/dev/null
  if [ $rep -le 2 ]; then
  RAGSCHED_B200_LIB=$L timeout 600 python bench.py --workload cfg4 --steps 8 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c12_${tag}_cfg4_$rep.json 2>/dev/null
  RAGSCHED_B200_LIB=$L timeout 600 python bench.py --workload cfg4 --queries 1024 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c12_${tag}_cfg4q1k_$rep.json 2>/dev/null
  RAGSCHED_B200_LIB=$L timeout 600 python bench.py --workload cfg2 --data doc_contiguous --steps 40 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/c12_${tag}_cfg2doc_$rep.json 2>/dev/null
  fi
done
done
for v in prof prof_live0; do
for a in "--workload cfg1" "--workload cfg2" "--workload cfg4"; do
  tag=$(echo $a | tr ' ' '_' | tr -d '-')
  RAGSCHED_B200_LIB=$PWD/paper_2412_10543_b200/_variants/$v.so timeout 600 python tools/pair_profile.py $a > gpurun_out/c12_${v}_$tag.txt 2>&1
done
done
echo done > gpurun_out/C12DONE
