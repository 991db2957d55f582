#!/bin/bash
# cooperative merge by slot ranks vs the bitonic sort: parity, A/B on doc-contiguous data, counters
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest -q tests/test_gpu_bursts.py tests/test_gpu_retrieval.py tests/test_gpu_fp32_edges.py -x > gpurun_out/c14_t.log 2>&1; echo "rc=$?" >> gpurun_out/c14_t.log
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest -q tests/test_gpu_bursts.py -x -k "mixed or duplicate" > gpurun_out/c14_memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/c14_memcheck.log
for rep in 1 2 3; do
for lib in libragsched_b200.so _variants/bitonic.so; do
  tag=$(basename $lib .so); L=$PWD/paper_2412_10543_b200/$lib
  RAGSCHED_B200_LIB=$L timeout 600 python bench.py --workload cfg2 --data doc_contiguous --steps 40 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/c14_${tag}_cfg2doc_$rep.json 2>/dev/null
  if [ $rep -le 2 ]; then
  RAGSCHED_B200_LIB=$L timeout 600 python bench.py --workload cfg4 --data doc_contiguous --steps 8 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c14_${tag}_cfg4doc_$rep.json 2>/dev/null
  RAGSCHED_B200_LIB=$L timeout 600 python bench.py --workload cfg1 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/c14_${tag}_cfg1_$rep.json 2>/dev/null
  fi
done
done
for v in prof prof_bitonic; do
  RAGSCHED_B200_LIB=$PWD/paper_2412_10543_b200/_variants/$v.so timeout 600 python tools/pair_profile.py --workload cfg2 --data doc_contiguous > gpurun_out/c14_${v}_cfg2doc.txt 2>&1
done
echo done > gpurun_out/C14DONE
