#!/bin/bash
# cooperative burst merge (RS_TOPK_COOP): correctness on the default build, then A/B vs lockstep-only (coop0)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest -q tests/test_gpu_bursts.py tests/test_gpu_retrieval.py tests/test_gpu_fuzz.py tests/test_gpu_retrieval_golden.py tests/test_gpu_fp32_edges.py -x > gpurun_out/c3_t.log 2>&1
echo "rc=$?" >> gpurun_out/c3_t.log
for rep in 1 2; do
for lib in libragsched_b200.so _variants/coop0.so _variants/g3.so _variants/g8.so _variants/m4g4.so; do
  tag=$(basename $lib .so)
  for D in doc_contiguous iso; do
    RAGSCHED_B200_LIB=$PWD/paper_2412_10543_b200/$lib timeout 600 python bench.py --workload cfg2 --data $D --steps 50 --warmup 5 --no-e2e --no-cpu-baseline \
      > gpurun_out/c3_${tag}_cfg2_${D}_$rep.json 2> gpurun_out/c3_${tag}_cfg2_${D}_$rep.err
  done
done
done
for lib in libragsched_b200.so _variants/coop0.so; do
  tag=$(basename $lib .so)
  RAGSCHED_B200_LIB=$PWD/paper_2412_10543_b200/$lib timeout 600 python bench.py --workload cfg4 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline \
    > gpurun_out/c3_${tag}_cfg4_iso.json 2> gpurun_out/c3_${tag}_cfg4_iso.err
  RAGSCHED_B200_LIB=$PWD/paper_2412_10543_b200/$lib timeout 600 python bench.py --workload cfg4 --data doc_contiguous --steps 10 --warmup 3 --no-e2e --no-cpu-baseline \
    > gpurun_out/c3_${tag}_cfg4_doc.json 2> gpurun_out/c3_${tag}_cfg4_doc.err
done
for v in prof_coop0 prof_def; do
  for D in iso doc_contiguous; do
    RAGSCHED_B200_LIB=$PWD/paper_2412_10543_b200/_variants/$v.so timeout 600 python tools/pair_profile.py \
      --workload cfg2 --data $D > gpurun_out/c3_${v}_cfg2_${D}.txt 2>&1
  done
done
echo done > gpurun_out/C3DONE
