#!/bin/bash
# burst merge policy A/B (interleaved): coop0 (lockstep only), default, A (coop at group sites only),
# D (one buffer check per two groups, BUF 24), D0 (D without coop)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest -q tests/test_gpu_bursts.py tests/test_gpu_fp32_edges.py -x > gpurun_out/c5_t.log 2>&1; echo "rc=$?" >> gpurun_out/c5_t.log
RAGSCHED_B200_LIB=$PWD/paper_2412_10543_b200/_variants/D.so timeout 600 python -m pytest -q tests/test_gpu_bursts.py tests/test_gpu_fp32_edges.py tests/test_gpu_retrieval.py -x > gpurun_out/c5_tD.log 2>&1; echo "rc=$?" >> gpurun_out/c5_tD.log
for rep in 1 2 3 4; do
for lib in _variants/coop0.so libragsched_b200.so _variants/A.so _variants/D.so _variants/D0.so; do
  tag=$(basename $lib .so)
  L=$PWD/paper_2412_10543_b200/$lib
  RAGSCHED_B200_LIB=$L timeout 600 python bench.py --workload cfg2 --data iso --steps 40 --warmup 5 --no-e2e --no-cpu-baseline \
      > gpurun_out/c5_${tag}_cfg2_iso_$rep.json 2> gpurun_out/c5_${tag}_cfg2_iso_$rep.err
  if [ $rep -le 2 ]; then
  RAGSCHED_B200_LIB=$L timeout 600 python bench.py --workload cfg2 --data doc_contiguous --steps 40 --warmup 5 --no-e2e --no-cpu-baseline \
      > gpurun_out/c5_${tag}_cfg2_doc_$rep.json 2> gpurun_out/c5_${tag}_cfg2_doc_$rep.err
  RAGSCHED_B200_LIB=$L timeout 600 python bench.py --workload cfg4 --steps 8 --warmup 3 --no-e2e --no-cpu-baseline \
      > gpurun_out/c5_${tag}_cfg4_iso_$rep.json 2> gpurun_out/c5_${tag}_cfg4_iso_$rep.err
  fi
done
done
echo done > gpurun_out/C5DONE
