#!/bin/bash
# cooperative burst merge: interleaved A/B (4 reps) of the lockstep-only build and three policies
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest -q tests/test_gpu_bursts.py -x > gpurun_out/c4_t.log 2>&1; echo "rc=$?" >> gpurun_out/c4_t.log
for rep in 1 2 3 4; do
for lib in _variants/coop0.so libragsched_b200.so _variants/m4g4.so _variants/g8.so; do
  tag=$(basename $lib .so)
  for D in iso doc_contiguous clustered; do
    RAGSCHED_B200_LIB=$PWD/paper_2412_10543_b200/$lib timeout 600 python bench.py --workload cfg2 --data $D --steps 40 --warmup 5 --no-e2e --no-cpu-baseline \
      > gpurun_out/c4_${tag}_cfg2_${D}_$rep.json 2> gpurun_out/c4_${tag}_cfg2_${D}_$rep.err
  done
  if [ $rep -le 2 ]; then
  RAGSCHED_B200_LIB=$PWD/paper_2412_10543_b200/$lib timeout 600 python bench.py --workload cfg3 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline \
      > gpurun_out/c4_${tag}_cfg3_iso_$rep.json 2> gpurun_out/c4_${tag}_cfg3_iso_$rep.err
  fi
done
done
echo done > gpurun_out/C4DONE
