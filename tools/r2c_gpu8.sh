#!/bin/bash
# refine_fp32_kernel: warps per CTA (8 / 4 / 2), interleaved cfg1 A/B + per-variant launch lists
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for rep in 1 2 3; do
for lib in libragsched_b200.so _variants/rw4.so _variants/rw2.so; do
  tag=$(basename $lib .so)
  RAGSCHED_B200_LIB=$PWD/paper_2412_10543_b200/$lib timeout 600 python bench.py --workload cfg1 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e \
    > gpurun_out/c8_${tag}_cfg1_$rep.json 2> gpurun_out/c8_${tag}_cfg1_$rep.err
done
done
for lib in libragsched_b200.so _variants/rw4.so _variants/rw2.so; do
  tag=$(basename $lib .so)
  RAGSCHED_B200_LIB=$PWD/paper_2412_10543_b200/$lib timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv \
    --log-file gpurun_out/c8_${tag}_launches.csv -k regex:refine python tools/one_search.py --workload cfg1 --reps 4 > /dev/null 2>&1
done
RAGSCHED_B200_LIB=$PWD/paper_2412_10543_b200/_variants/rw4.so timeout 900 python -m pytest -q tests/test_gpu_fp32_edges.py tests/test_gpu_retrieval.py -x > gpurun_out/c8_t_rw4.log 2>&1; echo "rc=$?" >> gpurun_out/c8_t_rw4.log
echo done > gpurun_out/C8DONE
