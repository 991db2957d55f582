#!/bin/bash
# after making the cooperative burst merge the default: full GPU suite, epilogue counters, bench lines, ncu of the fp32 tail
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/c6_tests.log 2>&1; echo "rc=$?" >> gpurun_out/c6_tests.log
for W in cfg2 cfg4; do for D in iso doc_contiguous clustered; do
  for v in prof prof_coop0; do
  RAGSCHED_B200_LIB=$PWD/paper_2412_10543_b200/_variants/$v.so timeout 600 python tools/pair_profile.py --workload $W --data $D \
    > gpurun_out/c6_${v}_${W}_${D}.txt 2>&1
  done
done; done
for D in iso doc_contiguous clustered; do
  timeout 600 python bench.py --workload cfg2 --data $D --steps 40 --warmup 5 > gpurun_out/c6_bench_cfg2_$D.json 2> gpurun_out/c6_bench_cfg2_$D.err
  timeout 900 python bench.py --workload cfg4 --data $D --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c6_bench_cfg4_$D.json 2> gpurun_out/c6_bench_cfg4_$D.err
done
timeout 600 python bench.py --workload cfg3 --steps 10 --warmup 3 > gpurun_out/c6_bench_cfg3.json 2> gpurun_out/c6_bench_cfg3.err
timeout 600 python bench.py --workload cfg1 --steps 50 --warmup 5 > gpurun_out/c6_bench_cfg1.json 2> gpurun_out/c6_bench_cfg1.err
timeout 600 python bench.py --workload cfg5 --steps 10 --warmup 3 > gpurun_out/c6_bench_cfg5.json 2> gpurun_out/c6_bench_cfg5.err
timeout 900 python bench.py > gpurun_out/c6_bench_default.json 2> gpurun_out/c6_bench_default.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:refine_fp32 --launch-skip 2 -c 1 \
  -o gpurun_out/c6_refine_cfg1 python tools/one_search.py --workload cfg1 > gpurun_out/c6_ncu_refine.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c6_launches_cfg1.csv \
  python tools/one_search.py --workload cfg1 --reps 4 > gpurun_out/c6_ncu_l1.log 2>&1
echo done > gpurun_out/C6DONE
