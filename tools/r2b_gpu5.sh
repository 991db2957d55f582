#!/bin/bash
# where the doc_contiguous epilogue time goes (timing variants, wrong results by design),
# and two DRAM over-fetch probes (persisting-L2 carve-out; queries >> corpus in L2)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for lib in libragsched_b200.so _variants/noins.so _variants/noslow.so; do
  for D in doc_contiguous iso; do
    tag=$(basename $lib .so)
    RAGSCHED_B200_LIB=$PWD/paper_2412_10543_b200/$lib timeout 600 python bench.py --workload cfg2 --data $D --steps 50 --warmup 5 --no-e2e --no-cpu-baseline \
      > gpurun_out/c5_${tag}_cfg2_${D}.json 2> gpurun_out/c5_${tag}_cfg2_${D}.err
  done
done
for P in 0 48; do
  timeout 900 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
     --clock-control none -k regex:score_topk_pair --launch-skip 2 -c 1 --csv \
     python tools/one_search.py --workload cfg4 --persist-mb $P > gpurun_out/c5_persist_${P}.csv 2>&1
done
for R in 40000 400000; do
  timeout 900 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
     --clock-control none -k regex:score_topk_pair --launch-skip 2 -c 1 --csv \
     python tools/one_search.py --workload cfg4 --corpus-rows $R > gpurun_out/c5_rows_${R}.csv 2>&1
done
echo done > gpurun_out/ALLDONE5
