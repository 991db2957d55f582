#!/bin/bash
# DRAM over-fetch experiment: segment length of the pair kernel's schedule
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
W=${1:-cfg4}
for S in 0 131072 65536 32768; do
  timeout 600 python bench.py --workload $W --steps 8 --warmup 3 --segment-rows $S --no-cpu-baseline --no-e2e \
     > gpurun_out/seg_${W}_${S}.json 2> gpurun_out/seg_${W}_${S}.err
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
     --clock-control none -k regex:score_topk_pair --launch-skip 2 -c 1 --csv \
     python tools/one_search.py --workload $W --segment-rows $S > gpurun_out/seg_${W}_${S}.ncu.csv 2>&1
done
