#!/bin/bash
# DRAM bytes of the fused search vs the number of query tiles (cfg4 corpus)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for Q in 128 256 512 1024 2048 4096 8192; do
  timeout 900 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
     --clock-control none -k regex:score_topk_pair --launch-skip 2 -c 1 --csv \
     python tools/one_search.py --workload cfg4 --queries $Q > gpurun_out/dram_q${Q}.csv 2>&1
done
