#!/bin/bash
# DRAM bytes + duration of one score kernel launch (ncu, 1 pass) for the default
# library and every variant under paper_2412_10543_b200/_variants/ (GPU box).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for lib in paper_2412_10543_b200/libragsched_b200.so paper_2412_10543_b200/_variants/*.so; do
  [ -e "$lib" ] || continue
  RAGSCHED_B200_LIB=$PWD/$lib timeout 600 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
    -k regex:score_topk --clock-control none -c 1 --csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e "$@" \
    2>/dev/null | grep -E '"(dram__bytes_read.sum|gpu__time_duration.sum|lts__t_sector_hit_rate.pct)"' \
    | awk -F'","' -v l="$(basename $lib)" '{printf "%-40s %-32s %s %s\n", l, $(NF-2), $NF, $(NF-1)}' | tr -d '"'
done
