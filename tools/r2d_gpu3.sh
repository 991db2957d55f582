#!/bin/bash
# probe pass at cfg1: per-launch durations (probe / fold / main) and per-role counters, on vs off
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for p in on off; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/d3_launch_$p.csv \
    python tools/one_search.py --workload cfg1 --probe $p --warmup 2 --reps 2 > gpurun_out/d3_launch_$p.log 2>&1
  RAGSCHED_B200_LIB=$PWD/paper_2412_10543_b200/_variants/prof.so timeout 600 python tools/pair_profile.py --workload cfg1 --probe $p > gpurun_out/d3_prof_$p.txt 2>&1
done
echo done > gpurun_out/D3DONE
