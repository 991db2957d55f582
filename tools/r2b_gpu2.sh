#!/bin/bash
# fused fp32 tail (merge + exact re-rank in one kernel, norms + tf32 split in one pass),
# epilogue event counters per data family, shorter-segment DRAM sweep, fp32 peaks
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
( time timeout 1500 python -m pytest -q tests -m gpu -x ) > gpurun_out/gputests2.log 2>&1
echo "gpu tests rc=$?" >> gpurun_out/gputests2.log
timeout 300 python tools/measure_fp32_peaks.py > gpurun_out/fp32_peaks.json 2> gpurun_out/fp32_peaks.err
timeout 600 python bench.py --workload cfg1 --steps 20 --warmup 5 > gpurun_out/bench_cfg1.json 2> gpurun_out/bench_cfg1.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
   --log-file gpurun_out/launches_cfg1.csv python bench.py --workload cfg1 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_cfg1.log 2>&1
for D in iso clustered doc_contiguous; do
  timeout 600 python bench.py --workload cfg2 --data $D --steps 50 --warmup 5 --no-e2e --no-cpu-baseline \
    > gpurun_out/data50_cfg2_${D}.json 2> gpurun_out/data50_cfg2_${D}.err
  RAGSCHED_B200_LIB=$PWD/paper_2412_10543_b200/_variants/prof.so timeout 600 python tools/pair_profile.py \
    --workload cfg2 --data $D > gpurun_out/prof_cfg2_${D}.txt 2>&1
done
for D in iso doc_contiguous; do
  RAGSCHED_B200_LIB=$PWD/paper_2412_10543_b200/_variants/prof.so timeout 900 python tools/pair_profile.py \
    --workload cfg4 --data $D > gpurun_out/prof_cfg4_${D}.txt 2>&1
done
for S in 16384 8192; do
  timeout 600 python bench.py --workload cfg4 --steps 8 --warmup 3 --segment-rows $S --no-cpu-baseline --no-e2e \
     > gpurun_out/seg_cfg4_${S}.json 2> gpurun_out/seg_cfg4_${S}.err
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
     --clock-control none -k regex:score_topk_pair --launch-skip 2 -c 1 --csv \
     python tools/one_search.py --workload cfg4 --segment-rows $S > gpurun_out/seg_cfg4_${S}.ncu.csv 2>&1
done
echo done > gpurun_out/ALLDONE2
