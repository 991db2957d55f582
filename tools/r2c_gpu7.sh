#!/bin/bash
# refine_fp32_kernel v3 (lists staged in shared memory, warp-per-row gathers): parity, memcheck, cfg1 timing, ncu
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest -q tests/test_gpu_fp32_edges.py tests/test_gpu_retrieval.py tests/test_gpu_retrieval_golden.py tests/test_gpu_fuzz.py tests/test_gpu_bursts.py tests/test_gpu_dist_multirank.py -x > gpurun_out/c7_t.log 2>&1; echo "rc=$?" >> gpurun_out/c7_t.log
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest -q tests/test_gpu_fp32_edges.py -x -k "not fullsize" > gpurun_out/c7_memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/c7_memcheck.log
for rep in 1 2 3; do
  timeout 600 python bench.py --workload cfg1 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/c7_bench_cfg1_$rep.json 2> gpurun_out/c7_bench_cfg1_$rep.err
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:refine_fp32 --launch-skip 2 -c 1 \
  -o gpurun_out/c7_refine_cfg1 python tools/one_search.py --workload cfg1 > gpurun_out/c7_ncu_refine.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c7_launches_cfg1.csv \
  python tools/one_search.py --workload cfg1 --reps 4 > gpurun_out/c7_ncu_l1.log 2>&1
echo done > gpurun_out/C7DONE
