#!/bin/bash
# round-2 final measurement on the current code: GPU suite, smoke, default line + reference arm, workload sweep,
# data families, ncu full captures of the pair kernel (cfg4 / cfg2 / cfg1 + refine), launch list of the default step
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > gpurun_out/c10_gpu.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/c10_tests.log 2>&1; echo "rc=$?" >> gpurun_out/c10_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/c10_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/c10_bench_default.json 2> gpurun_out/c10_bench_default.err
timeout 900 python bench.py --impl reference > gpurun_out/c10_ref.json 2> gpurun_out/c10_ref.err
: > gpurun_out/c10_workloads.jsonl
for args in "--workload cfg1" "--workload cfg2" "--workload cfg3" "--workload cfg5" \
            "--workload cfg4 --queries 4096" "--workload cfg4 --queries 1024" "--workload cfg4 --queries 256" \
            "--workload cfg4 --queries 128" "--workload cfg4 --queries 64" "--workload cfg4 --queries 16" \
            "--workload cfg2 --data clustered" "--workload cfg2 --data doc_contiguous" \
            "--workload cfg4 --data clustered" "--workload cfg4 --data doc_contiguous"; do
  timeout 900 python bench.py --no-cpu-baseline --steps 10 --warmup 3 $args 2>>gpurun_out/c10_workloads.err | tail -1 >> gpurun_out/c10_workloads.jsonl
done
timeout 300 python tools/select_bench.py > gpurun_out/c10_select_bench.log 2>&1
for W in cfg4 cfg2 cfg1; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:score_topk_pair --launch-skip 2 -c 1 \
    -o gpurun_out/c10_pair_$W python tools/one_search.py --workload $W > gpurun_out/c10_ncu_$W.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:refine_fp32 --launch-skip 2 -c 1 \
  -o gpurun_out/c10_refine_cfg1 python tools/one_search.py --workload cfg1 > gpurun_out/c10_ncu_refine.log 2>&1
timeout 900 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/c10_launches_cfg4.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c10_l4.log 2>&1
timeout 900 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/c10_launches_cfg1.csv python bench.py --workload cfg1 --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c10_l1.log 2>&1
echo done > gpurun_out/C10DONE
