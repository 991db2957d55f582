#!/bin/bash
# verification on the final code: GPU suite, smoke, default line + reference arm, cfg1/cfg2/cfg5 and doc-contiguous lines
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/c16_tests.log 2>&1; echo "rc=$?" >> gpurun_out/c16_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/c16_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/c16_bench_default.json 2> gpurun_out/c16_bench_default.err
timeout 900 python bench.py --impl reference > gpurun_out/c16_ref.json 2> gpurun_out/c16_ref.err
: > gpurun_out/c16_workloads.jsonl
for args in "--workload cfg1" "--workload cfg2" "--workload cfg3" "--workload cfg5" "--workload cfg2 --data doc_contiguous" \
            "--workload cfg4 --data doc_contiguous" "--workload cfg4 --queries 64"; do
  timeout 900 python bench.py --no-cpu-baseline --steps 10 --warmup 3 $args 2>>gpurun_out/c16_workloads.err | tail -1 >> gpurun_out/c16_workloads.jsonl
done
echo done > gpurun_out/C16DONE
