#!/bin/bash
# automatic lean / cooperative pair-kernel variant: tests, then interleaved A/B of auto vs forced on / off
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest -q tests/test_gpu_bursts.py tests/test_gpu_retrieval.py tests/test_gpu_fuzz.py -x > gpurun_out/c9_t.log 2>&1; echo "rc=$?" >> gpurun_out/c9_t.log
for rep in 1 2 3; do
for m in auto off on; do
  timeout 600 python bench.py --workload cfg2 --data iso --steps 40 --warmup 5 --no-e2e --no-cpu-baseline --burst-merge $m \
      > gpurun_out/c9_${m}_cfg2_iso_$rep.json 2> gpurun_out/c9_${m}_cfg2_iso_$rep.err
  timeout 600 python bench.py --workload cfg4 --steps 8 --warmup 3 --no-e2e --no-cpu-baseline --burst-merge $m \
      > gpurun_out/c9_${m}_cfg4_iso_$rep.json 2> gpurun_out/c9_${m}_cfg4_iso_$rep.err
  if [ $rep -le 2 ]; then
  timeout 600 python bench.py --workload cfg2 --data doc_contiguous --steps 40 --warmup 5 --no-e2e --no-cpu-baseline --burst-merge $m \
      > gpurun_out/c9_${m}_cfg2_doc_$rep.json 2> gpurun_out/c9_${m}_cfg2_doc_$rep.err
  fi
done
done
echo done > gpurun_out/C9DONE
