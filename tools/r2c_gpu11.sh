#!/bin/bash
# burst count posted by the last CTA (no stream copy); epilogue busy cycles of a unit's first tiles (profiling build)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest -q tests/test_gpu_bursts.py tests/test_gpu_retrieval.py tests/test_gpu_fp32_edges.py -x > gpurun_out/c11_t.log 2>&1; echo "rc=$?" >> gpurun_out/c11_t.log
for rep in 1 2; do
  timeout 600 python bench.py --workload cfg1 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/c11_cfg1_$rep.json 2> gpurun_out/c11_cfg1_$rep.err
  timeout 600 python bench.py --workload cfg1 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e --burst-merge off > gpurun_out/c11_cfg1off_$rep.json 2> /dev/null
  timeout 600 python bench.py --workload cfg2 --steps 40 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/c11_cfg2_$rep.json 2> gpurun_out/c11_cfg2_$rep.err
done
for a in "--workload cfg2 --data iso" "--workload cfg2 --data doc_contiguous" "--workload cfg4 --data iso" "--workload cfg1 --data iso" "--workload cfg3 --data iso"; do
  tag=$(echo $a | tr ' ' '_' | tr -d '-')
  RAGSCHED_B200_LIB=$PWD/paper_2412_10543_b200/_variants/prof.so timeout 600 python tools/pair_profile.py $a > gpurun_out/c11_prof$tag.txt 2>&1
done
echo done > gpurun_out/C11DONE
