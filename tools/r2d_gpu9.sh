#!/bin/bash
# end of round 2: full GPU suite, smoke, default bench + reference arm (driver args), timed-region launch list,
# ncu --set full of the pair kernel at nq 512 (drift limiter on)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/d9_tests.log 2>&1; echo "rc=$?" >> gpurun_out/d9_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/d9_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/d9_smoke.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/d9_bench.json 2> gpurun_out/d9_bench.err
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/d9_ref.json 2> gpurun_out/d9_ref.err
timeout 900 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/d9_launches_cfg4.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/d9_l4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:score_topk_pair --launch-skip 2 -c 1 \
  -o gpurun_out/d9_pair_q512 python tools/one_search.py --workload cfg4 --queries 512 > gpurun_out/d9_ncu_q512.log 2>&1
echo done > gpurun_out/D9DONE
