#!/bin/bash
# round-2 re-entry: full GPU suite + smoke, the default bench line, the reference arm,
# the data-robustness matrix, and the launch list of the default bench
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > gpurun_out/smi.txt 2>&1
( time timeout 2400 python -m pytest -q tests -m gpu -rs ) > gpurun_out/gputests.log 2>&1
echo "gpu tests rc=$?" >> gpurun_out/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
( time timeout 900 python bench.py --steps 20 --warmup 5 ) > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err
( time timeout 1500 python bench.py --impl reference --steps 20 --warmup 5 ) > gpurun_out/ref_cfg4.json 2> gpurun_out/ref_cfg4.err
bash tools/r2_data.sh
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
   --log-file gpurun_out/launches_cfg4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
echo done > gpurun_out/ALLDONE
