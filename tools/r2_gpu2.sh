#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
( time timeout 1200 python bench.py --impl reference --steps 20 --warmup 5 ) > gpurun_out/ref_cfg4.json 2> gpurun_out/ref_cfg4.err
timeout 600 python bench.py --workload cfg5 --steps 20 --warmup 5 > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
( time timeout 600 python bench.py --impl reference --workload cfg5 --steps 20 --warmup 5 ) > gpurun_out/ref_cfg5.json 2> gpurun_out/ref_cfg5.err
