#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 3000 python -m pytest -q tests -m gpu -x -s > gpurun_out/gputests4.log 2>&1
echo "gpu tests rc=$?" >> gpurun_out/gputests4.log
timeout 600 python tools/scalar_latency.py > gpurun_out/scalar_latency.txt 2>&1
timeout 900 python tools/dropin_sim.py > gpurun_out/dropin_sim.jsonl 2> gpurun_out/dropin_sim.err
