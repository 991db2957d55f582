#!/bin/bash
# compute-sanitizer memcheck over the round-2 additions (probe pass + fold kernel, drift limiter)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 compute-sanitizer --tool memcheck --leak-check no --print-limit 20 python -m pytest -q -x \
  "tests/test_gpu_probe.py::test_probe_ties_inside_probed_rows" "tests/test_gpu_probe.py::test_drift_limiter_shapes_match_oracle" \
  > gpurun_out/d10_memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/d10_memcheck.log
echo done > gpurun_out/D10DONE
