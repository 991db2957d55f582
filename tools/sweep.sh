#!/bin/bash
# Run bench.py (device-resident timing only) for the default library and every
# tuning variant under paper_2412_10543_b200/_variants/ (GPU box).
# usage: tools/sweep.sh [bench args...]
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for lib in paper_2412_10543_b200/libragsched_b200.so paper_2412_10543_b200/_variants/*.so; do
  [ -e "$lib" ] || continue
  out=$(RAGSCHED_B200_LIB=$PWD/$lib timeout 600 python bench.py --no-cpu-baseline --no-e2e "$@" 2>&1 | tail -1)
  python - "$lib" "$out" <<'EOF'
import json, sys
lib, out = sys.argv[1], sys.argv[2]
try:
    d = json.loads(out)
    r = d["roofline"]
    print(f"{lib.split('/')[-1]:55s} {d['value']:10.0f} q/s  {r['achieved']:7.1f} {r['unit']}  "
          f"kernel {r['kernel_ms']:.2f} ms  sm {d['clocks']['sm_mhz']} MHz")
except Exception as e:
    print(lib, "FAILED", out[-300:])
EOF
done
