"""Measure the fp32-path peaks the cfg1 roofline needs, the way the driver
measures MEASURED_PEAKS.json (torch.matmul 8192^3, best of 10 = burst, back to
back for 4 s = sustained, CUDA events):

* tf32 tensor-core GEMM (cuBLAS, allow_tf32) — the denominator of the
  3xTF32 kernel (3 tf32 MMAs per fp32 product);
* fp32 SGEMM on the CUDA cores (FFMA pipe, allow_tf32 off) — the exact-fp32
  alternative;
* bf16 GEMM as a cross-check against MEASURED_PEAKS.json.

Writes profiles/fp32_peaks.json.
"""

from __future__ import annotations

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def gemm_peak(dtype, tf32: bool, n=8192, sustain_s=4.0):
    import torch

    torch.backends.cuda.matmul.allow_tf32 = tf32
    torch.backends.cudnn.allow_tf32 = tf32
    a = torch.randn(n, n, device="cuda", dtype=dtype)
    b = torch.randn(n, n, device="cuda", dtype=dtype)
    flop = 2.0 * n ** 3
    for _ in range(3):
        a @ b
    torch.cuda.synchronize()
    best = 0.0
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        a @ b
        e1.record()
        torch.cuda.synchronize()
        best = max(best, flop / (e0.elapsed_time(e1) * 1e-3) / 1e12)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps, t0 = 0, time.perf_counter()
    e0.record()
    while time.perf_counter() - t0 < sustain_s:
        for _ in range(8):
            a @ b
        reps += 8
        torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    sus = flop * reps / (e0.elapsed_time(e1) * 1e-3) / 1e12
    torch.backends.cuda.matmul.allow_tf32 = False
    return round(best, 1), round(sus, 1)


def main():
    import torch

    out = {"gpu": torch.cuda.get_device_name(0), "how": "torch.matmul 8192^3 (2 N^3 flop): best of 10 (burst), "
           "back to back for 4 s (sustained), CUDA events"}
    out["tf32_tflops"], out["tf32_tflops_sustained"] = gemm_peak(torch.float32, True)
    out["fp32_ffma_tflops"], out["fp32_ffma_tflops_sustained"] = gemm_peak(torch.float32, False)
    out["bf16_tflops"], out["bf16_tflops_sustained"] = gemm_peak(torch.bfloat16, False)
    out["exact_fp32_via_3xtf32_tflops"] = round(out["tf32_tflops"] / 3, 1)
    out["exact_fp32_via_3xtf32_tflops_sustained"] = round(out["tf32_tflops_sustained"] / 3, 1)
    path = os.path.join(ROOT, "profiles", "fp32_peaks.json")
    json.dump(out, open(path, "w"), indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
