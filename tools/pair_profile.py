"""Per-role cycle accounting of the CTA-pair kernel (tuning build with
-DRS_PAIR_PROFILE=1, selected via RAGSCHED_B200_LIB).  Prints, for leader and
peer CTAs, the share of kernel time each role spends waiting."""

import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2412_10543_b200 import IndexFlatL2, _lib  # noqa: E402


def main(n=2_000_000, nq=8192, d=1024):
    lib = _lib.load()
    g = torch.Generator(device="cuda").manual_seed(0)
    c = torch.nn.functional.normalize(torch.randn(n, d, generator=g, device="cuda"), dim=1).bfloat16()
    q = torch.nn.functional.normalize(torch.randn(nq, d, generator=g, device="cuda"), dim=1).bfloat16()
    ix = IndexFlatL2(d, capacity=n)
    ix.add(c)
    ix.search_keys(q, 35)
    torch.cuda.synchronize()
    lib.rs_debug_pair_profile_reset()
    ix.search_keys(q, 35)
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * (1024 * 8))()
    lib.rs_debug_pair_profile(buf, 1024)
    a = np.frombuffer(buf, dtype=np.uint64).reshape(1024, 8).astype(np.float64)
    plan = ix.last_plan()
    ctas = 2 * plan["ctas"]
    a = a[:ctas]
    names = {0: "producer wait empty (ring full)", 1: "mma wait tempty (epilogue-bound)",
             2: "mma wait full (operand-bound)", 3: "epilogue wait tfull (4 warps)",
             5: "epilogue final flush (4 warps)", 4: "epilogue filter (4 warps)",
             6: "epilogue TMEM load wait (4 warps)"}
    for label, rows in (("leader", a[0::2]), ("peer", a[1::2])):
        # slot 7: every warp's lane 0 adds its elapsed cycles / 4 (4 epilogue
        # warps + TMEM, producer and MMA warps; the spare warp 4 exits at once)
        total = rows[:, 7] / 1.75
        print(f"{label}: kernel {total.mean() / 1e6:.2f} Mcycles")
        for i, nm in names.items():
            denom = total * (4 if i in (3, 4, 5, 6) else 1)
            print(f"   {nm:34s} {100 * (rows[:, i] / denom).mean():5.1f}%")
    print(plan)


if __name__ == "__main__":
    args = [int(x) for x in sys.argv[1:4]]
    main(*args)
