"""Per-role cycle accounting and epilogue event counts of the CTA-pair kernel
(tuning build with -DRS_PAIR_PROFILE=1, selected via RAGSCHED_B200_LIB):

    python -c "from paper_2412_10543_b200 import build as b; \
        b.build(defines=('RS_PAIR_PROFILE=1',), out='paper_2412_10543_b200/_variants/prof.so')"
    RAGSCHED_B200_LIB=$PWD/paper_2412_10543_b200/_variants/prof.so \
        python tools/pair_profile.py --workload cfg2 --data doc_contiguous

Prints, for leader and peer CTAs, the share of kernel time each role spends
waiting, then the epilogue's event counts per (query row, corpus tile):
slow-path 8-column groups (some lane of the warp passed the dot bound),
candidate appends, buffer flushes and warp insert steps.  One JSON line at
the end (for profiles/)."""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2412_10543_b200 import IndexFlatL2, _lib  # noqa: E402
from tools import synth  # noqa: E402

SLOTS = 16
NAMES = {0: "producer wait empty (ring full)", 1: "mma wait tempty (epilogue-bound)",
         2: "mma wait full (operand-bound)", 3: "epilogue wait tfull (4 warps)",
         5: "epilogue final flush (4 warps)", 4: "epilogue filter (4 warps)",
         6: "epilogue TMEM load wait (4 warps)"}
COUNTERS = {8: "slow-path groups", 9: "appends", 10: "flushes", 11: "insert steps", 12: "cooperative merges"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg2")
    ap.add_argument("--data", default="iso", choices=synth.DATA)
    ap.add_argument("--rows", type=int, default=None)
    ap.add_argument("--queries", type=int, default=None)
    ap.add_argument("--k", type=int, default=35)
    ap.add_argument("--probe", default="off", choices=("on", "off"))
    a = ap.parse_args()
    import bench

    cfg = dict(bench.WORKLOADS[a.workload])
    n, nq, d = a.rows or cfg["n"], a.queries or cfg["nq"], cfg["d"]
    dt = torch.bfloat16 if cfg["dtype"] == "bf16" else torch.float32
    lib = _lib.load()
    if not hasattr(lib, "rs_debug_pair_profile"):
        raise SystemExit("needs the RS_PAIR_PROFILE=1 build (RAGSCHED_B200_LIB)")
    lib.rs_debug_pair_profile.argtypes = [ctypes.c_void_p, ctypes.c_int]
    ix = IndexFlatL2(d, dtype=dt, capacity=n)
    ix.set_probe(a.probe)
    for r0 in range(0, n, 1 << 20):
        ix.add(synth.corpus_rows(r0, min(n, r0 + (1 << 20)), d, 0, dt, "cuda", a.data))
    q = synth.make_queries(nq, n, d, 0, dt, a.data).cuda()
    ix.search_keys(q, a.k)
    torch.cuda.synchronize()
    lib.rs_debug_pair_profile_reset()
    ix.search_keys(q, a.k)
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * (1024 * SLOTS))()
    lib.rs_debug_pair_profile(ctypes.addressof(buf), 1024)
    arr = np.frombuffer(buf, dtype=np.uint64).reshape(1024, SLOTS).astype(np.float64)
    plan = ix.last_plan()
    arr = arr[:2 * plan["ctas"]]
    out = {"workload": a.workload, "data": a.data, "rows": n, "queries": nq, "dim": d, "plan": plan}
    for label, rows in (("leader", arr[0::2]), ("peer", arr[1::2])):
        # slot 7: every warp's lane 0 adds its elapsed cycles (epilogue warps / 4)
        total = rows[:, 7] / 1.75
        out[label] = {"mcycles": round(total.mean() / 1e6, 3)}
        print(f"{label}: kernel {total.mean() / 1e6:.2f} Mcycles")
        for i, nm in NAMES.items():
            denom = total * (4 if i in (3, 4, 5, 6) else 1)
            share = 100 * (rows[:, i] / denom).mean()
            out[label][nm] = round(share, 2)
            print(f"   {nm:34s} {share:5.1f}%")
    # (query row, tile) visits: every row of every query tile meets every corpus
    # tile once (the counters also hold the probe launch's tiles, if any)
    out["probe_rows"] = ix.last_probe_rows()
    tiles = -(-n // 256) + out["probe_rows"] // 256
    rows_total = plan["qtiles"] * (256 if nq > 128 else 128)
    warp_tiles = rows_total / 32 * tiles
    c = arr[:, 8:13].sum(0)
    out["per_warp_tile"] = {nm: round(float(c[i - 8]) / warp_tiles, 4) for i, nm in COUNTERS.items()}
    out["appends_per_query"] = round(float(c[1]) / nq, 1)
    busy_early, busy_all, n_early = arr[:, 13].sum(), arr[:, 14].sum(), arr[:, 15].sum()
    if busy_all > 0:
        out["epilogue_busy"] = {"first4_share": round(float(busy_early / busy_all), 4),
                                "first4_cycles_per_tile": round(float(busy_early / max(n_early, 1)), 1),
                                "other_cycles_per_tile": round(float((busy_all - busy_early) /
                                                                     max(warp_tiles - n_early, 1)), 1),
                                "first4_tile_share": round(float(n_early / warp_tiles), 4)}
        print("epilogue busy cycles:", out["epilogue_busy"])
    print("epilogue events per (32 query rows, 256-row corpus tile):", out["per_warp_tile"])
    print("candidate appends per query:", out["appends_per_query"])
    print(json.dumps(out))


if __name__ == "__main__":
    main()
