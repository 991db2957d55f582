"""One fused search at a bench shape (for ncu): builds the tools/synth.py
corpus on the device, runs ``--warmup`` searches, then ``--reps`` more.

    ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum -k regex:score_topk_pair \\
        --launch-skip 2 -c 1 python tools/one_search.py --workload cfg4
"""

from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import bench
    from paper_2412_10543_b200 import IndexFlatL2
    from tools import synth

    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg4")
    ap.add_argument("--queries", type=int, default=None)
    ap.add_argument("--corpus-rows", type=int, default=None)
    ap.add_argument("--segment-rows", type=int, default=0)
    ap.add_argument("--data", default="iso")
    ap.add_argument("--probe", default="off", choices=("on", "off"))
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--reps", type=int, default=1)
    ap.add_argument("--persist-mb", type=int, default=0,
                    help="experiment: cudaLimitPersistingL2CacheSize (evict_last lines are protected inside it)")
    a = ap.parse_args()
    if a.persist_mb:
        import ctypes
        import glob

        import torch

        torch.cuda.init()
        libs = glob.glob(os.path.join(os.path.dirname(torch.__file__), "lib", "libcudart*.so*")) + \
            glob.glob("/usr/local/cuda/lib64/libcudart.so*")
        rt = ctypes.CDLL(libs[0])
        rc = rt.cudaDeviceSetLimit(ctypes.c_int(0x06), ctypes.c_size_t(a.persist_mb << 20))
        print("cudaDeviceSetLimit(PersistingL2CacheSize) rc", rc, "via", libs[0])
    cfg = dict(bench.WORKLOADS[a.workload])
    if a.queries:
        cfg["nq"] = a.queries
    if a.corpus_rows:
        cfg["n"] = a.corpus_rows
    dt = torch.bfloat16 if cfg["dtype"] == "bf16" else torch.float32
    dev = torch.device("cuda", 0)
    ix = IndexFlatL2(cfg["d"], dtype=dt, capacity=cfg["n"])
    ix.set_probe(a.probe)
    if a.segment_rows:
        ix.set_segment_rows(a.segment_rows)
    for r in range(0, cfg["n"], 1 << 20):
        ix.add(synth.corpus_rows(r, min(cfg["n"], r + (1 << 20)), cfg["d"], bench.SEED, dt, dev, a.data))
    q = synth.make_queries(cfg["nq"], cfg["n"], cfg["d"], bench.SEED, dt, a.data).to(dev)
    for _ in range(a.warmup + a.reps):
        ix.search_keys(q, bench.K)
    torch.cuda.synchronize()
    print("plan", ix.last_plan())


if __name__ == "__main__":
    main()
