"""The reference's own simulator (``ragsched.sim.run``, sim.py:150-325) run
stock and with this package's GPU drop-in installed (``dropin.install``):
byte-identical report / summary / trace files (the A9 writers,
metrics.py:151-214) and the wall time per simulated query of each.

    python tools/dropin_sim.py           # prints one JSON object per scenario

Needs the reference installed in ``baseline/_ref`` (tools/install_reference.sh)
and a GPU for the drop-in half.  Used by tests/test_gpu_reference_sim.py.
"""

from __future__ import annotations

import json
import os
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

# (name, arrival mode, fixed config (method, n[, il]) or None, noise or None (default), capacity GiB, queries)
SCENARIOS = [
    ("poisson_adaptive", "poisson", None, None, 16, 200),
    ("poisson_fixed_stuff15", "poisson", ("stuff", 15), None, 16, 200),
    ("sequential_adaptive_zero_noise", "sequential", None, (0.0, 0.0, 0.0, 0.0), 16, 200),
    ("poisson_adaptive_a6_noise", "poisson", None, (0.1, 0.0, 0.0, 0.0), 16, 200),
    ("poisson_adaptive_2gib", "poisson", None, None, 2, 200),
    ("poisson_fixed_map_reduce8_1gib", "poisson", ("map_reduce", 8, 100), None, 1, 200),
    ("poisson_adaptive_doc_level_1000", "poisson", None, None, 16, 1000),
]


def run(rs, mode: str, fixed=None, noise=None, capacity_gib: int = 16, n: int = 200, seed: int = 42,
        lengths: str = "single_hop_qa"):
    """One ``sim.run`` through whatever the reference module attributes are
    bound to right now (stock or drop-in)."""
    W, T, C, P = rs.workload, rs.types, rs.config, rs.profiler
    if n == 1000:
        lengths = "doc_level_qa"
    wl = W.gen_workload(W.WorkloadSpec(num_queries=n, arrival=W.ArrivalSpec(W.ArrivalMode(mode), 2.0),
                                       length_profile=W.DATASET_PROFILES[lengths],
                                       truth_distribution=W.TruthDistribution()), seed)
    cfg = None
    if fixed is not None:
        cfg = T.RagConfig(T.SynthesisMethod(fixed[0]), *fixed[1:])
    params = rs.sim.PipelineParams(meta=C.DEFAULT_META, out_budget=W.DATASET_PROFILES[lengths].out_budget,
                                   fixed_config=cfg,
                                   noise=P.NoiseParams(*noise) if noise is not None else P.NoiseParams())
    return rs.sim.run(wl, C.DEFAULT_MODEL, capacity_gib * 1024 ** 3, rs.sim.CostModel(), rs.sim.QualityModel(),
                      seed, params)


def report_bytes(rs, report) -> bytes:
    M = rs.metrics
    with tempfile.TemporaryDirectory() as d:
        r, s, t = (os.path.join(d, x) for x in ("report.jsonl", "summary.tsv", "trace.jsonl"))
        M.write_report(report, r)
        M.write_summary([M.summarize(report)], s)
        M.write_trace(report.trace, t)
        return b"\n--\n".join(open(p, "rb").read() for p in (r, s, t))


def compare(rs, scenario, repeats: int = 1) -> dict:
    """Stock vs drop-in on one scenario: identical bytes? wall s per query."""
    from paper_2412_10543_b200 import dropin

    name, mode, fixed, noise, cap, n = scenario
    t0 = time.perf_counter()
    for _ in range(repeats):
        stock = report_bytes(rs, run(rs, mode, fixed, noise, cap, n))
    t_stock = (time.perf_counter() - t0) / repeats
    originals = dropin.install(rs)
    try:
        run(rs, mode, fixed, noise, cap, min(n, 20))  # warm-up: CUDA context, library, allocator
        t0 = time.perf_counter()
        for _ in range(repeats):
            gpu = report_bytes(rs, run(rs, mode, fixed, noise, cap, n))
        t_gpu = (time.perf_counter() - t0) / repeats
    finally:
        dropin.uninstall(originals)
    return {"scenario": name, "queries": n, "identical": stock == gpu, "report_bytes": len(stock),
            "stock_us_per_query": 1e6 * t_stock / n, "dropin_us_per_query": 1e6 * t_gpu / n,
            "dropin_over_stock": t_gpu / t_stock}


def main():
    from oracle import refpath

    rs = refpath.import_ragsched()
    for sc in SCENARIOS:
        print(json.dumps(compare(rs, sc, repeats=2)), flush=True)


if __name__ == "__main__":
    main()
