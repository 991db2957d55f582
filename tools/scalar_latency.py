"""Per-call wall time of the scalar drop-in functions against the reference's
own (pure Python) functions, plus a cProfile of one drop-in sim.run.

    python tools/scalar_latency.py
"""

from __future__ import annotations

import cProfile
import io
import json
import os
import pstats
import random
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def bench(fn, args_list, reps=1):
    for a in args_list[:50]:
        fn(*a)
    t0 = time.perf_counter()
    for _ in range(reps):
        for a in args_list:
            fn(*a)
    return 1e6 * (time.perf_counter() - t0) / (reps * len(args_list))


def main():
    from oracle import refpath
    from paper_2412_10543_b200 import dropin

    rs = refpath.import_ragsched()
    M, P, S, Mem, Sim, T, C = rs.mapping, rs.profiler, rs.scheduler, rs.memory, rs.sim, rs.types, rs.config
    rng = random.Random(0)
    profs = [M.QueryProfile(rng.random() < .5, rng.random() < .5, rng.randint(1, 10),
                            T.IntRange(*sorted((rng.randint(30, 200), rng.randint(30, 200)))), 0.95)
             for _ in range(2000)]
    qs = [T.QueryRecord(id=f"q{i}", text="t", query_token_len=rng.randint(10, 3000)) for i in range(2000)]
    spaces = [M.map_profile(p) for p in profs]
    frees = [rng.randint(0, 40 * 1024 ** 3) for _ in range(2000)]
    kw = dict(model=C.DEFAULT_MODEL, meta=C.DEFAULT_META, out_budget=10)
    cfgs = [T.RagConfig(T.SynthesisMethod.STUFF, rng.randint(1, 35)) for _ in range(2000)]
    calls = [Mem.plan_calls(q, c, C.DEFAULT_META, C.DEFAULT_MODEL, 10).calls[0] for q, c in zip(qs, cfgs)]
    outs = [P.ProfilerOutput(profile=p, raw_text="", per_field_confidence={}) for p in profs]

    def suite():
        win = P.RecentSpaceWindow()
        return {
            "map_profile": bench(lambda p: M.map_profile(p), [(p,) for p in profs]),
            "gate_profile": bench(lambda o: P.gate_profile(o, win), [(o,) for o in outs]),
            "best_fit_select": bench(lambda s, q, f: S.best_fit_select(s, q, f, **kw),
                                     list(zip(spaces, qs, frees))),
            "fallback_config": bench(lambda p, q, f: S.fallback_config(p, q, f, **kw), list(zip(profs, qs, frees))),
            "plan_bytes": bench(lambda q, c: Mem.plan_bytes(q.query_token_len, c, 1000, 131072, 10), list(zip(qs, cfgs))),
            "call_latency": bench(lambda c: Sim.call_latency(c, 3, Sim.CostModel()), [(c,) for c in calls]),
        }

    stock = suite()
    orig = dropin.install(rs)
    gpu = suite()
    from tools import dropin_sim

    dropin_sim.run(rs, "poisson", n=20)
    pr = cProfile.Profile()
    pr.enable()
    dropin_sim.run(rs, "poisson", n=200)
    pr.disable()
    dropin.uninstall(orig)
    for k in stock:
        print(json.dumps({"function": k, "stock_us": round(stock[k], 2), "dropin_us": round(gpu[k], 2)}))
    s = io.StringIO()
    pstats.Stats(pr, stream=s).sort_stats("cumulative").print_stats(35)
    print(s.getvalue())
    s = io.StringIO()
    pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(25)
    print(s.getvalue())


if __name__ == "__main__":
    main()
