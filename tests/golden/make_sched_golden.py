"""Golden traces of the reference's stateful Scheduler (scheduler.py:194-469),
by RUNNING THE REFERENCE.  Dev container only (``/root/reference`` is absent on
the GPU box):  ``python tests/golden/make_sched_golden.py``.

Each scenario drives ``ragsched.scheduler.Scheduler`` with a seeded random
harness in the spirit of the reference's own stress test
(test_scheduler.py:321-395: submissions interleaved with completions of random
running calls, ``step`` after every event) and records every operation with
the reference's result — the admissions, the admitted calls, the completion
infos, the exceptions — plus the final ``Scheduler.trace``.  The replay test
(tests/test_gpu_scheduler.py) feeds the same operations to this package's
GPU-backed Scheduler and requires identical results.
"""

from __future__ import annotations

import gzip
import json
import os
import random
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from make_golden import FROM_BIT, PARAM_SETS, enc_space, params_kw, profile, random_arbitrary_space  # noqa: E402

from ragsched.mapping import IntRange, PrunedConfigSpace, map_profile  # noqa: E402
from ragsched.scheduler import PendingQuery, Scheduler, SchedulerParams  # noqa: E402
from ragsched.types import ModelSpec, QueryRecord  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "scheduler_traces.json.gz")
GiB = 1024 ** 3


def enc_adm(a):
    return [a.query_id, a.chosen_config.describe(), list(a.admitted_calls), list(a.deferred_calls), a.is_fallback]


def enc_call(c):
    return [c.query_id, c.call_index, c.prompt_tokens, c.max_output_tokens, c.kv_bytes]


def enc_info(i):
    return [i.query_done, i.config.describe(), i.is_fallback, list(i.newly_ready), i.winning_rerank]


def make_space(rng, mode, prof, mc):
    if mode == "mapped":
        return map_profile(prof, max_chunks=mc)
    if mode == "arbitrary":
        return random_arbitrary_space(rng, mc)
    if mode == "arbitrary35":  # chunk ranges beyond max_chunks: InvalidChunkCount from plan_calls
        return random_arbitrary_space(rng, 35)
    if mode == "fixed":  # single-candidate spaces for the fixed-config baseline
        m = rng.choice((1, 2, 4))
        n = rng.randint(1, min(mc, 12))
        il = rng.randint(30, 200)
        return PrunedConfigSpace(frozenset({FROM_BIT[m]}), IntRange(n, n), IntRange(il, il) if m == 4 else None)
    if mode == "fixed_bad":  # the baseline with a multi-candidate space somewhere
        if rng.random() < 0.9:
            return make_space(rng, "fixed", prof, mc)
        return map_profile(prof, max_chunks=mc)
    raise ValueError(mode)


def run(sc):
    rng = random.Random(sc["seed"])
    ps = PARAM_SETS[sc["ps"]]
    model0, meta, out, tmpl, mc, gran = params_kw(ps)
    model = ModelSpec(model0.num_layers, model0.num_kv_heads, model0.head_dim, model0.bytes_per_element,
                      max_context_tokens=sc.get("ctx", 131072))
    mc = sc.get("max_chunks", mc)
    params = SchedulerParams(model=model, meta=meta, out_budget=out, template_tokens=tmpl, max_chunks=mc,
                             granularity=gran, allow_fallback=sc.get("allow_fallback", True))
    sched = Scheduler(sc["capacity"], params)
    ops, running = [], []
    now, submitted, failed = 0.0, 0, False
    qlo, qhi = sc.get("qlen", (50, 2000))

    def pump():
        nonlocal failed
        try:
            adms, admitted = sched.step(now)
        except Exception as e:  # the reference raised: record and stop the scenario
            ops.append(["step", now, {"raise": [type(e).__name__, str(e)]}])
            failed = True
            return
        for ac in admitted:
            running.append((ac.query_id, ac.call_index))
        ops.append(["step", now, {"admissions": [enc_adm(a) for a in adms],
                                  "admitted": [enc_call(c) for c in admitted], "used": sched.used_bytes}])

    while not failed and (submitted < sc["n"] or running or sched.waiting or sched.active):
        now += 1.0
        if submitted < sc["n"] and (rng.random() < sc.get("p_submit", 0.6) or not running):
            burst = rng.randint(1, sc.get("burst", 1))
            for _ in range(min(burst, sc["n"] - submitted)):
                qid = f"q{submitted}"
                p = profile(rng.random() < 0.5, rng.random() < 0.5, rng.randint(1, 10),
                            *sorted((rng.randint(30, 200), rng.randint(30, 200))))
                space = make_space(rng, sc["mode"], p, mc)
                prof = None if rng.random() < sc.get("p_noprofile", 0.0) else p
                qlen = rng.randint(qlo, qhi)
                sched.submit(PendingQuery(query=QueryRecord(id=qid, text="t", query_token_len=qlen), space=space,
                                          arrival_time=now, profile=prof))
                ops.append(["submit", qid, qlen, list(enc_space(space)),
                            None if prof is None else [int(p.complexity_high), int(p.needs_joint_reasoning),
                                                       p.pieces_required, p.summary_len_range.low,
                                                       p.summary_len_range.high, p.confidence]])
                submitted += 1
            pump()
        elif running:
            if rng.random() < 0.03:  # a bogus completion: UnknownCall, state unchanged
                try:
                    sched.complete("nope", 0, now)
                except Exception as e:
                    ops.append(["complete", "nope", 0, now, None, {"raise": [type(e).__name__, str(e)]}])
            qid, idx = running.pop(rng.randrange(len(running)))
            conf = rng.random()
            info = sched.complete(qid, idx, now, rerank_confidence=conf)
            ops.append(["complete", qid, idx, now, conf, {"info": enc_info(info), "used": sched.used_bytes}])
            pump()
        else:
            break  # nothing running and the head can never be admitted (baseline deadlock guard)
    return {"name": sc["name"], "scenario": sc, "ops": ops, "trace": sched.trace, "failed": failed}


SCENARIOS = [
    dict(name="stress_s31_4g", seed=31, ps=1, capacity=4 * GiB, n=60, mode="mapped"),
    dict(name="stress_s77_1g", seed=77, ps=1, capacity=1 * GiB, n=60, mode="mapped"),
    dict(name="burst_s5_8g", seed=5, ps=0, capacity=8 * GiB, n=150, mode="mapped", burst=12, p_submit=0.35),
    dict(name="arbitrary_s11_2g", seed=11, ps=1, capacity=2 * GiB, n=80, mode="arbitrary", burst=4),
    dict(name="longdoc_s12_16g", seed=12, ps=2, capacity=16 * GiB, n=100, mode="mapped", qlen=(4000, 10000),
         burst=8),
    dict(name="summ_s13_16g", seed=13, ps=3, capacity=16 * GiB, n=100, mode="arbitrary", qlen=(4000, 12000),
         burst=8),
    dict(name="coarse_s14_3g", seed=14, ps=5, capacity=3 * GiB, n=80, mode="arbitrary", burst=5),
    dict(name="fp32cache_s15_6g", seed=15, ps=7, capacity=6 * GiB, n=80, mode="mapped", burst=3),
    dict(name="fixed_s16_4g", seed=16, ps=1, capacity=4 * GiB, n=60, mode="fixed", allow_fallback=False, burst=4),
    dict(name="fixed_s17_2g", seed=17, ps=0, capacity=2 * GiB, n=60, mode="fixed", allow_fallback=False, burst=6),
    # error paths (each ends at the reference's exception)
    dict(name="ctx_overflow_s18", seed=18, ps=1, capacity=16 * GiB, n=60, mode="mapped", ctx=5000, burst=3),
    dict(name="invalid_chunks_s19", seed=19, ps=1, capacity=8 * GiB, n=60, mode="arbitrary35", max_chunks=12),
    dict(name="no_profile_s20", seed=20, ps=1, capacity=1 * GiB, n=80, mode="mapped", p_noprofile=0.3, burst=6),
    dict(name="impossible_s21", seed=21, ps=2, capacity=GiB // 2, n=40, mode="mapped", qlen=(2000, 6000)),
    dict(name="fixed_bad_s22", seed=22, ps=1, capacity=8 * GiB, n=60, mode="fixed_bad", allow_fallback=False),
    dict(name="fixed_impossible_s23", seed=23, ps=2, capacity=GiB // 4, n=30, mode="fixed",
         allow_fallback=False, qlen=(3000, 6000)),
]


# -- the Scheduler as driven by the reference's own simulator (sim.run) ---------

def record_sim(name, mode, fixed=None, capacity=None, n=200, profile_name="single_hop_qa", out_budget=10):
    """Run ``ragsched.sim.run`` (the A-suite workload of test_acceptance.py:
    55-94) with a recording subclass of the reference Scheduler and keep its
    operations in the replay format."""
    import ragsched.sim as sim
    from ragsched.config import DEFAULT_CAPACITY_BYTES, DEFAULT_META, DEFAULT_MODEL
    from ragsched.profiler import NoiseParams
    from ragsched.sim import CostModel, PipelineParams, QualityModel
    from ragsched.workload import DATASET_PROFILES, ArrivalMode, ArrivalSpec, TruthDistribution, WorkloadSpec, \
        gen_workload

    ops = []

    class Recording(Scheduler):
        def submit(self, pending):
            p = pending.profile
            ops.append(["submit", pending.query.id, pending.query.query_token_len, list(enc_space(pending.space)),
                        None if p is None else [int(p.complexity_high), int(p.needs_joint_reasoning),
                                                p.pieces_required, p.summary_len_range.low,
                                                p.summary_len_range.high, p.confidence]])
            super().submit(pending)

        def step(self, now):
            adms, admitted = super().step(now)
            ops.append(["step", now, {"admissions": [enc_adm(a) for a in adms],
                                      "admitted": [enc_call(c) for c in admitted], "used": self.used_bytes}])
            return adms, admitted

        def complete(self, query_id, call_index, now, rerank_confidence=None):
            info = super().complete(query_id, call_index, now, rerank_confidence=rerank_confidence)
            ops.append(["complete", query_id, call_index, now, rerank_confidence,
                        {"info": enc_info(info), "used": self.used_bytes}])
            return info

    import ragsched.profiler as rprof

    gates = []
    orig_gate = rprof.QueryProfiler.gate

    def recording_gate(self, out):
        d = orig_gate(self, out)
        p = out.profile
        gates.append([[int(p.complexity_high), int(p.needs_joint_reasoning), p.pieces_required,
                       p.summary_len_range.low, p.summary_len_range.high, p.confidence],
                      [list(enc_space(d.space)), bool(d.used_fallback), d.confidence],
                      [self.threshold, list(enc_space(self.default_space)), self.max_chunks]])
        return d

    wl = gen_workload(WorkloadSpec(num_queries=n, arrival=ArrivalSpec(mode, 2.0),
                                   length_profile=DATASET_PROFILES[profile_name],
                                   truth_distribution=TruthDistribution()), 42)
    saved = sim.Scheduler
    sim.Scheduler = Recording
    rprof.QueryProfiler.gate = recording_gate
    try:
        report = sim.run(wl, DEFAULT_MODEL, capacity or DEFAULT_CAPACITY_BYTES, CostModel(), QualityModel(), 42,
                         PipelineParams(meta=DEFAULT_META, out_budget=out_budget, fixed_config=fixed,
                                        noise=NoiseParams()))
    finally:
        sim.Scheduler = saved
        rprof.QueryProfiler.gate = orig_gate
    sc = dict(name=name, sim=True, ps=0, capacity=capacity or DEFAULT_CAPACITY_BYTES,
              allow_fallback=fixed is None)
    return {"name": name, "scenario": sc, "ops": ops, "trace": report.trace, "failed": False,
            "results": len(report.results), "gates": gates}


if __name__ == "__main__":
    from ragsched.types import RagConfig, SynthesisMethod
    from ragsched.workload import ArrivalMode

    out = []
    for args in (("sim_adaptive_poisson", ArrivalMode.POISSON),
                 ("sim_adaptive_sequential", ArrivalMode.SEQUENTIAL),
                 ("sim_adaptive_poisson_2g", ArrivalMode.POISSON, None, 2 * GiB),
                 ("sim_fixed_st15_poisson", ArrivalMode.POISSON, RagConfig(SynthesisMethod.STUFF, 15)),
                 ("sim_fixed_mr8_poisson_1g", ArrivalMode.POISSON,
                  RagConfig(SynthesisMethod.MAP_REDUCE, 8, 100), GiB)):
        r = record_sim(*args)
        print(f"{r['name']:26s} ops={len(r['ops']):5d} trace={len(r['trace']):5d} results={r['results']} "
              f"gates={len(r['gates'])} gate fallbacks={sum(g[1][1] for g in r['gates'])}")
        out.append(r)
    for sc in SCENARIOS:
        r = run(sc)
        last = r["ops"][-1]
        print(f"{sc['name']:22s} ops={len(r['ops']):5d} trace={len(r['trace']):5d} "
              f"end={last[-1].get('raise', 'ok') if isinstance(last[-1], dict) else 'ok'}")
        out.append(r)
    with gzip.open(OUT, "wt") as f:
        json.dump(out, f)
    print("wrote", OUT, os.path.getsize(OUT), "bytes")
